"""paper_1612_08825_b200: the B200-native (sm_100a) hot path of convtact.

Drop-in for the convolution and time-to-contact entry points of the reference
package convtact (/root/reference/pkg/src/convtact/__init__.py:10-40): same
names, signatures and semantics, computed by hand-written CUDA kernels in
libconvtact_b200.so behind the C ABI of include/convtact_b200.h.  Out of scope
(host orchestration, not data-parallel compute): the CLI, NDT/PGM codecs,
the CPU bench/calibration harness and the FFT backend (conv_auto keeps the
reference's AUTO decision and tag, both executed by the direct kernels).
"""

from .conv import (
    DEFAULT_AUTO_THRESHOLD,
    BoundaryPolicy,
    ConvMethod,
    ConvPlan,
    ConvShape,
    conv_auto,
    conv_direct,
    direct_batch,
    reflect,
    xcorr_direct,
)
from .ingest import FormatError, image_read_pgm, image_write_pgm, tensor_read
from .kernels import KERNELS, GradientField, NamedKernel, gradient, kernel_lookup
from .synth import (
    ScoreReport,
    SynthConfig,
    SyntheticSequence,
    approach_stream,
    generate,
    make_texture,
    make_texture_device,
    make_textures,
    score_mse,
    write_sequence,
    zoom_frame,
    zoom_frames,
)
from .ttc import (
    TRACE_HEADER,
    FramePair,
    NormalSystem,
    TtcEstimate,
    build_normal_system,
    derivatives_3d,
    downsample,
    estimate_fixed,
    estimate_multiscale,
    radial_gradient,
    run_sequence,
    run_sequence_batch,
    pyramid_moments,
    run_sequence_host,
    solve_ttc,
    trace_lines,
    write_trace,
)

__version__ = "0.1.0"
