"""The drop-in boundary: the reference's hot-path entry points
exist under the same names with the same parameter names, order and defaults
(restated from the reference signatures cited per entry), and the result
types keep the reference's fields.  CPU only (no kernel is called)."""

import inspect

import paper_1612_08825_b200 as ct
from paper_1612_08825_b200 import BoundaryPolicy, ConvMethod, ConvShape

E = inspect.Parameter.empty

# name -> [(parameter, default)], reference file:line of the signature
SIGNATURES = {
    "conv_direct": [("signal", E), ("kernel", E), ("shape", ConvShape.FULL), ("boundary", BoundaryPolicy.ZERO)],  # conv.py:157
    "xcorr_direct": [("signal", E), ("kernel", E), ("shape", ConvShape.FULL), ("boundary", BoundaryPolicy.ZERO)],  # conv.py:153
    "conv_auto": [("signal", E), ("kernel", E), ("shape", ConvShape.FULL), ("boundary", BoundaryPolicy.ZERO),
                  ("method", ConvMethod.AUTO), ("threshold", None)],  # conv.py:183
    "derivatives_3d": [("pair", E)],  # ttc.py:82
    "radial_gradient": [("ex", E), ("ey", E)],  # ttc.py:94
    "build_normal_system": [("ex", E), ("ey", E), ("g", E), ("et", E), ("border", 1)],  # ttc.py:102
    "solve_ttc": [("system", E), ("c_min", 1e-9)],  # ttc.py:157
    "downsample": [("img", E)],  # ttc.py:187
    "estimate_fixed": [("pair", E), ("level", 0), ("c_min", 1e-9)],  # ttc.py:228
    "estimate_multiscale": [("pair", E), ("max_level", 5), ("c_min", 1e-9)],  # ttc.py:248
    "run_sequence": [("frames", E), ("level", 0), ("max_level", None), ("c_min", 1e-9)],  # ttc.py:282
}


def test_entry_point_signatures_match_the_reference():
    for name, params in SIGNATURES.items():
        fn = getattr(ct, name)
        sig = inspect.signature(fn)
        got = [(p.name, p.default) for p in sig.parameters.values()][: len(params)]
        assert got == params, (name, got)
        # any extra parameters of ours are keyword extensions with defaults
        for p in list(sig.parameters.values())[len(params):]:
            assert p.default is not E, (name, p.name)


def test_result_types_keep_the_reference_fields():
    # TtcEstimate (ttc.py:68-79), NormalSystem (ttc.py:54-65), FramePair (ttc.py:41-51)
    est_fields = ("a", "b", "c", "x0", "y0", "ttc", "residual", "misfit", "level", "degenerate")
    assert tuple(ct.TtcEstimate.__dataclass_fields__)[: len(est_fields)] == est_fields
    assert tuple(ct.NormalSystem.__dataclass_fields__)[:4] == ("m", "rhs", "et2", "count")
    assert tuple(ct.FramePair.__dataclass_fields__)[:2] == ("first", "second")
    assert {m.name for m in ConvShape} >= {"FULL", "SAME", "VALID"}
    assert {m.name for m in BoundaryPolicy} >= {"ZERO", "REPLICATE"}
    assert {m.name for m in ConvMethod} >= {"AUTO", "DIRECT", "FFT"}
