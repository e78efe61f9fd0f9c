"""Synthetic approach sequences generated on the device (inputs for tests and the benchmark).

Mirrors convtact.synth (/root/reference/pkg/src/convtact/synth.py):
  * make_texture: PCG64(seed) uniform noise (drawn on the host with numpy's
    generator, the same stream as the reference), two 3x3 binomial SAME /
    REPLICATE passes through this package's conv engine on the device, then
    a min-max rescale (synth.py:68-85);
  * zoom frames: separable Catmull-Rom magnification about the FOE, done by
    ct_zoom_frames (synth.py:88-126), bit-identical in float64;
  * generate(SynthConfig) -> SyntheticSequence(frames, truth, config):
    frames t = 0..frames-1 with magnification t0 / (t0 - t)
    (synth.py:129-143); sensor noise from the independent
    PCG64(SeedSequence([seed, 1])) stream when noise_sigma > 0;
  * score_mse: the trace-vs-truth MSE report (synth.py:186-208).

approach_stream() implements the long-video rule used for BASELINE config 5
(SURVEY.md D3): the reference forbids frames >= t0, so a 1024-frame stream is
a sequence of approach segments, each with its own seeded texture and
T0 ~ U[50, 500], cut while the true time to contact is still >= 20 frames.
"""

from __future__ import annotations

import csv
import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .conv import BoundaryPolicy, ConvShape, direct_batch

_B3 = np.outer(*(2 * [np.array([1.0, 2.0, 1.0]) / 4.0]))


@dataclass(frozen=True)
class SynthConfig:
    width: int = 256
    height: int = 256
    frames: int = 60
    t0: float = 100.0
    foe: tuple[float, float] = (0.4, 0.55)
    seed: int = 1
    noise_sigma: float = 0.0

    def __post_init__(self):  # synth.py:40-55
        if self.width < 16 or self.height < 16:
            raise ValueError(f"size {self.width}x{self.height} too small, need >= 16")
        if self.frames < 2:
            raise ValueError("need at least 2 frames")
        if not self.t0 > 0:
            raise ValueError("t0 must be positive")
        if self.frames >= self.t0:
            raise ValueError(f"frames ({self.frames}) must stay short of contact at t0 ({self.t0})")
        fx, fy = self.foe
        if not (0.0 < fx < 1.0 and 0.0 < fy < 1.0):
            raise ValueError(f"foe fractions must lie inside (0, 1), got {self.foe}")
        if self.noise_sigma < 0:
            raise ValueError("noise_sigma must be >= 0")

    @property
    def foe_px(self) -> tuple[float, float]:
        return self.foe[0] * self.width, self.foe[1] * self.height


def make_texture_device(width: int, height: int, seed: int, device="cuda") -> torch.Tensor:
    """Band-limited random texture in [0, 1] as a float64 CUDA tensor (synth.py:68-85)."""
    if width < 16 or height < 16:
        raise ValueError(f"texture {width}x{height} too small, need >= 16")
    rng = np.random.Generator(np.random.PCG64(seed))
    img = torch.from_numpy(rng.random((height, width))).to(device)
    for _ in range(2):
        img = direct_batch(img[None], _B3, ConvShape.SAME, BoundaryPolicy.REPLICATE, flip=False)[0]
    lo, hi = img.min(), img.max()
    if not bool(hi > lo):
        return torch.zeros_like(img)
    return (img - lo) / (hi - lo)


def make_texture(width: int, height: int, seed: int) -> np.ndarray:
    """synth.make_texture (synth.py:68-85): the texture as a float64 numpy array
    (computed on the device; make_texture_device keeps it there)."""
    return make_texture_device(width, height, seed).cpu().numpy()


def make_textures(width: int, height: int, seeds, device="cuda") -> torch.Tensor:
    """make_texture for many seeds at once: [len(seeds), height, width] float64.

    Same values as make_texture per seed (one batched conv launch per
    smoothing pass, batched min/max), for generating benchmark inputs.
    """
    if width < 16 or height < 16:
        raise ValueError(f"texture {width}x{height} too small, need >= 16")
    noise = np.stack([np.random.Generator(np.random.PCG64(s)).random((height, width)) for s in seeds])
    img = torch.from_numpy(noise).to(device)
    for _ in range(2):
        img = direct_batch(img, _B3, ConvShape.SAME, BoundaryPolicy.REPLICATE, flip=False)
    lo = img.amin(dim=(1, 2), keepdim=True)
    hi = img.amax(dim=(1, 2), keepdim=True)
    flat = (hi <= lo)
    out = (img - lo) / torch.where(flat, torch.ones_like(hi), hi - lo)
    return torch.where(flat, torch.zeros_like(out), out)


def zoom_frames(texture: torch.Tensor, foe_px, mags, dtype=torch.float64, out: torch.Tensor | None = None):
    """frames[t] = zoom_frame(texture, foe_px, mags[t]) on the device -> [len(mags), h, w]."""
    tex = texture.contiguous()
    if tex.dtype != torch.float64 or not tex.is_cuda:
        raise TypeError("texture must be a float64 CUDA tensor")
    h, w = tex.shape
    m = np.ascontiguousarray(mags, dtype=np.float64)
    if out is None:
        out = torch.empty((len(m), h, w), dtype=dtype, device=tex.device)
    L = _lib.load()
    _lib.check(L.ct_zoom_frames(_lib.dtype_code(out), _lib.ptr(tex), h, w, float(foe_px[0]), float(foe_px[1]),
                                m.ctypes.data_as(ctypes.c_void_p), len(m), _lib.ptr(out), None, 0,
                                _lib.stream_ptr()))
    return out


def zoom_frame(texture, foe_px, magnification: float):
    """synth.zoom_frame (synth.py:110-126): magnify about foe_px with edge
    clamping, on the device.  numpy in -> numpy out; a CUDA tensor stays."""
    if magnification < 1.0:
        raise ValueError(f"magnification must be >= 1, got {magnification}")
    on_dev = isinstance(texture, torch.Tensor) and texture.is_cuda
    tex = texture.to(torch.float64) if on_dev else torch.from_numpy(np.ascontiguousarray(texture, dtype=np.float64)).cuda()
    out = zoom_frames(tex, foe_px, [float(magnification)])[0]
    return out if on_dev else out.cpu().numpy()


@dataclass(frozen=True)
class SyntheticSequence:
    """synth.SyntheticSequence (synth.py:61-65).  ``frames`` is a numpy array
    from generate(cfg) and a CUDA tensor from generate(cfg, device=True)."""

    frames: object
    truth: np.ndarray  # rows (frame, ttc, foe_x, foe_y), FOE in array pixels
    config: SynthConfig


def generate(cfg: SynthConfig, device: bool = False, dtype=torch.float64) -> SyntheticSequence:
    """synth.generate (synth.py:129-143) with the frames zoomed on the device.

    Default: the reference's result, frames a float64 numpy array.  With
    device=True the frames stay on the GPU as a ``dtype`` CUDA tensor
    (rounded from float64; the benchmark / test input path)."""
    tex = make_texture_device(cfg.width, cfg.height, cfg.seed)
    mags = [cfg.t0 / (cfg.t0 - t) for t in range(cfg.frames)]
    frames = zoom_frames(tex, cfg.foe_px, mags, dtype=torch.float64)
    if cfg.noise_sigma > 0:
        noise_rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([cfg.seed, 1])))
        for t in range(cfg.frames):
            noise = torch.from_numpy(noise_rng.normal(0.0, cfg.noise_sigma, (cfg.height, cfg.width))).to(frames.device)
            frames[t] = torch.clamp(frames[t] + noise, 0.0, 1.0)
    fx, fy = cfg.foe_px
    truth = np.array([(t, cfg.t0 - t, fx, fy) for t in range(cfg.frames)], dtype=np.float64).reshape(-1, 4)
    out = frames.to(dtype) if device else frames.cpu().numpy()
    return SyntheticSequence(frames=out, truth=truth, config=cfg)


TRUTH_HEADER = "frame,ttc,foe_x,foe_y"


def write_sequence(seq: SyntheticSequence, outdir) -> None:
    """synth.write_sequence (synth.py:149-162): frame_%06d.pgm per frame plus
    truth.csv (host I/O; device frames are copied back)."""
    from pathlib import Path

    from .ingest import image_write_pgm
    out = Path(outdir)
    out.mkdir(parents=True, exist_ok=True)
    frames = seq.frames.detach().cpu().numpy() if isinstance(seq.frames, torch.Tensor) else seq.frames
    for t in range(frames.shape[0]):
        image_write_pgm(frames[t], out / f"frame_{t:06d}.pgm")
    lines = [TRUTH_HEADER] + [f"{int(r[0])},{format(r[1], '.17g')},{format(r[2], '.17g')},{format(r[3], '.17g')}"
                              for r in seq.truth]
    with open(out / "truth.csv", "w", newline="\n") as f:
        f.write("\n".join(lines) + "\n")


@dataclass(frozen=True)
class ScoreReport:
    mse: float
    compared: int
    excluded: int


def _read_ttc_column(path):  # synth.py:172-183
    with open(path, newline="") as f:
        reader = csv.DictReader(f)
        if reader.fieldnames is None or "frame" not in reader.fieldnames or "ttc" not in reader.fieldnames:
            raise ValueError(f"{path}: need a CSV with frame and ttc columns")
        rows = {}
        for rec in reader:
            rows[int(rec["frame"])] = (float(rec["ttc"]),
                                       rec.get("degenerate", "false").strip().lower() == "true")
    return rows


def score_mse(pred_path, truth_path) -> ScoreReport:
    """synth.score_mse (synth.py:186-208): MSE of predicted vs true ttc over the
    shared frame indices; degenerate / non-finite predictions are excluded but
    counted.  Host CSV bookkeeping (a trace from write_trace against truth.csv)."""
    pred = _read_ttc_column(pred_path)
    truth = _read_ttc_column(truth_path)
    shared = sorted(set(pred) & set(truth))
    if not shared:
        raise ValueError("prediction and truth share no frame indices")
    errs, excluded = [], 0
    for idx in shared:
        p, degenerate = pred[idx]
        if degenerate or not math.isfinite(p):
            excluded += 1
            continue
        errs.append((p - truth[idx][0]) ** 2)
    if not errs:
        raise ValueError("no comparable rows: every prediction was degenerate or non-finite")
    return ScoreReport(mse=float(np.mean(errs)), compared=len(errs), excluded=excluded)


@dataclass(frozen=True)
class Segment:
    start: int
    length: int
    t0: float
    texture_seed: int


def approach_segments(frames: int, seed: int, t0_range=(50.0, 500.0), min_ttc: float = 20.0) -> list[Segment]:
    """Split a long stream into approach segments.

    Segment k draws T0_k ~ U[t0_range] and a texture seed from PCG64(seed);
    it lasts floor(T0_k - min_ttc) + 1 frames (true TTC >= min_ttc on every
    frame) or until the stream ends.  The pair spanning a cut has no truth.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    segs, start = [], 0
    while start < frames:
        t0 = float(rng.uniform(*t0_range))
        tex_seed = int(rng.integers(0, 2**31 - 1))
        length = min(frames - start, int(math.floor(t0 - min_ttc)) + 1)
        segs.append(Segment(start, length, t0, tex_seed))
        start += length
    return segs


def approach_stream(frames: int, height: int, width: int, seed: int, dtype=torch.float32,
                    out: torch.Tensor | None = None, foe=(0.5, 0.5),
                    frame_range: tuple[int, int] | None = None) -> tuple[torch.Tensor, np.ndarray]:
    """A long synthetic approach video on the device (BASELINE config 5 inputs).

    Returns (frames [frames, h, w] in ``dtype``, truth ttc per frame with NaN
    on the first frame of every segment after the first -- the pair ending
    there spans a cut).  Frames are generated in float64 and rounded to
    ``dtype`` (SURVEY.md section 8(d) seeding convention).  frame_range=(a, b)
    builds only frames a..b-1 of the same stream (a temporal shard: its
    frames equal those of the whole-stream call), returned as [b - a, h, w].
    """
    a, b = (0, frames) if frame_range is None else (int(frame_range[0]), int(frame_range[1]))
    if not 0 <= a <= b <= frames:
        raise ValueError(f"frame_range {frame_range} outside [0, {frames}]")
    if out is None:
        out = torch.empty((b - a, height, width), dtype=dtype, device="cuda")
    truth = np.empty(b - a)
    foe_px = (foe[0] * width, foe[1] * height)
    for s in approach_segments(frames, seed):
        lo, hi = max(a, s.start), min(b, s.start + s.length)
        if lo >= hi:
            continue
        tex = make_texture_device(width, height, s.texture_seed)
        mags = [s.t0 / (s.t0 - (t - s.start)) for t in range(lo, hi)]
        zoom_frames(tex, foe_px, mags, dtype=dtype, out=out[lo - a:hi - a])
        truth[lo - a:hi - a] = [s.t0 - (t - s.start) for t in range(lo, hi)]
        if s.start > 0 and lo == s.start:
            truth[lo - a] = np.nan
    return out, truth
