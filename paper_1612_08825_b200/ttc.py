"""Time-to-contact / focus-of-expansion on the B200 (drop-in for convtact.ttc).

Same names, signatures, validation and degeneracy semantics as the reference
(/root/reference/pkg/src/convtact/ttc.py).  Every numeric step runs in
libconvtact_b200.so:

  derivatives_3d / radial_gradient / build_normal_system   ct_ttc_derivatives,
      ct_radial_gradient, ct_normal_system (field-level API, kept for callers)
  estimate_fixed / estimate_multiscale / run_sequence      ct_run_sequence: the
      fused moments kernel (frames read once, no derivative fields in HBM),
      the device pyramid, the device LDL^T solve and level selection
  solve_ttc                                                ct_ttc_solve
  downsample                                               ct_pyramid_down

numpy inputs are coerced to float64 (ttc.py:87, ttc.py:293) and results come
back on the host; CUDA tensors stay on the device and float32 stacks take the
fp32 path.  run_sequence_batch() is the batched entry the benchmark uses.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

DEFAULT_C_MIN = 1e-9
_PIVOT_TOL = 1e-10
_IMPROVE_EPS = 1e-3


@dataclass(frozen=True)
class FramePair:
    first: object
    second: object

    def __post_init__(self):  # ttc.py:46-51
        a, b = self.first, self.second
        if a.ndim != 2 or b.ndim != 2:
            raise ValueError("frames must be 2-D")
        if tuple(a.shape) != tuple(b.shape):
            raise ValueError(f"frame extents differ: {tuple(a.shape)} vs {tuple(b.shape)}")


@dataclass(frozen=True)
class NormalSystem:
    """3x3 Gram matrix and right-hand side of the least-squares problem (ttc.py:54-65)."""

    m: np.ndarray
    rhs: np.ndarray
    et2: float
    count: int


@dataclass(frozen=True)
class TtcEstimate:
    a: float
    b: float
    c: float
    x0: float
    y0: float
    ttc: float
    residual: float
    misfit: float
    level: int
    degenerate: bool


_FIELDS = ("a", "b", "c", "x0", "y0", "ttc", "residual", "misfit")


def estimate_from_row(row) -> TtcEstimate | None:
    """One 10-double estimate row (CT_NEST layout) -> TtcEstimate (None if level == -1)."""
    row = [float(x) for x in row]
    if row[8] < 0:
        return None
    return TtcEstimate(*row[:8], level=int(row[8]), degenerate=bool(row[9] != 0.0))


def _is_host(x) -> bool:
    return not (isinstance(x, torch.Tensor) and x.is_cuda)


def _back(t: torch.Tensor, like):
    if isinstance(like, torch.Tensor):
        return t if like.is_cuda else t.cpu()
    return t.cpu().numpy()


# ----------------------------------------------------------- field API ---

def derivatives_3d(pair: FramePair):
    """Ex, Ey, Et on the half-pixel grid, each (h-1, w-1) (ttc.py:82-91)."""
    h, w = pair.first.shape
    if h < 2 or w < 2:
        raise ValueError(f"need extents >= 2 for derivatives, got {(h, w)}")
    a, _ = _lib.to_device(pair.first)
    b, _ = _lib.to_device(pair.second)
    if a.dtype != b.dtype:
        a, b = a.double(), b.double()
    out = [torch.empty((h - 1, w - 1), dtype=a.dtype, device=a.device) for _ in range(3)]
    L = _lib.load()
    _lib.check(L.ct_ttc_derivatives(_lib.dtype_code(a), _lib.ptr(a), _lib.ptr(b), h, w, *(_lib.ptr(t) for t in out),
                                    _lib.stream_ptr()))
    return tuple(_back(t, pair.first) for t in out)


def radial_gradient(ex, ey):
    """G = x*Ex + y*Ey with coordinates centered on the derivative grid (ttc.py:94-99)."""
    x, _ = _lib.to_device(ex)
    y, _ = _lib.to_device(ey)
    if x.dtype != y.dtype:
        x, y = x.double(), y.double()
    gh, gw = x.shape
    g = torch.empty_like(x)
    L = _lib.load()
    _lib.check(L.ct_radial_gradient(_lib.dtype_code(x), _lib.ptr(x), _lib.ptr(y), gh, gw, _lib.ptr(g),
                                    _lib.stream_ptr()))
    return _back(g, ex)


def _system_from_sums(s) -> NormalSystem:
    s = [float(v) for v in s]
    m = np.array([[s[0], s[1], s[2]], [s[1], s[3], s[4]], [s[2], s[4], s[5]]])
    return NormalSystem(m=m, rhs=np.array(s[6:9]), et2=s[9], count=int(s[10]))


def build_normal_system(ex, ey, g, et, border: int = 1) -> NormalSystem:
    """ttc.py:102-120: Gram matrix of [Ex, Ey, G] and -[sum ExEt, EyEt, GEt] over the window."""
    shapes = [tuple(f.shape) for f in (ex, ey, g, et)]
    if not (shapes[0] == shapes[1] == shapes[2] == shapes[3]):
        raise ValueError("derivative fields must share extents")
    if border < 1:
        raise ValueError("border must cover the derivative-kernel radius (>= 1)")
    gh, gw = shapes[0]
    if gh <= 2 * border or gw <= 2 * border:
        raise ValueError(f"no interior left: grid {(gh, gw)}, border {border}")
    ts = [_lib.to_device(f)[0] for f in (ex, ey, g, et)]
    if len({t.dtype for t in ts}) > 1:
        ts = [t.double() for t in ts]
    dev = ts[0].device
    L = _lib.load()
    sums = torch.empty(11, dtype=torch.float64, device=dev)
    nbytes = L.ct_normal_system_workspace_bytes(gh, gw)
    ws = _lib.workspace(nbytes, dev)
    _lib.check(L.ct_normal_system(_lib.dtype_code(ts[0]), *(_lib.ptr(t) for t in ts), gh, gw, border, _lib.ptr(sums),
                                  _lib.ptr(ws), nbytes, _lib.stream_ptr()))
    return _system_from_sums(sums.cpu().numpy())


def solve_ttc(system: NormalSystem, c_min: float = DEFAULT_C_MIN) -> TtcEstimate:
    """Solve the normal equations; degeneracy is data, not failure (ttc.py:157-184)."""
    m = np.asarray(system.m, dtype=np.float64)
    rhs = np.asarray(system.rhs, dtype=np.float64)
    s = np.array([m[0, 0], m[0, 1], m[0, 2], m[1, 1], m[1, 2], m[2, 2], rhs[0], rhs[1], rhs[2],
                  float(system.et2), float(system.count)], dtype=np.float64)
    L = _lib.load()
    sd = torch.from_numpy(s).to("cuda")
    est = torch.empty(10, dtype=torch.float64, device=sd.device)
    _lib.check(L.ct_ttc_solve(_lib.ptr(sd), 1, float(c_min), 0, _lib.ptr(est), _lib.stream_ptr()))
    return estimate_from_row(est.cpu().numpy())


def downsample(img):
    """Halve both extents: 2x2 block mean, then 5x5 binomial SAME/REPLICATE (ttc.py:187-204)."""
    t, _ = _lib.to_device(img)
    if t.ndim != 2:
        raise ValueError("downsample expects a 2-D image")
    h, w = t.shape
    if h < 2 or w < 2:
        raise ValueError(f"cannot halve extents {(h, w)}")
    out = torch.empty((h // 2, w // 2), dtype=t.dtype, device=t.device)
    L = _lib.load()
    _lib.check(L.ct_pyramid_down(_lib.dtype_code(t), _lib.ptr(t), 1, h, w, _lib.ptr(out), _lib.stream_ptr()))
    return _back(out, img)


# ------------------------------------------------------- estimator API ---

def _level_extents(shape, level):  # ttc.py:207-212
    h, w = shape
    for _ in range(level):
        h //= 2
        w //= 2
    return h, w


def run_sequence_batch(frames, level: int | None = 0, max_level: int | None = None,
                       c_min: float = DEFAULT_C_MIN, out: torch.Tensor | None = None) -> torch.Tensor:
    """Batched run_sequence: frames [V, n, h, w] CUDA tensor -> estimates [V, n-1, 10] (device).

    One call runs the whole pipeline on the device (pyramid, fused moments,
    solve, level selection) with no host synchronisation.
    """
    if not (isinstance(frames, torch.Tensor) and frames.is_cuda and frames.ndim == 4):
        raise TypeError("run_sequence_batch expects a CUDA tensor [V, n, h, w]")
    f = frames.contiguous()
    if f.dtype not in (torch.float32, torch.float64):
        f = f.double()
    V, n, h, w = f.shape
    if n < 2:
        raise ValueError("need at least two frames")
    lv = int(level or 0)
    ml = -1 if max_level is None else int(max_level)
    if max_level is not None and ml < 0:
        raise ValueError("max_level must be >= 0")
    L = _lib.load()
    dt = _lib.dtype_code(f)
    nbytes = L.ct_run_sequence_workspace_bytes(dt, V, n, h, w, lv, ml)
    ws = _lib.workspace(nbytes, f.device)
    if out is None:
        out = torch.empty((V, n - 1, 10), dtype=torch.float64, device=f.device)
    _lib.check(L.ct_run_sequence(dt, _lib.ptr(f), V, n, h, w, lv, ml, float(c_min), _lib.ptr(out), _lib.ptr(ws),
                                 nbytes, _lib.stream_ptr()))
    return out


def pyramid_moments(frames, levels: int) -> torch.Tensor:
    """Per-level normal-system sums of every consecutive frame pair on the
    multiscale pyramid (ct_ttc_pyramid_moments): frames [V, n, h, w] CUDA
    tensor -> [levels, V, n-1, 11] float64 (m00 m01 m02 m11 m12 m22, rhs0..2,
    et2, count, as NormalSystem / build_normal_system, ttc.py:102-120).  Level l
    is the l-fold downsample (ttc.py:187-204); these are the systems
    estimate_multiscale solves level by level (ttc.py:248-279)."""
    if not (isinstance(frames, torch.Tensor) and frames.is_cuda and frames.ndim == 4):
        raise TypeError("pyramid_moments expects a CUDA tensor [V, n, h, w]")
    f = frames.contiguous()
    if f.dtype not in (torch.float32, torch.float64):
        f = f.double()
    V, n, h, w = f.shape
    L = _lib.load()
    dt = _lib.dtype_code(f)
    nbytes = L.ct_ttc_pyramid_moments_workspace_bytes(dt, V, n, h, w, int(levels))
    ws = _lib.workspace(nbytes, f.device)
    out = torch.empty((int(levels), V, max(n - 1, 0), 11), dtype=torch.float64, device=f.device)
    _lib.check(L.ct_ttc_pyramid_moments(dt, _lib.ptr(f), V, n, h, w, int(levels), _lib.ptr(out), _lib.ptr(ws),
                                        nbytes, _lib.stream_ptr()))
    return out


def run_sequence_host(frames: np.ndarray, level: int | None = 0, max_level: int | None = None,
                      c_min: float = DEFAULT_C_MIN) -> np.ndarray:
    """run_sequence for a HOST stack [V, n, h, w] (float64 or float32 numpy, ideally
    pinned): frames stream to the device in chunks overlapped with compute
    (ct_run_sequence_host).  Returns estimates [V, n-1, 10] on the host."""
    if isinstance(frames, torch.Tensor):
        f = frames.contiguous()
        hptr = f.data_ptr()
        dt = _lib.dtype_code(f)
        V, n, h, w = f.shape
    else:
        f = np.ascontiguousarray(frames)
        if f.dtype not in (np.float32, np.float64):
            f = f.astype(np.float64)
        hptr = f.ctypes.data
        dt = _lib.CT_F64 if f.dtype == np.float64 else _lib.CT_F32
        V, n, h, w = f.shape
    lv = int(level or 0)
    ml = -1 if max_level is None else int(max_level)
    L = _lib.load()
    nbytes = L.ct_run_sequence_host_workspace_bytes(dt, V, n, h, w, lv, ml)
    ws = _lib.workspace(nbytes, "cuda")
    est = _pinned_rows(V * (n - 1) * 10)
    _lib.check(L.ct_run_sequence_host(dt, ctypes.c_void_p(hptr), V, n, h, w, lv, ml, float(c_min),
                                      ctypes.c_void_p(est.data_ptr()), _lib.ptr(ws), nbytes, _lib.stream_ptr()))
    torch.cuda.current_stream().synchronize()
    return est.numpy().reshape(V, n - 1, 10).copy()


_PINNED = threading.local()


def _pinned_rows(count: int) -> torch.Tensor:
    """A reused page-locked staging buffer for estimate rows, one per thread
    (grown on demand; pinning a fresh buffer per call costs more than the
    rows' D2H).  Callers copy out before returning, so results never alias."""
    buf = getattr(_PINNED, "buf", None)
    if buf is None or buf.numel() < count:
        buf = torch.empty(max(count, 1 << 16), dtype=torch.float64).pin_memory()
        _PINNED.buf = buf
    return buf[:count]


def _stack_pair(pair: FramePair) -> tuple[torch.Tensor, bool]:
    a, host = _lib.to_device(pair.first)
    b, _ = _lib.to_device(pair.second)
    if a.dtype != b.dtype:
        a, b = a.double(), b.double()
    return torch.stack([a, b])[None], host


def estimate_fixed(pair: FramePair, level: int = 0, c_min: float = DEFAULT_C_MIN) -> TtcEstimate:
    """Estimate at one pyramid level; FOE mapped back to level-0 pixels (ttc.py:228-245)."""
    if level < 0:
        raise ValueError("level must be >= 0")
    h, w = _level_extents(tuple(pair.first.shape), level)
    if h < 4 or w < 4:
        raise ValueError(f"extents {tuple(pair.first.shape)} leave {(h, w)} after {level} halvings, need >= 4")
    st, _ = _stack_pair(pair)
    est = run_sequence_batch(st, level=level, c_min=c_min)
    return estimate_from_row(est[0, 0].cpu().numpy())


def estimate_multiscale(pair: FramePair, max_level: int = 5, c_min: float = DEFAULT_C_MIN) -> TtcEstimate:
    """Greedy coarse-to-fine level selection (ttc.py:248-279); all levels run on the device."""
    if max_level < 0:
        raise ValueError("max_level must be >= 0")
    st, _ = _stack_pair(pair)
    est = run_sequence_batch(st, max_level=max_level, c_min=c_min)
    return estimate_from_row(est[0, 0].cpu().numpy())


def run_sequence(frames, level: int | None = 0, max_level: int | None = None,
                 c_min: float = DEFAULT_C_MIN) -> list[TtcEstimate]:
    """Estimate over consecutive pairs of a [n, h, w] stack (ttc.py:282-305).

    Row i comes from frames (i, i+1).  Pass max_level for the multiscale search.
    """
    if isinstance(frames, torch.Tensor):
        f = frames
    else:
        f = np.asarray(frames, dtype=np.float64)
    if f.ndim != 3:
        raise ValueError(f"frame stack must be 3-D, got ndim {f.ndim}")
    if f.shape[0] < 2:
        raise ValueError("need at least two frames")
    lv = level or 0
    if max_level is None:
        if lv < 0:
            raise ValueError("level must be >= 0")
        h, w = _level_extents(tuple(f.shape[1:]), lv)
        if h < 4 or w < 4:
            raise ValueError(f"extents {tuple(f.shape[1:])} leave {(h, w)} after {lv} halvings, need >= 4")
    elif max_level < 0:
        raise ValueError("max_level must be >= 0")
    if isinstance(f, torch.Tensor) and f.is_cuda:
        est = run_sequence_batch(f[None], level=lv, max_level=max_level, c_min=c_min)[0].cpu().numpy()
    else:
        if isinstance(f, torch.Tensor):  # host tensors are coerced to float64 like numpy input (ttc.py:293)
            f = f.to(torch.float64).numpy()
        est = run_sequence_host(np.ascontiguousarray(f)[None], level=lv, max_level=max_level, c_min=c_min)[0]
    return [estimate_from_row(r) for r in est]


# --------------------------------------------------------------- trace ---

def _fmt(x: float) -> str:  # ttc.py:308-313
    if np.isnan(x):
        return "nan"
    if np.isinf(x):
        return "inf" if x > 0 else "-inf"
    return format(x, ".17g")


TRACE_HEADER = "frame,ttc,foe_x,foe_y,residual,level,degenerate"


def trace_lines(estimates) -> list[str]:
    """Trace CSV lines, one row per frame pair (ttc.py:319-327)."""
    lines = [TRACE_HEADER]
    for i, e in enumerate(estimates):
        flag = "true" if e.degenerate else "false"
        lines.append(f"{i},{_fmt(e.ttc)},{_fmt(e.x0)},{_fmt(e.y0)},{_fmt(e.residual)},{e.level},{flag}")
    return lines


def write_trace(estimates, path) -> None:
    with open(path, "w", newline="\n") as f:
        f.write("\n".join(trace_lines(estimates)) + "\n")
