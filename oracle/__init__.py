"""CPU oracle for the convtact hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline.  The product (``paper_1612_08825_b200``) never imports it.

Two halves:
  * ``libconvtact_oracle.so`` (convtact_oracle.c): a C restatement of the
    reference's float64 conv/TTC algorithm with the same per-element
    summation order (see that file's header);
  * this module: ctypes wrappers plus a numpy restatement of the reference's
    synthetic approach generator (synth.py:68-143), used to make inputs.

The restatement is pinned against golden fixtures produced by the reference
itself (tests/golden/make_golden.py -> tests/golden/*.npz).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libconvtact_oracle.so")
_lib = None

SHAPE_CODE = {"full": 0, "same": 1, "valid": 2}
BOUNDARY_CODE = {"zero": 0, "replicate": 1}
EST_FIELDS = ("a", "b", "c", "x0", "y0", "ttc", "residual", "misfit", "level", "degenerate")


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        I = ctypes.c_int
        D = ctypes.c_double
        L.or_direct.argtypes = [I, P, P, P, P, I, I, I, P]
        L.or_direct_batch.argtypes = [I, P, P, I64, P, P, I, I, I, P, I64, I]
        L.or_derivatives.argtypes = [P, P, I64, I64, P, P, P]
        L.or_radial_gradient.argtypes = [P, P, I64, I64, P]
        L.or_normal_system.argtypes = [P, P, P, P, I64, I64, I64, P]
        L.or_solve_ttc.argtypes = [P, D, P]
        L.or_solve_ttc.restype = None
        L.or_downsample.argtypes = [P, I64, I64, P]
        L.or_estimate_fixed.argtypes = [P, P, I64, I64, I, D, P]
        L.or_estimate_multiscale.argtypes = [P, P, I64, I64, I, D, P]
        L.or_run_sequence.argtypes = [P, I64, I64, I64, I, I, D, P, I]
        L.or_max_threads.argtypes = []
        L.or_derivatives.restype = None
        L.or_radial_gradient.restype = None
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(v) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(v, dtype=np.int64).reshape(-1))


def out_shape(ms, ns, shape: str):
    if shape == "full":
        return tuple(m + n - 1 for m, n in zip(ms, ns))
    if shape == "same":
        return tuple(ms)
    return tuple(m - n + 1 for m, n in zip(ms, ns))


def direct(s, k, shape: str = "full", boundary: str = "zero", flip: bool = True) -> np.ndarray:
    """conv._direct (conv.py:133-150); shape/boundary as lowercase strings."""
    s, k = _f64(s), _f64(k)
    assert s.ndim == k.ndim >= 1
    o = out_shape(s.shape, k.shape, shape)
    if shape == "valid" and min(o) < 1:
        raise ValueError("VALID needs signal >= kernel")
    out = np.empty(o, dtype=np.float64)
    rc = lib().or_direct(s.ndim, _p(s), _p(_i64(s.shape)), _p(k), _p(_i64(k.shape)),
                         SHAPE_CODE[shape], BOUNDARY_CODE[boundary], int(flip), _p(out))
    if rc:
        raise ValueError(f"oracle direct rc={rc}")
    return out


def direct_batch(s, k, shape="full", boundary="zero", flip=True, nthreads=0) -> np.ndarray:
    """Independent direct() over the leading axis of ``s`` (OpenMP over images)."""
    s, k = _f64(s), _f64(k)
    nb = s.shape[0]
    o = out_shape(s.shape[1:], k.shape, shape)
    out = np.empty((nb,) + o, dtype=np.float64)
    rc = lib().or_direct_batch(k.ndim, _p(s), _p(_i64(s.shape[1:])), nb, _p(k), _p(_i64(k.shape)),
                               SHAPE_CODE[shape], BOUNDARY_CODE[boundary], int(flip), _p(out),
                               int(np.prod(o)), int(nthreads))
    if rc:
        raise ValueError(f"oracle direct_batch rc={rc}")
    return out


def derivatives(a, b):
    a, b = _f64(a), _f64(b)
    h, w = a.shape
    ex, ey, et = (np.empty((h - 1, w - 1)) for _ in range(3))
    lib().or_derivatives(_p(a), _p(b), h, w, _p(ex), _p(ey), _p(et))
    return ex, ey, et


def radial_gradient(ex, ey):
    ex, ey = _f64(ex), _f64(ey)
    g = np.empty_like(ex)
    lib().or_radial_gradient(_p(ex), _p(ey), ex.shape[0], ex.shape[1], _p(g))
    return g


def normal_system(ex, ey, g, et, border=1) -> np.ndarray:
    """11 sums: m00 m01 m02 m11 m12 m22, rhs0..2 (negated), et2, count."""
    ex, ey, g, et = (_f64(x) for x in (ex, ey, g, et))
    sums = np.empty(11)
    rc = lib().or_normal_system(_p(ex), _p(ey), _p(g), _p(et), ex.shape[0], ex.shape[1], border, _p(sums))
    if rc:
        raise ValueError(f"oracle normal_system rc={rc}")
    return sums


def solve_ttc(sums, c_min=1e-9) -> np.ndarray:
    sums = _f64(sums)
    est = np.empty(10)
    lib().or_solve_ttc(_p(sums), float(c_min), _p(est))
    return est


def downsample(img) -> np.ndarray:
    img = _f64(img)
    h, w = img.shape
    out = np.empty((h // 2, w // 2))
    rc = lib().or_downsample(_p(img), h, w, _p(out))
    if rc:
        raise ValueError("cannot halve")
    return out


def estimate_fixed(a, b, level=0, c_min=1e-9) -> np.ndarray:
    a, b = _f64(a), _f64(b)
    est = np.empty(10)
    rc = lib().or_estimate_fixed(_p(a), _p(b), a.shape[0], a.shape[1], int(level), float(c_min), _p(est))
    if rc:
        raise ValueError(f"oracle estimate_fixed rc={rc}")
    return est


def estimate_multiscale(a, b, max_level=5, c_min=1e-9) -> np.ndarray:
    a, b = _f64(a), _f64(b)
    est = np.empty(10)
    rc = lib().or_estimate_multiscale(_p(a), _p(b), a.shape[0], a.shape[1], int(max_level),
                                      float(c_min), _p(est))
    if rc:
        raise ValueError(f"oracle estimate_multiscale rc={rc}")
    return est


def run_sequence(frames, level=0, max_level=None, c_min=1e-9, nthreads=0) -> np.ndarray:
    """[n-1, 10] estimate rows (EST_FIELDS order); level field -1 = None."""
    frames = _f64(frames)
    n, h, w = frames.shape
    est = np.empty((n - 1, 10))
    rc = lib().or_run_sequence(_p(frames), n, h, w, int(level or 0),
                               -1 if max_level is None else int(max_level), float(c_min), _p(est),
                               int(nthreads))
    if rc:
        raise ValueError(f"oracle run_sequence rc={rc}")
    return est


def max_threads() -> int:
    return int(lib().or_max_threads())


# ---------------------------------------------------------------- synth ---
# numpy restatement of the reference generator (synth.py:68-143); bit-exact
# with it (pinned by tests/test_oracle_golden.py).

_B3 = np.outer(*(2 * [np.array([1.0, 2.0, 1.0]) / 4.0]))


def make_texture(width: int, height: int, seed: int) -> np.ndarray:
    """synth.make_texture (synth.py:68-85)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    img = rng.random((height, width))
    for _ in range(2):
        img = direct(img, _B3, "same", "replicate", flip=False)
    lo, hi = img.min(), img.max()
    if hi <= lo:
        return np.zeros_like(img)
    return (img - lo) / (hi - lo)


def axis_taps(size: int, center: float, magnification: float):
    """synth._axis_taps (synth.py:88-107): clamped indices and Catmull-Rom weights."""
    p = np.arange(size, dtype=np.float64)
    src = center + (p - center) / magnification
    i0 = np.floor(src).astype(np.int64)
    f = src - i0
    idx = np.clip(np.stack([i0 - 1, i0, i0 + 1, i0 + 2], axis=1), 0, size - 1)
    f2 = f * f
    f3 = f2 * f
    w = np.stack([-0.5 * f3 + f2 - 0.5 * f, 1.5 * f3 - 2.5 * f2 + 1.0,
                  -1.5 * f3 + 2.0 * f2 + 0.5 * f, 0.5 * f3 - 0.5 * f2], axis=1)
    return idx, w


def zoom_frame(texture, foe_px, magnification: float) -> np.ndarray:
    """synth.zoom_frame (synth.py:110-126)."""
    texture = _f64(texture)
    if magnification == 1.0:
        return texture.copy()
    h, w = texture.shape
    ix, wx = axis_taps(w, foe_px[0], magnification)
    iy, wy = axis_taps(h, foe_px[1], magnification)
    tmp = np.zeros_like(texture)
    for b in range(4):
        tmp += wx[None, :, b] * texture[:, ix[:, b]]
    out = np.zeros_like(texture)
    for a in range(4):
        out += wy[:, a][:, None] * tmp[iy[:, a], :]
    return out


def generate(width=256, height=256, frames=60, t0=100.0, foe=(0.4, 0.55), seed=1,
             noise_sigma=0.0) -> np.ndarray:
    """synth.generate (synth.py:129-143): [frames, height, width] float64."""
    if frames >= t0:
        raise ValueError("frames must stay short of contact")
    texture = make_texture(width, height, seed)
    noise_rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 1])))
    foe_px = (foe[0] * width, foe[1] * height)
    out = np.empty((frames, height, width))
    for t in range(frames):
        fr = zoom_frame(texture, foe_px, t0 / (t0 - t))
        if noise_sigma > 0:
            fr = np.clip(fr + noise_rng.normal(0.0, noise_sigma, fr.shape), 0.0, 1.0)
        out[t] = fr
    return out
