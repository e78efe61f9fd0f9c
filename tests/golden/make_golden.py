"""Generate golden fixtures by running the UNMODIFIED reference package.

Run in the build container (the reference is not on the GPU box):

    python tests/golden/make_golden.py

It imports convtact from /root/reference/pkg/src with NUMBA_CACHE_DIR pointed
at a scratch directory, so nothing is written into the read-only reference
tree, and writes small .npz fixtures next to this file.  The seeds and input
conventions are the ones SURVEY.md section 8(d) fixes for the BASELINE configs.
"""

import hashlib
import os
import sys
import tempfile

os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "convtact_numba_cache"))
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import convtact  # noqa: E402
from convtact import BoundaryPolicy, ConvShape, conv_direct, xcorr_direct  # noqa: E402
from convtact import ttc as rttc  # noqa: E402
from convtact.synth import SynthConfig, generate  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
EST = ("a", "b", "c", "x0", "y0", "ttc", "residual", "misfit", "level", "degenerate")
SHAPES = {"full": ConvShape.FULL, "same": ConvShape.SAME, "valid": ConvShape.VALID}
BOUNDS = {"zero": BoundaryPolicy.ZERO, "replicate": BoundaryPolicy.REPLICATE}


def est_row(e):
    if e is None:
        return [np.nan] * 8 + [-1.0, np.nan]
    return [float(getattr(e, f)) for f in EST]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def conv_cases():
    rng = np.random.default_rng(2024)
    out = {}
    i = 0
    max_extent = {1: 9, 2: 7, 3: 5, 4: 4}
    for ndim in (1, 2, 3, 4):
        for _ in range(24):
            hi = max_extent[ndim]
            s = rng.uniform(-1, 1, tuple(rng.integers(1, hi + 1, ndim)))
            k = rng.uniform(-1, 1, tuple(rng.integers(1, hi + 1, ndim)))
            for shape in ("full", "same", "valid"):
                if shape == "valid" and any(m < n for m, n in zip(s.shape, k.shape)):
                    continue
                for bound in (("zero", "replicate") if shape == "same" else ("zero",)):
                    for flip in (0, 1):
                        fn = conv_direct if flip else xcorr_direct
                        r = fn(s, k, SHAPES[shape], BOUNDS[bound])
                        out[f"c{i}_s"] = s
                        out[f"c{i}_k"] = k
                        out[f"c{i}_out"] = r
                        out[f"c{i}_meta"] = np.array([list(SHAPES).index(shape), list(BOUNDS).index(bound), flip])
                        i += 1
    out["count"] = np.array(i)
    np.savez_compressed(os.path.join(HERE, "conv_cases.npz"), **out)
    print("conv cases", i)


def sample_idx(n, count, seed):
    return np.sort(np.random.default_rng(seed).choice(n, size=min(count, n), replace=False))


def conv_configs():
    out = {}
    # cfg1: 2-D FULL fp64, 256^2 (seed 0 uniform) * 5^2 (seed 1 normal)
    s = np.random.Generator(np.random.PCG64(0)).random((256, 256))
    k = np.random.Generator(np.random.PCG64(1)).standard_normal((5, 5))
    r = conv_direct(s, k, ConvShape.FULL)
    out["cfg1_out"] = r  # 260x260 f64, the full reference output
    # cfg3: 3-D FULL, inputs fp32-rounded then fed to the f64 reference
    s = np.random.Generator(np.random.PCG64(0)).random((128,) * 3).astype(np.float32).astype(np.float64)
    k = np.random.Generator(np.random.PCG64(1)).standard_normal((7,) * 3).astype(np.float32).astype(np.float64)
    r = conv_direct(s, k, ConvShape.FULL)
    idx = sample_idx(r.size, 20000, 3)
    out.update(cfg3_idx=idx, cfg3_val=r.ravel()[idx], cfg3_sum=r.sum(), cfg3_absmax=np.abs(r).max())
    # cfg4: large-kernel 2-D FULL
    s = np.random.Generator(np.random.PCG64(0)).random((2048, 2048)).astype(np.float32).astype(np.float64)
    k = np.random.Generator(np.random.PCG64(1)).standard_normal((31, 31)).astype(np.float32).astype(np.float64)
    r = conv_direct(s, k, ConvShape.FULL)
    idx = sample_idx(r.size, 40000, 4)
    out.update(cfg4_idx=idx, cfg4_val=r.ravel()[idx], cfg4_sum=r.sum(), cfg4_absmax=np.abs(r).max())
    np.savez_compressed(os.path.join(HERE, "conv_configs.npz"), **out)
    print("conv configs done")


def ttc_fixtures():
    out = {}
    # cfg2: single-scale TTC fp64, 64 frames 256^2 approaching plane, truth 100 - t
    cfg2 = SynthConfig(width=256, height=256, frames=64, t0=100.0, foe=(0.5, 0.5), seed=0, noise_sigma=0.0)
    seq = generate(cfg2)
    out["cfg2_frames_sha"] = np.array(sha(seq.frames))
    out["cfg2_frame0_row0"] = seq.frames[0, 0]
    out["cfg2_frame63_row128"] = seq.frames[63, 128]
    out["cfg2_l0"] = np.array([est_row(e) for e in rttc.run_sequence(seq.frames, level=0)])
    out["cfg2_l1"] = np.array([est_row(e) for e in rttc.run_sequence(seq.frames[:9], level=1)])
    out["cfg2_l2"] = np.array([est_row(e) for e in rttc.run_sequence(seq.frames[:9], level=2)])
    out["cfg2_ms5"] = np.array([est_row(e) for e in rttc.run_sequence(seq.frames[:9], max_level=5)])
    # default suite, seed 1 (test_output.txt:136 anchors pair 0)
    seq1 = generate(SynthConfig(seed=1))
    out["def1_frames_sha"] = np.array(sha(seq1.frames))
    out["def1_l0"] = np.array([est_row(e) for e in rttc.run_sequence(seq1.frames, level=0)])
    # noisy multiscale (test_ttc.py:215-223 setting)
    cfgn = SynthConfig(width=128, height=128, frames=12, t0=60.0, foe=(0.5, 0.5), seed=2, noise_sigma=0.05)
    seqn = generate(cfgn)
    out["noisy_frames_sha"] = np.array(sha(seqn.frames))
    out["noisy_ms5"] = np.array([est_row(e) for e in rttc.run_sequence(seqn.frames, max_level=5)])
    out["noisy_l0"] = np.array([est_row(e) for e in rttc.run_sequence(seqn.frames, level=0)])
    # intermediate fields on a small odd-sized pair
    rng = np.random.default_rng(77)
    a = rng.random((37, 50))
    b = a + 0.01 * rng.standard_normal((37, 50))
    pair = rttc.FramePair(a, b)
    ex, ey, et = rttc.derivatives_3d(pair)
    g = rttc.radial_gradient(ex, ey)
    ns = rttc.build_normal_system(ex, ey, g, et, border=1)
    ns2 = rttc.build_normal_system(ex, ey, g, et, border=3)
    out.update(small_a=a, small_b=b, small_ex=ex, small_ey=ey, small_et=et, small_g=g)
    def sums(n):
        return np.array([n.m[0, 0], n.m[0, 1], n.m[0, 2], n.m[1, 1], n.m[1, 2], n.m[2, 2],
                         n.rhs[0], n.rhs[1], n.rhs[2], n.et2, n.count])
    out["small_sums_b1"] = sums(ns)
    out["small_sums_b3"] = sums(ns2)
    out["small_est"] = np.array(est_row(rttc.solve_ttc(ns)))
    out["small_down"] = rttc.downsample(a)
    out["small_down2"] = rttc.downsample(rttc.downsample(a))
    # multiscale on fp32-rounded frames (cfg5 convention, reduced size)
    cfg5s = SynthConfig(width=480, height=270, frames=4, t0=300.0, foe=(0.5, 0.5), seed=11, noise_sigma=0.0)
    f5 = generate(cfg5s).frames.astype(np.float32)
    out["c5_frames32_sha"] = np.array(hashlib.sha256(f5.tobytes()).hexdigest())
    out["c5_ms3"] = np.array([est_row(e) for e in rttc.run_sequence(f5.astype(np.float64), max_level=3)])
    out["c5_l"] = np.array([[est_row(rttc.estimate_fixed(rttc.FramePair(f5[0].astype(np.float64), f5[1].astype(np.float64)), level=l))
                             for l in range(4)]])[0]
    out["c5_down"] = rttc.downsample(f5[0].astype(np.float64))
    np.savez_compressed(os.path.join(HERE, "ttc_fixtures.npz"), **out)
    print("ttc fixtures done")


def gradient_fixtures():
    from convtact.kernels import KERNELS, gradient
    rng = np.random.default_rng(99)
    img = rng.random((37, 53))
    out = {"img": img}
    for name in KERNELS:
        f = gradient(img, name)
        out[f"{name}_ex"], out[f"{name}_ey"], out[f"{name}_mag"], out[f"{name}_dir"] = f.ex, f.ey, f.mag, f.dir
    np.savez_compressed(os.path.join(HERE, "gradient_fixtures.npz"), **out)
    print("gradient fixtures done")


def nonfinite_fixtures():
    """NaN / Inf propagation through the hot path (the reference has no guard:
    IEEE semantics of its numpy / numba arithmetic decide every field)."""
    rng = np.random.default_rng(2718)
    frames = generate(SynthConfig(width=64, height=48, frames=5, t0=40.0, foe=(0.45, 0.55), seed=3)).frames.copy()
    frames[1, 10, 10] = np.nan
    frames[3, 5, 7] = np.inf
    out = {"frames": frames}
    for key, kw in (("l0", dict(level=0)), ("l1", dict(level=1)), ("ms2", dict(max_level=2))):
        out[key] = np.array([est_row(e) for e in rttc.run_sequence(frames, **kw)])
    s = rng.random((20, 30))
    s[4, 5] = np.nan
    s[17, 0] = -np.inf
    k = rng.standard_normal((3, 4))
    out["conv_s"], out["conv_k"] = s, k
    out["conv_full"] = conv_direct(s, k, ConvShape.FULL)
    out["xcorr_same_rep"] = xcorr_direct(s, k, ConvShape.SAME, BoundaryPolicy.REPLICATE)
    np.savez_compressed(os.path.join(HERE, "nonfinite_fixtures.npz"), **out)
    print("nonfinite fixtures done")


SECTIONS = {"gradient": lambda: gradient_fixtures(), "conv_cases": lambda: conv_cases(),
            "ttc": lambda: ttc_fixtures(), "conv_configs": lambda: conv_configs(),
            "nonfinite": lambda: nonfinite_fixtures()}

if __name__ == "__main__":
    print("reference convtact", convtact.__version__)
    for name in (sys.argv[1:] or SECTIONS):  # default: every fixture file
        SECTIONS[name]()
