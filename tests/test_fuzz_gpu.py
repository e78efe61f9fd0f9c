"""Seeded randomized sweeps of the GPU path against the CPU oracle.

Shapes, kernel extents (every width class: compile-time tiled widths, the
runtime-width strip kernel, ranks >= 4), modes, boundaries, dtypes and
batch sizes are drawn from a fixed PCG64 stream; float64 must be
bit-identical to the oracle (the reference's FMA order), float32 within
1e-5 relative inf-norm of the float64 oracle on the rounded inputs (480
cases).  The TTC sweep draws 40 float64 stacks of random size, length, noise
and level / max_level: identical level choices and degeneracy, TTC within
1e-9."""

import numpy as np
import pytest
import torch

import oracle as O
import paper_1612_08825_b200 as ct
from conftest import rel_inf
from paper_1612_08825_b200 import BoundaryPolicy, ConvShape

pytestmark = pytest.mark.gpu

SHAPE_NAMES = {ConvShape.FULL: "full", ConvShape.SAME: "same", ConvShape.VALID: "valid"}


def _case(rng):
    ndim = int(rng.choice([1, 2, 2, 3, 4]))
    ks = [int(rng.integers(1, 18 if ndim <= 2 else 8)) for _ in range(ndim)]
    if ndim <= 2 and rng.random() < 0.3:
        ks[-1] = int(rng.integers(18, 41))  # wide kernels: strip kernel beyond the tiled widths
    ss = [int(rng.integers(1, 70 if ndim <= 2 else 18)) for _ in range(ndim)]
    return ss, ks


@pytest.mark.parametrize("chunk", range(8))
def test_conv_fuzz_vs_oracle(chunk):
    rng = np.random.Generator(np.random.PCG64(1000 + chunk))
    for _ in range(60):
        ss, ks = _case(rng)
        shape = [ConvShape.FULL, ConvShape.SAME, ConvShape.VALID][int(rng.integers(0, 3))]
        if shape == ConvShape.VALID and any(s < k for s, k in zip(ss, ks)):
            shape = ConvShape.FULL
        bnd = BoundaryPolicy.REPLICATE if rng.random() < 0.4 else BoundaryPolicy.ZERO
        flip = bool(rng.random() < 0.5)
        s = rng.random(ss)
        k = rng.standard_normal(ks)
        fn = ct.conv_direct if flip else ct.xcorr_direct
        ob = SHAPE_NAMES[shape]
        ref = O.direct(s, k, ob, bnd.name.lower() if shape == ConvShape.SAME else "zero", flip=flip)
        got = fn(s, k, shape, bnd)
        assert np.array_equal(got, ref), (ss, ks, ob, bnd, flip, float(np.abs(got - ref).max()))
        if len(ss) <= 3:
            s32, k32 = s.astype(np.float32), k.astype(np.float32)
            got32 = fn(torch.from_numpy(s32).cuda(), torch.from_numpy(k32), shape, bnd).cpu().numpy()
            ref32 = O.direct(s32.astype(np.float64), k32.astype(np.float64), ob,
                             bnd.name.lower() if shape == ConvShape.SAME else "zero", flip=flip)
            assert rel_inf(got32, ref32) <= 1e-5, (ss, ks, ob, bnd, flip)


def test_conv_batched_fuzz_vs_oracle():
    rng = np.random.Generator(np.random.PCG64(77))
    for _ in range(12):
        ss, ks = _case(rng)
        ss, ks = ss[:3], ks[:3]
        b = int(rng.integers(1, 6))
        s = rng.random([b] + ss)
        k = rng.standard_normal(ks)
        got = ct.direct_batch(torch.from_numpy(s).cuda(), k, ConvShape.FULL, flip=True).cpu().numpy()
        for i in range(b):
            assert np.array_equal(got[i], O.direct(s[i], k, "full")), (ss, ks, i)


def test_ttc_fuzz_vs_oracle():
    rng = np.random.Generator(np.random.PCG64(4242))
    for i in range(40):
        h, w = int(rng.integers(5, 140)), int(rng.integers(5, 300))
        n = int(rng.integers(2, 7))
        frames = O.generate(max(w, 16), max(h, 16), n, float(rng.uniform(n + 5, 300)),
                            (float(rng.uniform(0.2, 0.8)), float(rng.uniform(0.2, 0.8))), 500 + i,
                            float(rng.choice([0.0, 0.02])))[:, :h, :w].copy()
        kw = dict(max_level=int(rng.integers(0, 5))) if rng.random() < 0.5 else dict(level=0)
        ref = O.run_sequence(frames, **kw)
        got = np.array([[np.nan] * 8 + [-1.0, np.nan] if e is None else
                        [float(getattr(e, f)) for f in O.EST_FIELDS] for e in ct.run_sequence(frames, **kw)])
        assert np.array_equal(got[:, 8], ref[:, 8]) and np.array_equal(got[:, 9], ref[:, 9]), (h, w, n, kw)
        fin = np.isfinite(ref[:, 5])
        if fin.any():
            err = np.max(np.abs(got[fin, 5] - ref[fin, 5]) / np.abs(ref[fin, 5]))
            assert err <= 1e-9, (h, w, n, kw, err)
