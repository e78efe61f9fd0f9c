"""GPU parity of the direct convolution kernels (K1-K4) against the reference
fixtures and the CPU oracle.  float64 must be bit-identical (same per-output
FMA order as the reference); float32 within 1e-5 relative inf-norm of the
float64 oracle on the float32-rounded inputs."""

import numpy as np
import pytest
import torch

import oracle as O
import paper_1612_08825_b200 as ct
from conftest import rel_inf
from paper_1612_08825_b200 import BoundaryPolicy, ConvMethod, ConvShape

pytestmark = pytest.mark.gpu

SHAPES = (ConvShape.FULL, ConvShape.SAME, ConvShape.VALID)
BOUNDS = (BoundaryPolicy.ZERO, BoundaryPolicy.REPLICATE)
F, S, V = ConvShape.FULL, ConvShape.SAME, ConvShape.VALID


def test_reference_fixture_cases_bit_exact(golden):
    z = golden("conv_cases.npz")
    for i in range(int(z["count"])):
        sh, bd, fl = (int(v) for v in z[f"c{i}_meta"])
        fn = ct.conv_direct if fl else ct.xcorr_direct
        got = fn(z[f"c{i}_s"], z[f"c{i}_k"], SHAPES[sh], BOUNDS[bd])
        ref = z[f"c{i}_out"]
        assert got.shape == ref.shape, i
        assert np.array_equal(got, ref), f"case {i}: max dev {np.abs(got - ref).max()}"


def test_cfg1_full_fp64_bit_exact(golden):
    c = golden("conv_configs.npz")
    s = np.random.Generator(np.random.PCG64(0)).random((256, 256))
    k = np.random.Generator(np.random.PCG64(1)).standard_normal((5, 5))
    got = ct.conv_direct(s, k, F)
    assert got.shape == (260, 260)
    assert np.array_equal(got, c["cfg1_out"])


def test_cfg1_batched_launch_matches_single(golden):
    c = golden("conv_configs.npz")
    base = np.random.Generator(np.random.PCG64(0)).random((256, 256))
    k = np.random.Generator(np.random.PCG64(1)).standard_normal((5, 5))
    rng = np.random.default_rng(5)
    batch = np.stack([base] + [rng.random((256, 256)) for _ in range(6)])
    out = ct.direct_batch(torch.from_numpy(batch).cuda(), k, F, flip=True).cpu().numpy()
    assert np.array_equal(out[0], c["cfg1_out"])
    for i in range(1, 7):
        assert np.array_equal(out[i], O.direct(batch[i], k, "full"))


def test_cfg3_fp32_within_tolerance(golden):
    c = golden("conv_configs.npz")
    s = np.random.Generator(np.random.PCG64(0)).random((128,) * 3).astype(np.float32)
    k = np.random.Generator(np.random.PCG64(1)).standard_normal((7,) * 3).astype(np.float32)
    got = ct.conv_direct(torch.from_numpy(s).cuda(), torch.from_numpy(k), F).cpu().numpy().astype(np.float64)
    assert got.shape == (134,) * 3
    ref_vals = c["cfg3_val"]
    err = np.abs(got.ravel()[c["cfg3_idx"]] - ref_vals).max() / float(c["cfg3_absmax"])
    assert err <= 1e-5, err
    assert abs(got.sum() - float(c["cfg3_sum"])) <= 1e-5 * abs(float(c["cfg3_sum"]))


def test_cfg4_fp32_within_tolerance(golden):
    c = golden("conv_configs.npz")
    s = np.random.Generator(np.random.PCG64(0)).random((2048, 2048)).astype(np.float32)
    k = np.random.Generator(np.random.PCG64(1)).standard_normal((31, 31)).astype(np.float32)
    got = ct.conv_direct(torch.from_numpy(s).cuda(), torch.from_numpy(k), F).cpu().numpy().astype(np.float64)
    assert got.shape == (2078, 2078)
    err = np.abs(got.ravel()[c["cfg4_idx"]] - c["cfg4_val"]).max() / float(c["cfg4_absmax"])
    assert err <= 1e-5, err


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("ndim", [1, 2, 3])
def test_random_shapes_all_modes_vs_oracle(dtype, ndim):
    rng = np.random.default_rng(100 + ndim)
    widths = [1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 13, 15, 16, 31, 33]
    for it in range(24):
        kx = widths[it % len(widths)]
        ks = tuple(int(rng.integers(1, 6)) for _ in range(ndim - 1)) + (kx,)
        ss = tuple(int(rng.integers(1, 40 if ndim < 3 else 14)) for _ in range(ndim - 1)) + (int(rng.integers(1, 90)),)
        s = rng.uniform(-1, 1, ss).astype(dtype)
        k = rng.uniform(-1, 1, ks).astype(dtype)
        for shape in SHAPES:
            if shape == V and any(m < n for m, n in zip(ss, ks)):
                continue
            for bd in (BOUNDS if shape == S else BOUNDS[:1]):
                for flip in (0, 1):
                    fn = ct.conv_direct if flip else ct.xcorr_direct
                    ref = O.direct(s.astype(np.float64), k.astype(np.float64), shape.value, bd.value, bool(flip))
                    if dtype == np.float64:
                        got = fn(s, k, shape, bd)
                        assert np.array_equal(got, ref), (ss, ks, shape, bd, flip)
                    else:
                        got = fn(torch.from_numpy(s).cuda(), torch.from_numpy(k), shape, bd).cpu().numpy()
                        assert got.dtype == np.float32
                        assert rel_inf(got, ref) <= 1e-5, (ss, ks, shape, bd, flip)


def test_rank4_and_rank5_generic_path():
    rng = np.random.default_rng(5)
    s = rng.uniform(-1, 1, (3, 4, 2, 3))
    k = rng.uniform(-1, 1, (2, 2, 2, 2))
    for shape in SHAPES:
        for bd in BOUNDS:
            assert np.array_equal(ct.conv_direct(s, k, shape, bd), O.direct(s, k, shape.value, bd.value, True))
    s5 = rng.uniform(-1, 1, (2, 3, 2, 3, 4))
    k5 = rng.uniform(-1, 1, (1, 2, 2, 1, 3))
    assert np.array_equal(ct.xcorr_direct(s5, k5, F), O.direct(s5, k5, "full", "zero", False))


def test_pinned_reference_values():  # test_conv.py:38-74
    s = np.array([1.0, 2.0, 3.0])
    k = np.array([1.0, 1.0])
    assert ct.conv_direct(s, k, F).tolist() == [1.0, 3.0, 5.0, 3.0]
    assert ct.conv_direct(s, k, S).tolist() == [1.0, 3.0, 5.0]
    assert ct.conv_direct(s, k, V).tolist() == [3.0, 5.0]
    k2 = np.array([1.0, 0.0, -1.0])
    assert ct.conv_direct(s, k2, F).tolist() == [1.0, 2.0, 2.0, -2.0, -3.0]
    assert ct.xcorr_direct(s, k2, F).tolist() == [-1.0, -2.0, -2.0, 2.0, 3.0]
    s5 = np.arange(1.0, 6.0)
    assert ct.conv_direct(s5, np.array([2.0, 3.0]), S).tolist() == ct.conv_direct(s5, np.array([2.0, 3.0]), F)[:5].tolist()
    assert ct.conv_direct(s5, np.ones(4), S).tolist() == ct.conv_direct(s5, np.ones(4), F)[1:6].tolist()
    out = ct.conv_direct(np.array([1.0, 2.0, 3.0]), np.ones(3) / 3.0, S, BoundaryPolicy.REPLICATE)
    assert np.allclose(out, [4 / 3, 2.0, 8 / 3], atol=1e-15)
    s3 = np.array([10.0, 20.0, 30.0])
    assert ct.xcorr_direct(s3, np.array([1.0, 1.0]), S, BoundaryPolicy.REPLICATE).tolist() == [20.0, 30.0, 50.0]
    assert ct.conv_direct(s3, np.array([1.0, 1.0]), S, BoundaryPolicy.REPLICATE).tolist() == [20.0, 30.0, 50.0]


def test_errors_are_value_errors():  # test_conv.py:76-85
    with pytest.raises(ValueError):
        ct.conv_direct(np.ones(3), np.ones(5), V)
    with pytest.raises(ValueError):
        ct.conv_direct(np.ones((4, 2)), np.ones((2, 3)), V)
    with pytest.raises(ValueError):
        ct.conv_direct(np.ones((3, 3)), np.ones(3), F)
    # numpy scalars are promoted to 1-D by ascontiguousarray, as in the
    # reference (conv.py:101-102): no zero-rank error, a 1-element result
    assert ct.conv_direct(np.float64(2.0), np.float64(3.0), F).tolist() == [6.0]
    assert ct.conv_direct(np.zeros((0,)), np.ones(3), S).shape == (0,)


def test_kernel_larger_than_signal_and_empty():  # test_conv.py:230-242
    rng = np.random.default_rng(11)
    for ms, ns in [((9,), (3,)), ((2,), (5,)), ((7, 6), (3, 4)), ((3, 3), (5, 2)), ((5, 6, 4), (2, 3, 3)),
                   ((2, 2, 2), (3, 1, 4))]:
        s = rng.uniform(-1, 1, ms)
        k = rng.uniform(-1, 1, ns)
        assert np.array_equal(ct.conv_direct(s, k, F), O.direct(s, k, "full"))
        assert np.array_equal(ct.conv_direct(s, k, S), O.direct(s, k, "same"))
    # empty signal: FULL is all zeros of extent n-1
    out = ct.conv_direct(np.zeros((0,)), np.ones(3), F)
    assert out.shape == (2,) and not out.any()


def test_conv_auto_dispatch_and_tags():  # test_conv.py:207-227, test_acceptance.py:134-145
    s = np.ones((40, 40))
    _, m1 = ct.conv_auto(s, np.ones((3, 3)), S, threshold=900)
    _, m2 = ct.conv_auto(s, np.ones((31, 31)), S, threshold=900)
    assert m1 == ConvMethod.DIRECT and m2 == ConvMethod.FFT
    _, m3 = ct.conv_auto(s, np.ones((30, 30)), S, threshold=900)
    _, m4 = ct.conv_auto(s, np.ones((30, 30)), S, threshold=901)
    assert m3 == ConvMethod.FFT and m4 == ConvMethod.DIRECT
    signal = np.ones(2000)
    for n in range(890, 910):
        _, chosen = ct.conv_auto(signal, np.ones(n), S, method=ConvMethod.AUTO, threshold=900)
        assert chosen == (ConvMethod.DIRECT if n < 900 else ConvMethod.FFT)
    rng = np.random.default_rng(4)
    s2 = rng.standard_normal((12, 13))
    k2 = rng.standard_normal((4, 5))
    r1, t1 = ct.conv_auto(s2, k2, S, BoundaryPolicy.REPLICATE, ConvMethod.DIRECT)
    r2, t2 = ct.conv_auto(s2, k2, S, BoundaryPolicy.REPLICATE, ConvMethod.FFT)
    assert (t1, t2) == (ConvMethod.DIRECT, ConvMethod.FFT)
    assert np.allclose(r1, r2, atol=1e-10)


def test_properties_linearity_commutativity_delta():  # test_conv.py:181-243
    rng = np.random.default_rng(0)
    s = rng.standard_normal((6, 7))
    k1, k2 = rng.standard_normal((3, 3)), rng.standard_normal((3, 3))
    assert np.allclose(ct.conv_direct(s, 2.0 * k1 - 0.5 * k2, F),
                       2.0 * ct.conv_direct(s, k1, F) - 0.5 * ct.conv_direct(s, k2, F), atol=1e-12)
    assert np.allclose(ct.conv_direct(s, k1, F), ct.conv_direct(k1, s, F), atol=1e-12)
    assert np.array_equal(ct.conv_direct(s, np.array([[1.0]]), F), s)
    out = ct.conv_direct(np.full((4, 5), 3.0), np.array([[1.0, 2.0], [0.5, 1.5]]), S, BoundaryPolicy.REPLICATE)
    assert np.allclose(out, 3.0 * 5.0, atol=1e-12)
    assert np.allclose(ct.conv_direct(s, k1, F), ct.xcorr_direct(s, ct.reflect(k1), F), atol=0)


def test_large_batch_fullsize_roundtrip_property():
    # size-independent check at the bench size: linearity in the signal across a big batch
    rng = np.random.default_rng(8)
    k = rng.standard_normal((5, 5))
    a = torch.rand((64, 256, 256), dtype=torch.float64, device="cuda")
    b = torch.rand((64, 256, 256), dtype=torch.float64, device="cuda")
    oa = ct.direct_batch(a, k)
    ob = ct.direct_batch(b, k)
    oab = ct.direct_batch(a + b, k)
    assert torch.allclose(oab, oa + ob, rtol=0, atol=1e-12)
    i = 37
    assert np.array_equal(oa[i].cpu().numpy(), O.direct(a[i].cpu().numpy(), k, "full"))


@pytest.mark.parametrize("kind", ["0", "1", "2", "6"])
def test_each_kernel_variant_matches_oracle(kind, monkeypatch):
    """Pin each tiled variant (0 register-tiled, 1 fp32 row-pair FFMA2, 2 TMA-staged
    persistent) and compare with the oracle: fp64 bit-exact, fp32 within 1e-5."""
    monkeypatch.setenv("CT_CONV_KIND", kind)
    rng = np.random.default_rng(int(kind) + 40)
    for ms, ns, shape in [((256, 256), (5, 5), F), ((300, 260), (3, 3), F), ((97, 131), (5, 5), S),
                          ((64, 96), (7, 9), F), ((40, 200), (5, 31), F), ((33, 47), (5, 5), V)]:
        s64 = rng.random((3,) + ms)
        k64 = rng.standard_normal(ns)
        got = ct.direct_batch(torch.from_numpy(s64).cuda(), k64, shape, flip=True).cpu().numpy()
        for i in range(3):
            assert np.array_equal(got[i], O.direct(s64[i], k64, shape.value, "zero", True)), (kind, ms, ns)
        s32 = s64.astype(np.float32)
        k32 = k64.astype(np.float32)
        g32 = ct.direct_batch(torch.from_numpy(s32).cuda(), k32, shape, flip=True).cpu().numpy()
        for i in range(3):
            ref = O.direct(s32[i].astype(np.float64), k32.astype(np.float64), shape.value, "zero", True)
            assert rel_inf(g32[i], ref) <= 1e-5, (kind, ms, ns)


@pytest.mark.parametrize("kind", ["0", "1", "3", "4", "5", "7"])
def test_each_3d_kernel_variant_matches_oracle(kind, monkeypatch):
    """3-D shapes with each tiled variant pinned (3 = TMA-staged z-slices, used for
    zero extension with 16-byte rows; odd rows fall back): fp64 bit-exact, fp32 1e-5."""
    monkeypatch.setenv("CT_CONV_KIND", kind)
    rng = np.random.default_rng(int(kind) + 70)
    for ms, ns, shape in [((20, 33, 64), (5, 5, 5), F), ((17, 40, 36), (3, 3, 3), S),
                          ((9, 24, 32), (3, 5, 7), V), ((12, 30, 41), (3, 3, 5), F),
                          ((6, 70, 300), (2, 4, 9), S), ((30, 20, 28), (7, 7, 7), F),
                          ((40, 12, 20), (7, 7, 7), V), ((3, 90, 76), (5, 5, 5), S)]:
        s64 = rng.random((2,) + ms)
        k64 = rng.standard_normal(ns)
        got = ct.direct_batch(torch.from_numpy(s64).cuda(), k64, shape, flip=False).cpu().numpy()
        for i in range(2):
            assert np.array_equal(got[i], O.direct(s64[i], k64, shape.value, "zero", False)), (kind, ms, ns)
        s32 = s64.astype(np.float32)
        k32 = k64.astype(np.float32)
        g32 = ct.direct_batch(torch.from_numpy(s32).cuda(), k32, shape, flip=False).cpu().numpy()
        for i in range(2):
            ref = O.direct(s32[i].astype(np.float64), k32.astype(np.float64), shape.value, "zero", False)
            assert rel_inf(g32[i], ref) <= 1e-5, (kind, ms, ns)


def test_cuda_graph_capture_replays_bit_identical():
    """direct_batch can be captured into a CUDA graph after a warm-up call (no
    host synchronisation or host->device copy on the launch path; the autotuner
    never times candidates while the stream is capturing) and the replay equals
    the eager result."""
    rng = np.random.default_rng(5)
    k = rng.standard_normal((5, 5))
    s = torch.from_numpy(rng.random((64, 300, 260))).cuda()
    eager = ct.direct_batch(s, k, F)
    out = torch.empty_like(eager)
    ct.direct_batch(s, k, F, out=out)  # warm-up: device taps cached, variant chosen
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ct.direct_batch(s, k, F, out=out)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager)


# widths without a tiled instantiation take the width-generic strip kernel
# (xcorr_strip: runtime width, 8-tap compile-time strips + exact tail);
# fp64 stays bit-identical to the reference order, fp32 within 1e-5
STRIP_CASES = [
    ((300,), (13,)), ((257,), (40,)), ((70, 90), (13, 13)), ((64, 77), (5, 10)), ((50, 61), (3, 16)),
    ((41, 45), (12, 17)), ((33, 40), (20, 33)), ((19, 23, 29), (3, 4, 13)), ((12, 14, 20), (5, 2, 10)),
]


@pytest.mark.parametrize("ss,ks", STRIP_CASES)
def test_width_generic_strip_kernel_fp64_bit_exact(ss, ks):
    rng = np.random.default_rng(sum(ss) + 7 * sum(ks))
    s = rng.random(ss)
    k = rng.standard_normal(ks)
    for shape in SHAPES:
        if shape == V and any(a < b for a, b in zip(ss, ks)):
            continue
        for bd in BOUNDS:
            for fn, flip in ((ct.conv_direct, True), (ct.xcorr_direct, False)):
                got = fn(s, k, shape, bd)
                ref = O.direct(s, k, shape.name.lower(), bd.name.lower() if shape == S else "zero", flip=flip)
                assert np.array_equal(got, ref), (ss, ks, shape, bd, flip, np.abs(got - ref).max())


@pytest.mark.parametrize("ss,ks", STRIP_CASES[2:7])
def test_width_generic_strip_kernel_fp32(ss, ks):
    rng = np.random.default_rng(3 + sum(ss))
    s = rng.random(ss).astype(np.float32)
    k = rng.standard_normal(ks).astype(np.float32)
    got = ct.conv_direct(torch.from_numpy(s).cuda(), torch.from_numpy(k), F).cpu().numpy()
    assert got.dtype == np.float32
    assert rel_inf(got, O.direct(s.astype(np.float64), k.astype(np.float64), "full")) <= 1e-5


def test_width_generic_batches_and_large_kernels():
    # batched launch == the oracle per image; a 90x90 kernel (8100 taps) still stages in shared memory
    rng = np.random.default_rng(13)
    s = torch.from_numpy(rng.random((5, 96, 130))).cuda()
    k = rng.standard_normal((13, 13))
    a = ct.direct_batch(s, k, F, flip=True).cpu().numpy()
    for i in range(5):
        assert np.array_equal(a[i], O.direct(s[i].cpu().numpy(), k, "full"))
    big = rng.standard_normal((90, 90))           # 8100 taps: shared-memory bound still fits
    t = rng.random((120, 130))
    assert np.array_equal(ct.xcorr_direct(t, big, F), O.direct(t, big, "full", flip=False))


@pytest.mark.parametrize("kind", ["4", "7"])
def test_zwalk_work_balanced_runs_match_flat_split_and_oracle(kind, monkeypatch):
    """A batch large enough that the z-walk kernels cut every column into runs of
    equal work (one run per CTA): identical bits to the flat split (the
    per-output tap order does not depend on where a run starts) and to the
    oracle in fp64 (kind 4); fp32 within 1e-5 (kinds 4 and 7, plane pairs)."""
    monkeypatch.setenv("CT_CONV_KIND", kind)
    rng = np.random.default_rng(90 + int(kind))
    k64 = rng.standard_normal((7, 7, 7))
    s64 = rng.random((8, 64, 96, 96))
    for dt in (np.float32, np.float64):
        if kind == "7" and dt is np.float64:
            continue  # the plane-pair kernel is fp32 only
        s, k = torch.from_numpy(s64.astype(dt)).cuda(), k64.astype(dt)
        monkeypatch.delenv("CT_ZW_FLAT", raising=False)
        bal = ct.direct_batch(s, k, F, flip=False).cpu().numpy()
        monkeypatch.setenv("CT_ZW_FLAT", "1")
        flat = ct.direct_batch(s, k, F, flip=False).cpu().numpy()
        monkeypatch.delenv("CT_ZW_FLAT", raising=False)
        assert np.array_equal(bal, flat), (kind, dt)
        for i in (0, 7):
            ref = O.direct(s64[i].astype(dt).astype(np.float64), k.astype(np.float64), "full", "zero", False)
            if dt is np.float64:
                assert np.array_equal(bal[i], ref), (kind, i)
            else:
                assert rel_inf(bal[i], ref) <= 1e-5, (kind, i)


def test_strip_kernel_paths_agree_bit_for_bit(monkeypatch):
    """The width-generic 2-D paths -- TMA-staged tiles with the fitted thread
    block (default), the LDG-staged kernel (CT_CONV_NOTMA) and the fixed 32 x 8
    block (CT_STRIP_FIXED_TILE) -- give the oracle's bits in fp64 and agree with
    one another in fp32 (same per-output tap order on every path)."""
    rng = np.random.default_rng(77)
    for ms, ns, shape in [((268, 300), (13, 13), F), ((130, 257), (10, 17), S), ((96, 200), (12, 20), V),
                          ((64, 512), (33, 33), F)]:
        s64 = rng.random((3,) + ms)
        k64 = rng.standard_normal(ns)
        outs = {}
        for name, env in (("tma", {}), ("ldg", {"CT_CONV_NOTMA": "1"}), ("fixed", {"CT_STRIP_FIXED_TILE": "1"}),
                          ("ldg_fixed", {"CT_CONV_NOTMA": "1", "CT_STRIP_FIXED_TILE": "1"})):
            for key in ("CT_CONV_NOTMA", "CT_STRIP_FIXED_TILE"):
                monkeypatch.delenv(key, raising=False)
            for key, val in env.items():
                monkeypatch.setenv(key, val)
            g64 = ct.direct_batch(torch.from_numpy(s64).cuda(), k64, shape, flip=True).cpu().numpy()
            g32 = ct.direct_batch(torch.from_numpy(s64.astype(np.float32)).cuda(), k64.astype(np.float32), shape,
                                  flip=True).cpu().numpy()
            outs[name] = (g64, g32)
        for key in ("CT_CONV_NOTMA", "CT_STRIP_FIXED_TILE"):
            monkeypatch.delenv(key, raising=False)
        for i in range(3):
            ref = O.direct(s64[i], k64, shape.value, "zero", True)
            for name, (g64, _) in outs.items():
                assert np.array_equal(g64[i], ref), (name, ms, ns)
        for name, (_, g32) in outs.items():
            assert np.array_equal(g32, outs["tma"][1]), (name, ms, ns)
