"""GPU parity of the TTC path (K5-K7 + pyramid + generator) against the
reference fixtures and the CPU oracle.

Tolerances (BASELINE north_star, relative inf-norm per SURVEY.md D5):
  * float64 derivative fields, G, downsample, generator frames: bit-exact
    (same per-element operation order as the reference);
  * float64 normal-system sums: 1e-12 relative (reduction order differs);
  * float64 per-pair TTC (and a, b, c, FOE): 1e-9 relative;
  * float32 path (config 5 convention, oracle = float64 reference on the
    float32-rounded frames): sums and TTC within 1e-4 relative.
"""

import hashlib

import numpy as np
import pytest
import torch

import oracle as O
import paper_1612_08825_b200 as ct
from conftest import rel_inf
from paper_1612_08825_b200 import FramePair, NormalSystem

pytestmark = pytest.mark.gpu

EST = ("a", "b", "c", "x0", "y0", "ttc", "residual", "misfit", "level", "degenerate")


def rows(ests):
    return np.array([[float(getattr(e, f)) for f in EST] for e in ests])


def assert_est_close(got, ref, rtol, fields=(0, 1, 2, 3, 4, 5)):
    got = np.asarray(got)
    ref = np.asarray(ref)
    assert got.shape == ref.shape
    assert np.array_equal(got[..., 8], ref[..., 8]), "level differs"
    assert np.array_equal(got[..., 9], ref[..., 9]), "degenerate flag differs"
    for f in fields:
        g, r = got[..., f], ref[..., f]
        assert np.array_equal(np.isnan(g), np.isnan(r)), EST[f]
        fin = np.isfinite(r)
        assert np.array_equal(np.isinf(g), np.isinf(r)), EST[f]
        if fin.any():
            err = np.max(np.abs(g[fin] - r[fin]) / np.maximum(np.abs(r[fin]), 1e-300))
            assert err <= rtol, f"{EST[f]} rel err {err:.3e} > {rtol}"


@pytest.fixture(scope="module")
def cfg2_frames():
    return O.generate(256, 256, 64, 100.0, (0.5, 0.5), 0, 0.0)


def test_device_generator_bit_exact(golden, cfg2_frames):
    t = golden("ttc_fixtures.npz")
    seq = ct.generate(ct.SynthConfig(width=256, height=256, frames=64, t0=100.0, foe=(0.5, 0.5), seed=0))
    f, truth = seq.frames, seq.truth
    assert isinstance(f, np.ndarray) and f.dtype == np.float64 and truth.shape == (64, 4)
    assert hashlib.sha256(f.tobytes()).hexdigest() == str(t["cfg2_frames_sha"])
    assert np.array_equal(truth[:, 1], 100.0 - np.arange(64))
    fn = ct.generate(ct.SynthConfig(width=128, height=128, frames=12, t0=60.0, foe=(0.5, 0.5), seed=2,
                                    noise_sigma=0.05), device=True).frames
    assert fn.is_cuda
    assert hashlib.sha256(fn.cpu().numpy().tobytes()).hexdigest() == str(t["noisy_frames_sha"])


def test_fields_bit_exact(golden):
    t = golden("ttc_fixtures.npz")
    a, b = t["small_a"], t["small_b"]
    ex, ey, et = ct.derivatives_3d(FramePair(a, b))
    assert np.array_equal(ex, t["small_ex"]) and np.array_equal(ey, t["small_ey"]) and np.array_equal(et, t["small_et"])
    g = ct.radial_gradient(ex, ey)
    assert np.array_equal(g, t["small_g"])
    ns = ct.build_normal_system(ex, ey, g, et, border=1)
    ref = t["small_sums_b1"]
    got = np.array([ns.m[0, 0], ns.m[0, 1], ns.m[0, 2], ns.m[1, 1], ns.m[1, 2], ns.m[2, 2], *ns.rhs, ns.et2, ns.count])
    assert np.max(np.abs(got - ref) / np.abs(ref)) <= 1e-12
    ns3 = ct.build_normal_system(ex, ey, g, et, border=3)
    assert ns3.count == t["small_sums_b3"][10]
    assert np.array_equal(ct.downsample(a), t["small_down"])
    assert np.array_equal(ct.downsample(ct.downsample(a)), t["small_down2"])


def test_solver_bit_exact_given_sums(golden):
    t = golden("ttc_fixtures.npz")
    s = t["small_sums_b1"]
    sys_ = NormalSystem(m=np.array([[s[0], s[1], s[2]], [s[1], s[3], s[4]], [s[2], s[4], s[5]]]), rhs=s[6:9],
                        et2=s[9], count=int(s[10]))
    est = ct.solve_ttc(sys_)
    assert np.array_equal(rows([est])[0], t["small_est"], equal_nan=True)


def test_solver_reference_cases():  # test_ttc.py:80-122
    rng = np.random.default_rng(42)
    for _ in range(50):
        r = rng.standard_normal((3, 3))
        m = r.T @ r + 1e-3 * np.eye(3)
        rhs = rng.standard_normal(3)
        est = ct.solve_ttc(NormalSystem(m=m, rhs=rhs, et2=50.0, count=10))
        assert not est.degenerate
        assert np.allclose([est.a, est.b, est.c], np.linalg.solve(m, rhs), rtol=1e-8, atol=1e-10)
        sums = np.array([m[0, 0], m[0, 1], m[0, 2], m[1, 1], m[1, 2], m[2, 2], *rhs, 50.0, 10.0])
        assert np.array_equal(rows([est])[0], O.solve_ttc(sums), equal_nan=True)
    est = ct.solve_ttc(NormalSystem(m=np.diag([2.0, 4.0, 8.0]), rhs=np.array([2.0, 4.0, 8.0]), et2=20.0, count=4))
    assert est.residual == pytest.approx(1.5) and est.misfit == pytest.approx(0.3)
    assert est.ttc == pytest.approx(1.0) and est.x0 == pytest.approx(-1.0) and est.y0 == pytest.approx(-1.0)
    zero = ct.solve_ttc(NormalSystem(m=np.zeros((3, 3)), rhs=np.zeros(3), et2=0.0, count=9))
    assert zero.degenerate and np.isnan(zero.ttc) and np.isinf(zero.misfit)
    assert ct.solve_ttc(NormalSystem(m=np.diag([1.0, 1.0, 1e-15]), rhs=np.ones(3), et2=1.0, count=9)).degenerate
    inf = ct.solve_ttc(NormalSystem(m=np.eye(3), rhs=np.array([0.5, -0.25, 0.0]), et2=1.0, count=4))
    assert not inf.degenerate and np.isinf(inf.ttc) and inf.ttc > 0 and np.isnan(inf.x0) and inf.a == pytest.approx(0.5)


def test_cfg2_run_sequence_level0(golden, cfg2_frames):
    t = golden("ttc_fixtures.npz")
    got = rows(ct.run_sequence(cfg2_frames, level=0))
    assert_est_close(got, t["cfg2_l0"], 1e-9, fields=(0, 1, 2, 3, 4, 5, 6, 7))
    # SURVEY.md 8(c) anchors
    assert got[0, 5] == pytest.approx(97.315722253398093, rel=1e-9)
    assert got[31, 5] == pytest.approx(63.514498981613194, rel=1e-9)
    assert got[62, 5] == pytest.approx(33.849933824360562, rel=1e-9)


@pytest.mark.parametrize("key,kw", [("cfg2_l1", dict(level=1)), ("cfg2_l2", dict(level=2)),
                                    ("cfg2_ms5", dict(max_level=5))])
def test_cfg2_levels_and_multiscale(golden, cfg2_frames, key, kw):
    t = golden("ttc_fixtures.npz")
    got = rows(ct.run_sequence(cfg2_frames[:9], **kw))
    assert_est_close(got, t[key], 1e-9)


def test_device_resident_batch_matches_host_path(cfg2_frames):
    f = torch.from_numpy(cfg2_frames).cuda()
    batch = torch.stack([f, f.flip(0), f * 0.5 + 0.25])
    est = ct.run_sequence_batch(batch, level=0).cpu().numpy()
    for v in range(3):
        ref = O.run_sequence(batch[v].cpu().numpy(), level=0)
        assert_est_close(est[v], ref, 1e-9, fields=(0, 1, 2, 3, 4, 5, 6, 7))
    host = ct.run_sequence_host(batch.cpu().numpy(), level=0)
    assert np.array_equal(host, est)  # same kernels, same reduction order -> identical


def test_moments_sums_vs_oracle_fp64(cfg2_frames):
    from paper_1612_08825_b200 import _lib
    f = torch.from_numpy(cfg2_frames[:12]).cuda()
    L = _lib.load()
    n = 12
    sums = torch.empty((n - 1, 11), dtype=torch.float64, device="cuda")
    nb = L.ct_ttc_moments_workspace_bytes(_lib.CT_F64, 1, n, 256, 256)
    ws = _lib.workspace(nb, "cuda")
    _lib.check(L.ct_ttc_moments(_lib.CT_F64, _lib.ptr(f), 1, n, 256, 256, _lib.ptr(sums), _lib.ptr(ws), nb,
                                _lib.stream_ptr()))
    got = sums.cpu().numpy()
    for i in range(n - 1):
        ex, ey, et = O.derivatives(cfg2_frames[i], cfg2_frames[i + 1])
        ref = O.normal_system(ex, ey, O.radial_gradient(ex, ey), et, 1)
        assert np.max(np.abs(got[i] - ref) / np.abs(ref)) <= 1e-12, i


def test_odd_shapes_fallback_loader():
    # widths whose rows are not 16-byte multiples take the non-TMA loader
    rng = np.random.default_rng(3)
    for h, w in [(37, 50), (33, 257), (300, 29), (5, 5), (64, 511)]:
        fr = O.generate(max(w, 16), max(h, 16), 4, 30.0, (0.4, 0.6), 7, 0.0)[:, :h, :w] + 0.01 * rng.random((4, h, w))
        got = rows(ct.run_sequence(fr, level=0))
        ref = O.run_sequence(fr, level=0)
        assert_est_close(got, ref, 1e-9)
        # residual/misfit come from et2 - v.rhs, a cancellation that amplifies
        # the 1e-16 sum differences on tiny interiors (3x3 at 5x5 frames)
        assert_est_close(got, ref, 1e-6, fields=(6, 7))


def test_noisy_multiscale_vs_reference(golden):
    t = golden("ttc_fixtures.npz")
    fn = ct.generate(ct.SynthConfig(width=128, height=128, frames=12, t0=60.0, foe=(0.5, 0.5), seed=2,
                                    noise_sigma=0.05), device=True).frames
    got = rows(ct.run_sequence(fn.cpu().numpy(), max_level=5))
    assert_est_close(got, t["noisy_ms5"], 1e-9)
    got0 = rows(ct.run_sequence(fn, level=0))  # device tensor input
    assert_est_close(got0, t["noisy_l0"], 1e-9)


def test_fp32_multiscale_config5_convention(golden):
    t = golden("ttc_fixtures.npz")
    f64 = O.generate(480, 270, 4, 300.0, (0.5, 0.5), 11, 0.0)
    f32 = torch.from_numpy(f64.astype(np.float32)).cuda()
    est = ct.run_sequence_batch(f32[None], max_level=3).cpu().numpy()[0]
    ref = t["c5_ms3"]
    assert np.array_equal(est[:, 8], ref[:, 8])
    assert_est_close(est, ref, 1e-4, fields=(2, 5))
    # each level separately
    for lv in range(4):
        e = ct.run_sequence_batch(f32[None, :2], level=lv).cpu().numpy()[0, 0]
        assert abs(e[5] - t["c5_l"][lv][5]) <= 1e-4 * abs(t["c5_l"][lv][5]), lv
    # fp32 pyramid level vs float64 reference downsample of the rounded frame
    d = ct.downsample(f32[0]).cpu().numpy()
    assert rel_inf(d, t["c5_down"]) <= 1e-6


def test_degenerate_and_none_semantics():  # test_ttc.py:125-129, 200-212
    est = ct.estimate_fixed(FramePair(np.full((32, 32), 0.5), np.full((32, 32), 0.5)), level=0)
    assert est.degenerate and np.isnan(est.ttc)
    assert ct.estimate_multiscale(FramePair(np.zeros((32, 32)), np.zeros((32, 32))), max_level=3).degenerate
    assert ct.estimate_multiscale(FramePair(np.ones((3, 8)), np.ones((3, 8))), max_level=2) is None
    with pytest.raises(ValueError):
        ct.estimate_fixed(FramePair(np.ones((16, 16)), np.ones((16, 16))), level=3)
    with pytest.raises(ValueError):
        ct.estimate_fixed(FramePair(np.ones((16, 16)), np.ones((16, 16))), level=-1)
    with pytest.raises(ValueError):
        ct.run_sequence(np.ones((1, 8, 8)))
    with pytest.raises(ValueError):
        ct.run_sequence(np.ones((8, 8)))
    with pytest.raises(ValueError):
        FramePair(np.ones((3, 3)), np.ones((3, 4)))


def test_multiscale_zero_levels_equals_fixed():  # test_ttc.py:190-197
    f = O.generate(64, 64, 2, 30.0, (0.5, 0.5), 6, 0.0)
    pair = FramePair(f[0], f[1])
    ms = ct.estimate_multiscale(pair, max_level=0)
    fx = ct.estimate_fixed(pair, level=0)
    assert ms.level == 0 and ms.ttc == fx.ttc


def test_shard_count_invariance_bitwise(cfg2_frames):
    # temporal sharding with a one-frame halo gives identical rows (no cross-pair state)
    full = ct.run_sequence_batch(torch.from_numpy(cfg2_frames).cuda()[None], level=0)[0].cpu().numpy()
    for shards in (2, 3, 8):
        bounds = np.linspace(0, 63, shards + 1).astype(int)
        parts = [ct.run_sequence_batch(torch.from_numpy(cfg2_frames[a:b + 1]).cuda()[None], level=0)[0].cpu().numpy()
                 for a, b in zip(bounds[:-1], bounds[1:])]
        assert np.array_equal(np.concatenate(parts), full)


def test_full_size_batch_properties():
    # size-independent checks at the bench size: pair (t, t) gives Et == 0 -> zero
    # misfit numerator and degenerate-free; swapping every frame pair in time flips c
    f = ct.generate(ct.SynthConfig(width=256, height=256, frames=64, t0=100.0, foe=(0.5, 0.5), seed=0), device=True).frames
    fwd = ct.run_sequence_batch(f[None], level=0)[0].cpu().numpy()
    rev = ct.run_sequence_batch(f.flip(0)[None], level=0)[0].cpu().numpy()[::-1]
    # reversing time negates Et: c (and a, b) flip sign exactly
    assert np.array_equal(rev[:, 2], -fwd[:, 2])
    assert np.array_equal(rev[:, 0], -fwd[:, 0])


def test_batched_textures_match_single():
    seeds = [0, 5, 17]
    batch = ct.make_textures(64, 48, seeds)
    for j, s in enumerate(seeds):
        assert torch.equal(batch[j], ct.make_texture_device(64, 48, s))
        assert np.array_equal(batch[j].cpu().numpy(), ct.make_texture(64, 48, s))
    ref = O.make_texture(64, 48, 5)
    assert np.array_equal(batch[1].cpu().numpy(), ref)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("hw", [(270, 480), (135, 244), (66, 130), (101, 77), (9, 1100), (300, 36)])
def test_blur_variants_bit_identical(monkeypatch, dtype, hw):
    """The three multiscale blur stages (TMA-fed per-warp window, register
    window with global loads, shared-memory tile) use the same FMA chains:
    multiscale estimates must be bit-identical (odd widths take the
    shared-memory stage in every mode)."""
    f = torch.from_numpy(O.generate(hw[1], hw[0], 5, 80.0, (0.4, 0.55), 3, 0.0)).to(dtype).cuda()
    lv = 3 if min(hw) >= 64 else 1
    a = ct.run_sequence_batch(f[None], max_level=lv).cpu().numpy()
    monkeypatch.setenv("CT_BLUR_REGS", "1")
    b = ct.run_sequence_batch(f[None], max_level=lv).cpu().numpy()
    monkeypatch.setenv("CT_BLUR_SMEM", "1")
    c = ct.run_sequence_batch(f[None], max_level=lv).cpu().numpy()
    assert np.array_equal(np.nan_to_num(a, nan=7.0), np.nan_to_num(b, nan=7.0))
    assert np.array_equal(np.nan_to_num(a, nan=7.0), np.nan_to_num(c, nan=7.0))


@pytest.mark.parametrize("bc", ["128", "256"])
def test_wide_frames_both_tile_widths_vs_oracle(monkeypatch, bc):
    """Frames wider than one tile (several column tiles, TMA stride BC-4) with
    either tile width agree with the oracle: fp64 TTC 1e-9, fp32 multiscale 1e-4."""
    monkeypatch.setenv("CT_MOM_BC", bc)
    f64 = O.generate(700, 90, 5, 60.0, (0.45, 0.5), 9, 0.0)
    got = ct.run_sequence_batch(torch.from_numpy(f64).cuda()[None], level=0).cpu().numpy()[0]
    ref = O.run_sequence(f64, level=0)
    assert_est_close(got, ref, 1e-9)
    f32 = f64.astype(np.float32)
    got32 = ct.run_sequence_batch(torch.from_numpy(f32).cuda()[None], max_level=2).cpu().numpy()[0]
    ref32 = O.run_sequence(f32.astype(np.float64), max_level=2)
    assert np.array_equal(got32[:, 8], ref32[:, 8])
    assert_est_close(got32, ref32, 1e-4, fields=(5,))


def test_randomized_shapes_levels_and_precisions():
    """Seeded sweep over frame shapes around the tiling boundaries (band
    heights, 255/256/257-column tiles, multi-tile strides), frame counts,
    fixed levels and multiscale, both precisions, batched videos."""
    rng = np.random.default_rng(2024)
    shapes = [(17, 256), (33, 255), (48, 257), (65, 380), (16, 129), (100, 124), (31, 1000), (70, 508)]
    for i, (h, w) in enumerate(shapes):
        n = int(rng.integers(2, 6))
        nv = int(rng.integers(1, 4))
        vids = np.stack([O.generate(w, h, n, float(rng.uniform(30, 200)), (float(rng.uniform(0.3, 0.7)), 0.5),
                                    100 + 10 * i + v, 0.002) for v in range(nv)])
        dev = torch.from_numpy(vids).cuda()
        lv = int(rng.integers(0, 2)) if min(h, w) >= 32 else 0
        got = ct.run_sequence_batch(dev, level=lv).cpu().numpy()
        for v in range(nv):
            ref = O.run_sequence(vids[v], level=lv)
            assert_est_close(got[v], ref, 1e-9)
        if min(h, w) >= 64:
            got = ct.run_sequence_batch(dev, max_level=2).cpu().numpy()
            for v in range(nv):
                assert_est_close(got[v], O.run_sequence(vids[v], max_level=2), 1e-9)
        f32 = vids.astype(np.float32)
        got = ct.run_sequence_batch(torch.from_numpy(f32).cuda(), level=0).cpu().numpy()
        for v in range(nv):
            ref = O.run_sequence(f32[v].astype(np.float64), level=0)
            assert_est_close(got[v], ref, 1e-4, fields=(5,))


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_pyramid_moments_vs_oracle(dtype):
    """ct_ttc_pyramid_moments: per-level sums equal the oracle's normal system
    on the oracle's downsampled frames (fp64 1e-12 relative; fp32 frames 1e-5
    against the fp64 reference of the rounded frames), and level 0 equals
    ct_ttc_moments."""
    f64 = O.generate(300, 140, 4, 80.0, (0.45, 0.5), 21, 0.0)
    f = f64.astype(np.float32).astype(np.float64) if dtype == torch.float32 else f64
    dev = torch.from_numpy(f).to(dtype).cuda()[None]
    got = ct.pyramid_moments(dev, 3).cpu().numpy()
    assert got.shape == (3, 1, 3, 11)
    lv = [f[i] for i in range(4)]
    tol = 1e-12 if dtype == torch.float64 else 1e-5
    for level in range(3):
        for i in range(3):
            ex, ey, et = O.derivatives(lv[i], lv[i + 1])
            ref = O.normal_system(ex, ey, O.radial_gradient(ex, ey), et, 1)
            err = np.max(np.abs(got[level, 0, i, :10] - ref[:10])) / np.max(np.abs(ref[:10]))
            assert err <= tol, (level, i, err)
            assert got[level, 0, i, 10] == ref[10]
        lv = [O.downsample(x) for x in lv]
    with pytest.raises(ValueError, match="halvings"):
        ct.pyramid_moments(dev, 7)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_fused_multiscale_epilogue_matches_composed_stages(dtype):
    """run_sequence's multiscale pipeline (block means fused into the level-0
    moments, blurs emitting the next level's block means, levels >= 1 in one
    moments launch, one finalize + solve + level-walk epilogue) equals the
    composed C-ABI stages: ct_ttc_pyramid_moments, ct_ttc_solve per level,
    ct_ttc_multiscale_select.  Same sums up to the reduction order: selected
    level and degeneracy identical, a/b/c/FOE/TTC within 1e-12 (fp64) or
    1e-6 (fp32), on a batch of three videos with 1080p-like aspect."""
    from paper_1612_08825_b200 import _lib
    L = _lib.load()
    vids = np.stack([O.generate(384, 216, 7, float(t0), (0.45, 0.55), 40 + v, 0.001)
                     for v, t0 in enumerate((60.0, 150.0, 400.0))])
    dev = torch.from_numpy(vids).to(dtype).cuda()
    nl = 4
    got = ct.run_sequence_batch(dev, max_level=nl - 1).cpu().numpy()
    sums = ct.pyramid_moments(dev, nl)                      # [nl, V, n-1, 11]
    V, npair = sums.shape[1], sums.shape[2]
    count = V * npair
    est_levels = torch.empty((count, nl, 10), dtype=torch.float64, device="cuda")
    for lv in range(nl):
        e = torch.empty((count, 10), dtype=torch.float64, device="cuda")
        s = sums[lv].reshape(count, 11).contiguous()
        _lib.check(L.ct_ttc_solve(_lib.ptr(s), count, 1e-9, lv, _lib.ptr(e), _lib.stream_ptr()))
        est_levels[:, lv] = e
    best = torch.empty((count, 10), dtype=torch.float64, device="cuda")
    _lib.check(L.ct_ttc_multiscale_select(_lib.ptr(est_levels), count, nl, _lib.ptr(best), _lib.stream_ptr()))
    ref = best.cpu().numpy().reshape(V, npair, 10)
    assert_est_close(got, ref, 1e-12 if dtype == torch.float64 else 1e-6)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_run_sequence_cuda_graph_replay(dtype):
    """The device pipeline (multiscale and single-scale) captures into a CUDA
    graph (kernel parameters and TMA maps are by value, workspaces come from
    the capture pool) and replays bit-identically to eager calls on new
    frame contents copied into the static input."""
    g = torch.Generator(device="cuda").manual_seed(11)
    static = torch.rand((2, 6, 270, 480), dtype=dtype, device="cuda", generator=g)
    for kw in ({"max_level": 2}, {"level": 0}):
        ct.run_sequence_batch(static, **kw)  # warm (first-call setup outside the capture)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            out = ct.run_sequence_batch(static, **kw)
        for _ in range(3):
            new = torch.rand(static.shape, dtype=dtype, device="cuda", generator=g)
            static.copy_(new)
            graph.replay()
            torch.cuda.synchronize()
            ref = ct.run_sequence_batch(new, **kw)
            assert torch.equal(out.nan_to_num(7.0), ref.nan_to_num(7.0))


# fp32 multiscale path at 1080x1920 against the fp64 reference on the
# fp32-rounded frames.  Measured on B200 (round 2): c and ttc 1.5e-7 relative,
# residual and misfit 4.4e-6, FOE within 2.4e-4 px (x0 1.6e-4, y0 2.3e-4).  a and b are near zero for a
# centred FOE (a = -c * x0 with x0 ~ 1.5 px from the grid centre), so their
# relative error (up to 1.2e-3) measures nothing; they are held to the FOE
# scale instead: |da| <= tol * |c| (an FOE shift of tol px), same for b.
CFG5_TOL = {"c": 1e-6, "ttc": 1e-6, "residual": 2e-5, "misfit": 2e-5}
CFG5_FOE_PX = 1e-2


def field_errors(got, ref):
    errs = {}
    for f, name in enumerate(EST[:8]):
        g, r = got[..., f], ref[..., f]
        assert np.array_equal(np.isnan(g), np.isnan(r)), name
        assert np.array_equal(np.isinf(g), np.isinf(r)), name
        fin = np.isfinite(r)
        errs[name] = float(np.max(np.abs(g[fin] - r[fin]) / np.maximum(np.abs(r[fin]), 1e-300))) if fin.any() else 0.0
    return errs


def test_cfg5_full_size_parity_every_field():
    """BASELINE config 5 at its own shape (SURVEY.md 8(d) parity subset): 17-frame
    windows of two 1080x1920 fp32 approach streams -- video 0 (seed 1000, frames
    0..16, slow approach, TTC ~ 285) and video 4 (seed 1004, frames 22..38,
    which cross the segment cut at frame 31: the approach restarts with a new
    texture and T0) -- through run_sequence_batch(max_level=3), every
    estimate field against the oracle (ttc.py:248-279) on the rounded frames."""
    import paper_1612_08825_b200.synth as S
    v0, _ = S.approach_stream(17, 1080, 1920, seed=1000, dtype=torch.float32)
    v4, truth4 = S.approach_stream(39, 1080, 1920, seed=1004, dtype=torch.float32)
    assert np.isnan(truth4[31])  # the window really spans a cut
    vids = torch.stack([v0, v4[22:39]])
    got = ct.run_sequence_batch(vids, max_level=3).cpu().numpy()
    host = vids.cpu().numpy().astype(np.float64)
    errs = {}
    for v in range(2):
        ref = O.run_sequence(host[v], max_level=3)
        assert np.array_equal(got[v][:, 8], ref[:, 8]), ("selected level differs", v, got[v][:, 8], ref[:, 8])
        assert np.array_equal(got[v][:, 9], ref[:, 9]), "degenerate flag differs"
        for k, e in field_errors(got[v], ref).items():
            errs[k] = max(errs.get(k, 0.0), e)
        fin = np.isfinite(ref[:, 2]) & (ref[:, 9] == 0)
        for f, name in ((0, "a_over_c_px"), (1, "b_over_c_px"), (3, "x0_px"), (4, "y0_px")):
            d = np.abs(got[v][fin, f] - ref[fin, f])
            if f < 2:
                d = d / np.abs(ref[fin, 2])
            errs[name] = max(errs.get(name, 0.0), float(d.max()))
    print("cfg5 1080p fp32 max errors (relative; *_px absolute in pixels):", errs)
    bad = {k: e for k, e in errs.items() if e > CFG5_TOL.get(k, CFG5_FOE_PX if k.endswith("_px") else np.inf)}
    assert not bad, f"fields over tolerance {bad}; all errors {errs}"


def test_fp32_derivative_fields_parity():
    """north_star: fp32 derivative arrays within 1e-5 relative (inf-norm, SURVEY
    D5) of the reference on the fp32-rounded frames (ttc.py:82-99)."""
    f = O.generate(480, 270, 2, 80.0, (0.45, 0.55), 13, 0.0).astype(np.float32)
    a, b = torch.from_numpy(f[0]).cuda(), torch.from_numpy(f[1]).cuda()
    ex, ey, et = ct.derivatives_3d(FramePair(a, b))
    assert ex.dtype == torch.float32 and ex.is_cuda
    rex, rey, ret = O.derivatives(f[0].astype(np.float64), f[1].astype(np.float64))
    for got, ref in ((ex, rex), (ey, rey), (et, ret)):
        assert rel_inf(got.cpu().numpy(), ref) <= 1e-5
    g = ct.radial_gradient(ex, ey)
    assert rel_inf(g.cpu().numpy(), O.radial_gradient(rex, rey)) <= 1e-5
    # host float32 input is coerced to float64 like the reference (ttc.py:87): bit-exact
    hx, _, _ = ct.derivatives_3d(FramePair(torch.from_numpy(f[0]), torch.from_numpy(f[1])))
    assert hx.dtype == torch.float64 and np.array_equal(hx.numpy(), rex)


def test_trace_format(tmp_path):  # test_ttc.py:232-247 (ttc.py:308-332)
    from paper_1612_08825_b200 import TRACE_HEADER, trace_lines, write_trace
    ests = [
        ct.solve_ttc(NormalSystem(m=np.diag([2.0, 4.0, 8.0]), rhs=np.array([2.0, 4.0, 8.0]), et2=20.0, count=4)),
        ct.solve_ttc(NormalSystem(m=np.eye(3), rhs=np.array([0.5, 0.0, 0.0]), et2=1.0, count=4)),
        ct.solve_ttc(NormalSystem(m=np.zeros((3, 3)), rhs=np.zeros(3), et2=0.0, count=4)),
    ]
    lines = trace_lines(ests)
    assert lines[0] == TRACE_HEADER == "frame,ttc,foe_x,foe_y,residual,level,degenerate"
    assert lines[1].startswith("0,1,") and lines[1].endswith(",0,false")
    f2 = lines[2].split(",")
    assert f2[1] == "inf" and f2[2] == "nan" and f2[6] == "false"
    f3 = lines[3].split(",")
    assert f3[1] == "nan" and f3[6] == "true"
    p = tmp_path / "trace.csv"
    write_trace(ests, p)
    assert p.read_text().splitlines() == lines


def test_multiscale_accepts_any_max_level():
    # the reference walks until the extents drop below 4 (ttc.py:264-279);
    # max_level beyond the pyramid depth (or beyond 31) is not an error
    f = O.generate(64, 64, 3, 30.0, (0.5, 0.5), 6, 0.0)
    a = rows(ct.run_sequence(f, max_level=4))
    b = rows(ct.run_sequence(f, max_level=50))
    assert np.array_equal(a, b, equal_nan=True)
    assert ct.estimate_multiscale(FramePair(f[0], f[1]), max_level=1000).level == a[0, 8]


def test_synth_drop_in_helpers(tmp_path):
    # synth.generate -> SyntheticSequence, zoom_frame, score_mse (synth.py:61-208)
    cfg = ct.SynthConfig(width=64, height=48, frames=5, t0=40.0, foe=(0.4, 0.6), seed=3)
    seq = ct.generate(cfg)
    assert isinstance(seq, ct.SyntheticSequence) and seq.config == cfg
    assert np.array_equal(seq.frames, O.generate(64, 48, 5, 40.0, (0.4, 0.6), 3, 0.0))
    assert np.array_equal(seq.truth[:, 1], 40.0 - np.arange(5)) and seq.truth[0, 2] == 0.4 * 64
    tex = ct.make_texture(64, 48, 3)
    assert np.array_equal(ct.zoom_frame(tex, cfg.foe_px, 1.0), tex)
    assert np.array_equal(ct.zoom_frame(tex, cfg.foe_px, 1.25), O.zoom_frame(tex, cfg.foe_px, 1.25))
    with pytest.raises(ValueError):
        ct.zoom_frame(tex, cfg.foe_px, 0.9)
    ct.write_trace(ct.run_sequence(seq.frames), tmp_path / "pred.csv")
    (tmp_path / "truth.csv").write_text("frame,ttc,foe_x,foe_y\n" + "".join(
        f"{int(r[0])},{float(r[1])!r},{float(r[2])!r},{float(r[3])!r}\n" for r in seq.truth))
    rep = ct.score_mse(tmp_path / "pred.csv", tmp_path / "truth.csv")
    assert rep.compared + rep.excluded == 4 and rep.mse >= 0


def test_host_paths_pageable_and_pinned_match_device():
    """run_sequence_host streams pinned frames directly and pageable frames
    through its pinned staging ring in 8 MB chunks (one-frame halo between
    chunks); both equal the device-resident run bit for bit, multiscale too."""
    g = torch.Generator(device="cuda").manual_seed(5)
    dev = torch.rand((2, 100, 256, 256), dtype=torch.float64, device="cuda", generator=g)  # 50 MB per video
    for kw in ({"level": 0}, {"max_level": 2}):
        ref = ct.run_sequence_batch(dev, **kw).cpu().numpy()
        pageable = dev.cpu().numpy()
        pinned = dev.cpu().pin_memory()
        assert np.array_equal(ct.run_sequence_host(pageable, **kw), ref, equal_nan=True)
        assert np.array_equal(ct.run_sequence_host(pinned, **kw), ref, equal_nan=True)
    f32 = dev[0].float().cpu().numpy()  # the reference-style call on a float32 array: coerced to float64
    est = ct.run_sequence(f32, level=0)
    want = ct.run_sequence_batch(torch.from_numpy(f32.astype(np.float64)).cuda()[None], level=0)[0].cpu().numpy()
    assert np.array_equal(rows(est)[:, :8], want[:, :8], equal_nan=True)


def test_nonfinite_inputs_match_the_reference(golden):
    """NaN / Inf pixels propagate exactly as in the reference (fixtures produced by
    the reference itself): single-scale, level 1 and multiscale rows, and
    convolution outputs, NaN positions and values identical."""
    z = golden("nonfinite_fixtures.npz")
    for key, kw in (("l0", dict(level=0)), ("l1", dict(level=1)), ("ms2", dict(max_level=2))):
        got = np.array([[np.nan] * 8 + [-1.0, np.nan] if e is None else [float(getattr(e, f)) for f in EST]
                        for e in ct.run_sequence(z["frames"], **kw)])
        assert np.array_equal(got, z[key], equal_nan=True), key
    assert np.array_equal(ct.conv_direct(z["conv_s"], z["conv_k"]), z["conv_full"], equal_nan=True)
    assert np.array_equal(ct.xcorr_direct(z["conv_s"], z["conv_k"], ct.ConvShape.SAME, ct.BoundaryPolicy.REPLICATE),
                          z["xcorr_same_rep"], equal_nan=True)


def test_host_path_concurrent_callers():
    """Two host threads streaming pageable videos at once (the copy pool and the
    pinned rings are shared / per thread): each gets its own video's rows."""
    from concurrent.futures import ThreadPoolExecutor
    g = torch.Generator(device="cuda").manual_seed(9)
    dev = torch.rand((4, 40, 256, 256), dtype=torch.float64, device="cuda", generator=g)
    ref = ct.run_sequence_batch(dev, level=0).cpu().numpy()
    vids = [dev[v:v + 1].cpu().numpy() for v in range(4)]

    def work(v):
        return ct.run_sequence_host(vids[v], level=0)

    with ThreadPoolExecutor(2) as ex:
        outs = list(ex.map(work, [0, 1, 2, 3, 0, 1, 2, 3]))
    for k, o in enumerate(outs):
        assert np.array_equal(o[0], ref[k % 4], equal_nan=True), k


def test_4k_frames_multiscale_every_field():
    """Larger than config 5: 2160 x 3840 fp32 frames (16 column tiles, five
    pyramid levels), two pairs against the oracle on the rounded frames; the
    same field tolerances as the 1080p config-5 test."""
    import paper_1612_08825_b200.synth as S
    fr, _ = S.approach_stream(3, 2160, 3840, seed=77, dtype=torch.float32)
    got = ct.run_sequence_batch(fr[None], max_level=4).cpu().numpy()[0]
    ref = O.run_sequence(fr.cpu().numpy().astype(np.float64), max_level=4)
    assert np.array_equal(got[:, 8], ref[:, 8]) and np.array_equal(got[:, 9], ref[:, 9])
    errs = field_errors(got, ref)
    assert errs["c"] <= CFG5_TOL["c"] and errs["ttc"] <= CFG5_TOL["ttc"], errs
    assert errs["residual"] <= CFG5_TOL["residual"] and errs["misfit"] <= CFG5_TOL["misfit"], errs
    fin = np.isfinite(ref[:, 2]) & (ref[:, 9] == 0)
    assert np.all(np.abs(got[fin, 3] - ref[fin, 3]) <= CFG5_FOE_PX * 2 ** ref[fin, 8])
    assert np.all(np.abs(got[fin, 4] - ref[fin, 4]) <= CFG5_FOE_PX * 2 ** ref[fin, 8])


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_multiscale_group_schedules_are_bit_identical(dtype, monkeypatch):
    """The multiscale pipeline's video groups (CT_MS_PARTS) and the way they are
    scheduled (CT_MS_SCHED: alternating equal-priority streams, or level-0
    passes on a low-priority stream with the tails on a high-priority one) only
    change which launches run side by side: every video's rows are the same
    bits as with one group."""
    vids = np.stack([O.generate(200, 152, 6, 50.0 + 30.0 * v, (0.5, 0.5), 70 + v, 0.002) for v in range(5)])
    dev = torch.from_numpy(vids).to(dtype).cuda()
    monkeypatch.setenv("CT_MS_PARTS", "1")
    monkeypatch.delenv("CT_MS_SCHED", raising=False)
    ref = ct.run_sequence_batch(dev, max_level=3).cpu().numpy()
    for parts, sched in (("2", "0"), ("3", "1"), ("5", "1"), ("4", "0")):
        monkeypatch.setenv("CT_MS_PARTS", parts)
        monkeypatch.setenv("CT_MS_SCHED", sched)
        for _ in range(2):  # twice: the second call reuses the streams and events
            got = ct.run_sequence_batch(dev, max_level=3).cpu().numpy()
            assert np.array_equal(got, ref, equal_nan=True), (parts, sched)
