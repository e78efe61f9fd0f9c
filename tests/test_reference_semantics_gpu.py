"""The reference's own behavioural tests and end-to-end acceptance numbers,
restated against this package's GPU path (test_ttc.py:22-222 and
test_acceptance.py:148-320 semantics; the golden end-to-end figures are the
ones the reference printed in pkg/test_output.txt:208-214, reproduced here to
the printed digits because the device pipeline matches the reference to
<= 1e-9 per estimate)."""

import numpy as np
import pytest
import torch

import paper_1612_08825_b200 as ct
from paper_1612_08825_b200 import FramePair, SynthConfig

pytestmark = pytest.mark.gpu

T0 = 100.0
SIZE = 256
SEEDS = (1, 2, 3)


# ------------------------------------------------------------ TTC semantics ---

def test_stencils_on_a_linear_brightness_field():  # test_ttc.py:22-40
    e = np.array([[0.0, 1.0], [2.0, 3.0]])
    ex, ey, et = ct.derivatives_3d(FramePair(e, e + 4.0))
    assert ex.shape == (1, 1) and (ex[0, 0], ey[0, 0], et[0, 0]) == (1.0, 2.0, 4.0)
    yy, xx = np.mgrid[0:8, 0:9].astype(np.float64)
    base = 2 * xx + 3 * yy
    ex, ey, et = ct.derivatives_3d(FramePair(base, base + 5.0))
    assert np.allclose(ex, 2.0, atol=1e-12) and np.allclose(ey, 3.0, atol=1e-12) and np.allclose(et, 5.0, atol=1e-12)


def test_gradient_ramps_are_centred():  # test_ttc.py:50-56
    g = ct.radial_gradient(np.ones((5, 7)), np.zeros((5, 7)))
    assert np.array_equal(g, np.broadcast_to(np.arange(7) - 3.0, (5, 7)))
    g = ct.radial_gradient(np.zeros((5, 7)), np.ones((5, 7)))
    assert np.array_equal(g, np.broadcast_to((np.arange(5) - 2.0)[:, None], (5, 7)))


def test_normal_system_symmetric_psd_and_border_errors():  # test_ttc.py:59-77
    rng = np.random.default_rng(0)
    f = [rng.standard_normal((12, 15)) for _ in range(4)]
    ns = ct.build_normal_system(*f, border=2)
    assert np.array_equal(ns.m, ns.m.T) and np.all(np.linalg.eigvalsh(ns.m) >= -1e-9)
    assert ns.count == (12 - 4) * (15 - 4)
    with pytest.raises(ValueError):
        ct.build_normal_system(*f, border=0)
    with pytest.raises(ValueError):
        ct.build_normal_system(*f, border=6)


def test_pure_translation_has_no_expansion():  # test_ttc.py:132-139
    tex = ct.make_texture(64, 64, 9)
    est = ct.estimate_fixed(FramePair(tex, np.roll(tex, 1, axis=1)), level=0)
    assert not est.degenerate
    assert abs(est.a - 1.0) <= 0.05 and abs(est.b) < 0.05 and abs(est.c) < 1e-3 * abs(est.a)


def test_downsample_constants_and_coordinates():  # test_ttc.py:142-157
    out = ct.downsample(np.full((10, 13), 0.25))
    assert out.shape == (5, 6) and np.allclose(out, 0.25, atol=1e-14)
    with pytest.raises(ValueError):
        ct.downsample(np.ones((1, 8)))
    x = np.mgrid[0:16, 0:16][1].astype(np.float64)
    ramp = ct.downsample(x)  # level-1 sample j sits at level-0 coordinate 2j + 0.5
    assert np.allclose(ramp[2:-2, 2:-2], (2.0 * np.arange(8) + 0.5)[None, 2:-2], atol=1e-12)


def test_known_zoom_and_foe_level_scaling():  # test_ttc.py:160-180
    seq = ct.generate(SynthConfig(width=128, height=128, frames=2, t0=50.0, foe=(0.5, 0.5), seed=4))
    est = ct.estimate_fixed(FramePair(seq.frames[0], seq.frames[1]), level=0)
    assert not est.degenerate and abs(est.ttc - 50.0) <= 5.0 and abs(est.x0) < 3.0 and abs(est.y0) < 3.0
    seq = ct.generate(SynthConfig(width=256, height=256, frames=2, t0=40.0, foe=(0.375, 0.625), seed=5))
    est = ct.estimate_fixed(FramePair(seq.frames[0], seq.frames[1]), level=2)
    assert est.level == 2  # FOE comes back in level-0 pixels: array pixel (96, 160)
    assert np.hypot(est.x0 + 127.5 - 96.0, est.y0 + 127.5 - 160.0) < 8.0


def test_multiscale_picks_minimum_misfit_and_helps_under_noise():  # test_ttc.py:200-222
    seq = ct.generate(SynthConfig(width=256, height=256, frames=2, t0=100.0, foe=(0.4, 0.55), seed=1))
    pair = FramePair(seq.frames[0], seq.frames[1])
    ms = ct.estimate_multiscale(pair, max_level=5)
    assert all(ms.misfit <= ct.estimate_fixed(pair, level=lv).misfit + 1e-15 for lv in range(ms.level + 1))
    cfg = SynthConfig(width=128, height=128, frames=12, t0=60.0, foe=(0.5, 0.5), seed=2, noise_sigma=0.05)
    frames = ct.generate(cfg).frames
    truth = cfg.t0 - np.arange(11)

    def mse(ests):
        v = np.array([e.ttc for e in ests])
        ok = np.isfinite(v)
        return np.mean((v[ok] - truth[ok]) ** 2)

    assert mse(ct.run_sequence(frames, max_level=5)) < mse(ct.run_sequence(frames, level=0))


# ------------------------------------------------------ acceptance criteria ---

@pytest.fixture(scope="module")
def clean():
    suite = {s: ct.generate(SynthConfig(seed=s)) for s in SEEDS}
    return suite, {s: ct.run_sequence(seq.frames, level=0) for s, seq in suite.items()}


def _worst(values):
    """(worst value, (seed, frame)) over {seed: [(frame, value)]}, first maximum in seed/frame order."""
    best, where = -1.0, None
    for s in SEEDS:
        for t, v in values[s]:
            if v > best:
                best, where = v, (s, t)
    return best, where


def test_criterion_06_ttc_recovery_golden(clean):
    _, l0 = clean
    rel = {s: [(t, abs(e.ttc - (T0 - t)) / (T0 - t)) for t, e in enumerate(l0[s]) if T0 - t >= 20] for s in SEEDS}
    worst, where = _worst(rel)
    # the reference prints "worst rel err 11.72% at seed 2 frame 58" (it misses its own 10 % bar)
    assert f"{worst * 100:.2f}" == "11.72" and where == (2, 58)


def test_criterion_07_foe_recovery_golden(clean):
    suite, l0 = clean
    err = {}
    for s in SEEDS:
        fx, fy = suite[s].config.foe_px
        err[s] = [(t, float(np.hypot(e.x0 + (SIZE - 1) / 2 - fx, e.y0 + (SIZE - 1) / 2 - fy)))
                  for t, e in enumerate(l0[s]) if T0 - t >= 20]
    worst, where = _worst(err)
    assert f"{worst:.2f}" == "1.19" and where == (3, 1) and worst <= 0.05 * SIZE


def test_criterion_08_multiscale_benefit_golden():
    noisy = {s: ct.generate(SynthConfig(seed=s, noise_sigma=0.05)).frames for s in SEEDS}
    sq = {lv: [] for lv in (0, 2, 4, 5)}
    sq_ms = []
    for s in SEEDS:
        for lv in sq:
            sq[lv] += [(e.ttc - (T0 - t)) ** 2 for t, e in enumerate(ct.run_sequence(noisy[s], level=lv))
                       if np.isfinite(e.ttc)]
        sq_ms += [(e.ttc - (T0 - t)) ** 2 for t, e in enumerate(ct.run_sequence(noisy[s], max_level=5))
                  if np.isfinite(e.ttc)]
    mse = {lv: float(np.mean(v)) for lv, v in sq.items()}
    mse_ms = float(np.mean(sq_ms))
    printed = [f"{mse_ms:.2f}"] + [f"{mse[lv]:.2f}" for lv in (0, 2, 4, 5)]
    assert printed == ["8.39", "1504.42", "31.33", "230830.48", "160647.91"], printed
    assert mse_ms <= 1.1 * min(mse.values()) and mse_ms < mse[0]


def test_criterion_09_scale_invariance_golden(clean):
    suite, l0 = clean
    rel = {}
    for s in SEEDS:
        l1 = ct.run_sequence(suite[s].frames, level=1)
        rel[s] = [(t, abs(e1.ttc - e0.ttc) / e0.ttc) for t, (e0, e1) in enumerate(zip(l0[s], l1)) if T0 - t >= 20]
    worst, where = _worst(rel)
    assert f"{worst * 100:.2f}" == "10.78" and where == (2, 18)


def test_criterion_12_determinism(clean, tmp_path):
    suite, _ = clean
    again = ct.generate(SynthConfig(seed=1))
    assert np.array_equal(again.frames, suite[1].frames) and np.array_equal(again.truth, suite[1].truth)
    cfg = SynthConfig(seed=2, noise_sigma=0.05)
    assert np.array_equal(ct.generate(cfg).frames, ct.generate(cfg).frames)
    ct.write_sequence(again, tmp_path / "d1")
    ct.write_sequence(again, tmp_path / "d2")
    for name in ("truth.csv", "frame_000000.pgm", "frame_000059.pgm"):
        assert (tmp_path / "d1" / name).read_bytes() == (tmp_path / "d2" / name).read_bytes()
    ct.write_trace(ct.run_sequence(again.frames[:10], level=0), tmp_path / "a.csv")
    ct.write_trace(ct.run_sequence(torch.from_numpy(again.frames[:10]).cuda(), level=0), tmp_path / "b.csv")
    assert (tmp_path / "a.csv").read_bytes() == (tmp_path / "b.csv").read_bytes()
