"""Pin the CPU oracle against fixtures produced by the reference itself
(tests/golden/make_golden.py).  CPU only; these prove the checker before it
is used to check the GPU path."""

import hashlib

import numpy as np
import pytest

import oracle as O

SHAPES = ("full", "same", "valid")
BOUNDS = ("zero", "replicate")


def test_conv_cases_bit_exact(golden):
    z = golden("conv_cases.npz")
    n = int(z["count"])
    assert n > 500
    for i in range(n):
        sh, bd, fl = (int(v) for v in z[f"c{i}_meta"])
        got = O.direct(z[f"c{i}_s"], z[f"c{i}_k"], SHAPES[sh], BOUNDS[bd], bool(fl))
        assert np.array_equal(got, z[f"c{i}_out"]), f"case {i}"


def test_cfg1_full_output_bit_exact(golden):
    c = golden("conv_configs.npz")
    s = np.random.Generator(np.random.PCG64(0)).random((256, 256))
    k = np.random.Generator(np.random.PCG64(1)).standard_normal((5, 5))
    got = O.direct(s, k, "full")
    assert np.array_equal(got, c["cfg1_out"])
    # SURVEY.md 8(c) anchors
    assert got[0, 0] == 0.22012389008920766
    assert abs(got.sum() - 2356.9480520543348) < 1e-9


def test_cfg3_samples_bit_exact(golden):
    c = golden("conv_configs.npz")
    s = np.random.Generator(np.random.PCG64(0)).random((128,) * 3).astype(np.float32).astype(np.float64)
    k = np.random.Generator(np.random.PCG64(1)).standard_normal((7,) * 3).astype(np.float32).astype(np.float64)
    got = O.direct(s, k, "full")
    assert got.shape == (134,) * 3
    assert np.array_equal(got.ravel()[c["cfg3_idx"]], c["cfg3_val"])
    assert got.sum() == pytest.approx(float(c["cfg3_sum"]), rel=1e-12)


def test_ttc_fields_and_solve_bit_exact(golden):
    t = golden("ttc_fixtures.npz")
    a, b = t["small_a"], t["small_b"]
    ex, ey, et = O.derivatives(a, b)
    assert np.array_equal(ex, t["small_ex"]) and np.array_equal(ey, t["small_ey"]) and np.array_equal(et, t["small_et"])
    g = O.radial_gradient(ex, ey)
    assert np.array_equal(g, t["small_g"])
    s1 = O.normal_system(ex, ey, g, et, 1)
    assert np.array_equal(s1, t["small_sums_b1"])
    assert np.array_equal(O.normal_system(ex, ey, g, et, 3), t["small_sums_b3"])
    assert np.array_equal(O.solve_ttc(s1), t["small_est"], equal_nan=True)
    assert np.array_equal(O.downsample(a), t["small_down"])
    assert np.array_equal(O.downsample(O.downsample(a)), t["small_down2"])


def test_generator_bit_exact(golden):
    t = golden("ttc_fixtures.npz")
    f = O.generate(256, 256, 64, 100.0, (0.5, 0.5), 0, 0.0)
    assert hashlib.sha256(f.tobytes()).hexdigest() == str(t["cfg2_frames_sha"])
    assert np.array_equal(f[0, 0], t["cfg2_frame0_row0"])
    fn = O.generate(128, 128, 12, 60.0, (0.5, 0.5), 2, 0.05)
    assert hashlib.sha256(fn.tobytes()).hexdigest() == str(t["noisy_frames_sha"])


@pytest.mark.parametrize("key,kw,nfr", [("cfg2_l0", dict(level=0), 64), ("cfg2_l1", dict(level=1), 9),
                                        ("cfg2_l2", dict(level=2), 9), ("cfg2_ms5", dict(max_level=5), 9)])
def test_cfg2_estimates_bit_exact(golden, key, kw, nfr):
    t = golden("ttc_fixtures.npz")
    f = O.generate(256, 256, 64, 100.0, (0.5, 0.5), 0, 0.0)
    got = O.run_sequence(f[:nfr], **kw)
    assert np.array_equal(got, t[key], equal_nan=True)


def test_published_anchor_seed1_pair0(golden):
    # pkg/test_output.txt:136, printed on the reference's development host for
    # SynthConfig(seed=1) pair 0: a=0.2662447623728236, b=-0.14063136884859345,
    # c=0.010388552681548783, x0=-25.628667489524663.  a and b reproduce
    # exactly; c and x0 differ in the last ulp (numba/BLAS FMA choices differ
    # across hosts).
    t = golden("ttc_fixtures.npz")
    f = O.generate(256, 256, 60, 100.0, (0.4, 0.55), 1, 0.0)
    got = O.run_sequence(f[:2], level=0)[0]
    assert got[0] == 0.2662447623728236
    assert got[1] == -0.14063136884859345
    assert abs(got[2] - 0.010388552681548783) <= 2e-18
    assert abs(got[3] - -25.628667489524663) <= 1e-13
    assert np.array_equal(O.run_sequence(f, level=0), t["def1_l0"], equal_nan=True)


def test_noisy_multiscale_bit_exact(golden):
    t = golden("ttc_fixtures.npz")
    fn = O.generate(128, 128, 12, 60.0, (0.5, 0.5), 2, 0.05)
    assert np.array_equal(O.run_sequence(fn, max_level=5), t["noisy_ms5"], equal_nan=True)
    assert np.array_equal(O.run_sequence(fn, level=0), t["noisy_l0"], equal_nan=True)


def test_fp32_rounded_multiscale_bit_exact(golden):
    t = golden("ttc_fixtures.npz")
    f5 = O.generate(480, 270, 4, 300.0, (0.5, 0.5), 11, 0.0).astype(np.float32)
    assert hashlib.sha256(f5.tobytes()).hexdigest() == str(t["c5_frames32_sha"])
    assert np.array_equal(O.run_sequence(f5.astype(np.float64), max_level=3), t["c5_ms3"], equal_nan=True)


def test_oracle_thread_count_invariance():
    f = O.generate(64, 64, 9, 40.0, (0.5, 0.5), 3, 0.0)
    assert np.array_equal(O.run_sequence(f, level=0, nthreads=1), O.run_sequence(f, level=0, nthreads=4))


def test_gradient_fixtures_restated(golden):
    # kernels.gradient (kernels.py:63-72) = SAME/REPLICATE xcorr + hypot/atan2
    g = golden("gradient_fixtures.npz")
    img = g["img"]
    pairs = {"roberts": ([[1.0, 0.0], [0.0, -1.0]], [[0.0, 1.0], [-1.0, 0.0]]),
             "prewitt2": ([[-0.5, 0.5], [-0.5, 0.5]], [[-0.5, -0.5], [0.5, 0.5]]),
             "prewitt3": ([[-1.0, 0.0, 1.0]] * 3, [[-1.0] * 3, [0.0] * 3, [1.0] * 3]),
             "sobel": ([[-1.0, 0.0, 1.0], [-2.0, 0.0, 2.0], [-1.0, 0.0, 1.0]],
                       [[-1.0, -2.0, -1.0], [0.0, 0.0, 0.0], [1.0, 2.0, 1.0]])}
    for name, (kx, ky) in pairs.items():
        ex = O.direct(img, np.array(kx), "same", "replicate", flip=False)
        ey = O.direct(img, np.array(ky), "same", "replicate", flip=False)
        assert np.array_equal(ex, g[f"{name}_ex"]) and np.array_equal(ey, g[f"{name}_ey"]), name
        assert np.array_equal(np.hypot(ex, ey), g[f"{name}_mag"]), name
        assert np.array_equal(np.arctan2(ey, ex), g[f"{name}_dir"]), name


def test_nonfinite_fixtures_restated(golden):
    """NaN / Inf inputs: the oracle reproduces the reference's IEEE propagation
    field for field (fixtures from the reference itself, make_golden.py nonfinite)."""
    z = golden("nonfinite_fixtures.npz")
    for key, kw in (("l0", dict(level=0)), ("l1", dict(level=1)), ("ms2", dict(max_level=2))):
        assert np.array_equal(O.run_sequence(z["frames"], **kw), z[key], equal_nan=True), key
    assert np.array_equal(O.direct(z["conv_s"], z["conv_k"], "full"), z["conv_full"], equal_nan=True)
    assert np.array_equal(O.direct(z["conv_s"], z["conv_k"], "same", "replicate", flip=False), z["xcorr_same_rep"],
                          equal_nan=True)
