"""GPU parity of the fused gradient-field kernel (kernels.py:63-72; SURVEY.md
8(f) row 3) against the reference fixtures: ex/ey bit-identical (same FMA tap
order as the conv engine), mag/dir within 4 ulp-scale relative error (CUDA's
hypot/atan2 vs the host libm)."""

import numpy as np
import pytest
import torch

import paper_1612_08825_b200 as ct

pytestmark = pytest.mark.gpu

RAMP_SCALE = {"roberts": np.sqrt(2.0), "prewitt2": 1.0, "prewitt3": 6.0, "sobel": 8.0}


def test_fixtures(golden):
    g = golden("gradient_fixtures.npz")
    img = g["img"]
    for name in ct.KERNELS:
        f = ct.gradient(img, name)
        assert np.array_equal(f.ex, g[f"{name}_ex"]) and np.array_equal(f.ey, g[f"{name}_ey"]), name
        ref_mag, ref_dir = g[f"{name}_mag"], g[f"{name}_dir"]
        assert np.max(np.abs(f.mag - ref_mag) / np.maximum(np.abs(ref_mag), 1e-300)) <= 1e-15, name
        assert np.max(np.abs(f.dir - ref_dir)) <= 4e-16 * np.pi * 4, name


def test_reference_identities():  # test_kernels.py / criterion 11 (test_acceptance.py:245-278)
    y, x = np.mgrid[0:12, 0:14].astype(np.float64)
    ramp = 3.0 * x + 4.0 * y
    rng = np.random.default_rng(77)
    for name, scale in RAMP_SCALE.items():
        f = ct.gradient(ramp, name)
        assert np.allclose(f.mag[2:-2, 2:-2] / scale, 5.0, atol=1e-12), name
        c = ct.gradient(np.full((9, 11), 0.7), name)
        assert np.allclose(c.mag, 0.0, atol=1e-14)
        z = ct.gradient(np.zeros((6, 6)), name)
        assert np.all(z.dir == 0.0)
        img = rng.random((20, 20))
        fi, ft = ct.gradient(img, name), ct.gradient(img.T, name)
        assert np.all((fi.dir >= -np.pi) & (fi.dir <= np.pi))
        if name == "roberts":
            assert np.allclose(ft.ex, fi.ex.T, atol=1e-12) and np.allclose(ft.ey, -fi.ey.T, atol=1e-12)
        else:
            assert np.allclose(ft.ex, fi.ey.T, atol=1e-12) and np.allclose(ft.ey, fi.ex.T, atol=1e-12)
    with pytest.raises(KeyError):
        ct.kernel_lookup("scharr")
    with pytest.raises(ValueError):
        ct.gradient(np.ones(5), "sobel")


def test_device_tensor_and_fp32():
    img = torch.rand((64, 80), dtype=torch.float32, device="cuda")
    f = ct.gradient(img, "sobel")
    assert f.ex.is_cuda and f.ex.dtype == torch.float32
    ref = ct.gradient(img.double().cpu().numpy(), "sobel")
    assert np.max(np.abs(f.mag.cpu().numpy() - ref.mag)) <= 1e-5 * np.max(ref.mag)
