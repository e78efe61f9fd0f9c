"""ctypes binding of libconvtact_b200.so (the C ABI in include/convtact_b200.h).

The library is the only compute path: there is no CPU fallback.  Importing
this module never touches the GPU; the first call loads the library and
raises RuntimeError if it is missing or no CUDA device is visible.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

# CT_LIB_PATH points at an alternative build (A/B tuning runs only)
LIB_PATH = os.environ.get("CT_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libconvtact_b200.so")

CT_OK, CT_EINVAL, CT_ECUDA, CT_EUNSUPPORTED = 0, 1, 2, 3
CT_F64, CT_F32 = 0, 1
CT_FULL, CT_SAME, CT_VALID = 0, 1, 2
CT_ZERO, CT_REPLICATE = 0, 1
CT_NSUMS = 11
CT_NEST = 10

# Every symbol include/convtact_b200.h declares (tests check the exports).
EXPORTS = (
    "ct_last_error", "ct_version", "ct_xcorr_nd", "ct_direct", "ct_ttc_derivatives",
    "ct_radial_gradient", "ct_normal_system_workspace_bytes", "ct_normal_system",
    "ct_ttc_moments_workspace_bytes", "ct_ttc_moments", "ct_ttc_solve", "ct_pyramid_down",
    "ct_ttc_multiscale_select", "ct_run_sequence_workspace_bytes", "ct_run_sequence",
    "ct_run_sequence_host_workspace_bytes", "ct_run_sequence_host", "ct_zoom_frames",
    "ct_zoom_frames_workspace_bytes", "ct_gradient", "ct_decode_samples",
    "ct_ttc_pyramid_moments_workspace_bytes", "ct_ttc_pyramid_moments",
)

_lib = None


def load(require_gpu: bool = True):
    """Load the shared library (and by default insist on a CUDA device)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P, I, I64, D, SZ = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_size_t
        L.ct_last_error.restype = ctypes.c_char_p
        L.ct_version.restype = ctypes.c_char_p
        L.ct_xcorr_nd.argtypes = [I, I, P, P, I64, P, P, P, P, P, I, P, P]
        L.ct_direct.argtypes = [I, I, P, P, I64, P, P, P, I, I, I, P, P]
        L.ct_ttc_derivatives.argtypes = [I, P, P, I64, I64, P, P, P, P]
        L.ct_radial_gradient.argtypes = [I, P, P, I64, I64, P, P]
        L.ct_normal_system_workspace_bytes.argtypes = [I64, I64]
        L.ct_normal_system_workspace_bytes.restype = SZ
        L.ct_normal_system.argtypes = [I, P, P, P, P, I64, I64, I64, P, P, SZ, P]
        L.ct_ttc_moments_workspace_bytes.argtypes = [I, I64, I64, I64, I64]
        L.ct_ttc_moments_workspace_bytes.restype = SZ
        L.ct_ttc_moments.argtypes = [I, P, I64, I64, I64, I64, P, P, SZ, P]
        L.ct_ttc_solve.argtypes = [P, I64, D, I, P, P]
        L.ct_pyramid_down.argtypes = [I, P, I64, I64, I64, P, P]
        L.ct_ttc_multiscale_select.argtypes = [P, I64, I, P, P]
        L.ct_run_sequence_workspace_bytes.argtypes = [I, I64, I64, I64, I64, I, I]
        L.ct_run_sequence_workspace_bytes.restype = SZ
        L.ct_run_sequence.argtypes = [I, P, I64, I64, I64, I64, I, I, D, P, P, SZ, P]
        L.ct_run_sequence_host_workspace_bytes.argtypes = [I, I64, I64, I64, I64, I, I]
        L.ct_run_sequence_host_workspace_bytes.restype = SZ
        L.ct_run_sequence_host.argtypes = [I, P, I64, I64, I64, I64, I, I, D, P, P, SZ, P]
        L.ct_zoom_frames.argtypes = [I, P, I64, I64, D, D, P, I64, P, P, SZ, P]
        L.ct_zoom_frames_workspace_bytes.argtypes = [I64, I64]
        L.ct_zoom_frames_workspace_bytes.restype = SZ
        L.ct_gradient.argtypes = [I, P, I64, I64, I64, P, P, I64, I64, P, P, P, P, P]
        L.ct_decode_samples.argtypes = [I, P, I64, D, P, P]
        L.ct_ttc_pyramid_moments_workspace_bytes.argtypes = [I, I64, I64, I64, I64, I]
        L.ct_ttc_pyramid_moments_workspace_bytes.restype = SZ
        L.ct_ttc_pyramid_moments.argtypes = [I, P, I64, I64, I64, I64, I, P, P, SZ, P]
        _lib = L
    if require_gpu and not torch.cuda.is_available():
        raise RuntimeError("convtact_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    return _lib


def check(rc: int) -> None:
    if rc == CT_OK:
        return
    msg = load(require_gpu=False).ct_last_error().decode(errors="replace")
    if rc == CT_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"convtact_b200 error {rc}: {msg}")


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor):
    return ctypes.c_void_p(t.data_ptr())


def i64_array(vals) -> ctypes.Array:
    vals = [int(v) for v in vals]
    return (ctypes.c_int64 * max(len(vals), 1))(*vals)


def dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float64:
        return CT_F64
    if t.dtype == torch.float32:
        return CT_F32
    raise TypeError(f"unsupported dtype {t.dtype}")


def workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


def to_device(x, keep_f32: bool = True) -> tuple[torch.Tensor, bool]:
    """Coerce an array-like to a contiguous CUDA tensor.

    Returns (tensor, was_numpy).  numpy / lists are coerced to float64 as the
    reference does (conv.py:101-102, ttc.py:293), and so are host (CPU) torch
    tensors; only CUDA tensors keep float32 (the fp32 path) -- other dtypes
    become float64.
    """
    if isinstance(x, torch.Tensor):
        t = x
        if not t.is_cuda:  # host tensors are coerced like numpy input (float64)
            return t.to(device="cuda", dtype=torch.float64).contiguous(), True
        if t.dtype not in (torch.float32, torch.float64) or (t.dtype == torch.float32 and not keep_f32):
            t = t.to(torch.float64)
        return t.contiguous(), False
    a = np.ascontiguousarray(x, dtype=np.float64)
    return torch.from_numpy(a).to("cuda", non_blocking=False), True


def version() -> str:
    return load(require_gpu=False).ct_version().decode()
