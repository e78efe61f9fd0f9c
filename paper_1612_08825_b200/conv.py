"""n-D direct convolution / cross-correlation on the B200 (drop-in for convtact.conv).

Same names, signatures, shape law and boundary semantics as the reference
(/root/reference/pkg/src/convtact/conv.py):

  FULL   m + n - 1
  SAME   m, anchored so SAME(i) = FULL(i + floor((n - 1) / 2))
  VALID  m - n + 1, requires m >= n everywhere

conv(s, k) == xcorr(s, reflect(k)).  REPLICATE only matters for SAME.

Inputs: numpy arrays / array-likes are coerced to C-contiguous float64 (as
the reference does, conv.py:101-102) and results come back as numpy;
CUDA tensors stay on the device (float32 tensors take the fp32 path).  The
arithmetic runs in libconvtact_b200.so (ct_direct); there is no CPU path.
"""

from __future__ import annotations

import ctypes
from collections import OrderedDict
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _lib

DEFAULT_AUTO_THRESHOLD = 900


class ConvShape(Enum):
    FULL = "full"
    SAME = "same"
    VALID = "valid"


class ConvMethod(Enum):
    DIRECT = "direct"
    FFT = "fft"
    AUTO = "auto"


class BoundaryPolicy(Enum):
    ZERO = "zero"
    REPLICATE = "replicate"


@dataclass(frozen=True)
class ConvPlan:
    """Resolved operation parameters (conv.py:52-59)."""

    method: ConvMethod = ConvMethod.AUTO
    shape: ConvShape = ConvShape.FULL
    boundary: BoundaryPolicy = BoundaryPolicy.ZERO
    threshold: int = DEFAULT_AUTO_THRESHOLD


_SHAPE = {ConvShape.FULL: _lib.CT_FULL, ConvShape.SAME: _lib.CT_SAME, ConvShape.VALID: _lib.CT_VALID}
_BOUND = {BoundaryPolicy.ZERO: _lib.CT_ZERO, BoundaryPolicy.REPLICATE: _lib.CT_REPLICATE}


def reflect(k):
    """Reverse every axis (point reflection through the kernel center), conv.py:62-64."""
    if isinstance(k, torch.Tensor):
        return torch.flip(k, dims=tuple(range(k.ndim)))
    k = np.asarray(k)
    return k[(slice(None, None, -1),) * k.ndim]


def out_shape(sshape, kshape, shape: ConvShape):
    if shape == ConvShape.FULL:
        return tuple(m + n - 1 for m, n in zip(sshape, kshape))
    if shape == ConvShape.SAME:
        return tuple(sshape)
    return tuple(m - n + 1 for m, n in zip(sshape, kshape))


def _check_pair(sndim: int, kndim: int) -> None:  # conv.py:86-90
    if sndim != kndim:
        raise ValueError(f"rank mismatch: signal ndim {sndim}, kernel ndim {kndim}")
    if sndim < 1:
        raise ValueError("zero-rank tensors not supported")


def _check_valid(sshape, kshape) -> None:  # conv.py:93-98
    for ax, (m, n) in enumerate(zip(sshape, kshape)):
        if m < n:
            raise ValueError(f"VALID needs signal >= kernel on every axis, axis {ax} has {m} < {n}")


def _host_kernel(kernel, dtype: torch.dtype) -> np.ndarray:
    if isinstance(kernel, torch.Tensor):
        kernel = kernel.detach().cpu().numpy()
    return np.ascontiguousarray(kernel, dtype=np.float64 if dtype == torch.float64 else np.float32)


_KD_CACHE: "OrderedDict[tuple, torch.Tensor]" = OrderedDict()


def _device_kernel(k: np.ndarray, device: torch.device) -> torch.Tensor:
    """Device copy of the taps (only the generic rank >= 4 kernel reads them;
    the tiled kernels take the host copy through the parameter bank).  Cached
    by content so repeated calls do no host->device copy (and can be captured
    into a CUDA graph after a warm-up call)."""
    key = (k.dtype.str, k.shape, k.tobytes(), device.index)
    kd = _KD_CACHE.get(key)
    if kd is None:
        kd = torch.from_numpy(k).to(device)
        _KD_CACHE[key] = kd
        if len(_KD_CACHE) > 64:
            _KD_CACHE.popitem(last=False)
    else:
        _KD_CACHE.move_to_end(key)
    return kd


def direct_batch(signals, kernel, shape=ConvShape.FULL, boundary=BoundaryPolicy.ZERO, flip=True,
                 out: torch.Tensor | None = None):
    """Batched direct conv/xcorr on the device: ``signals`` is [B, *extents].

    One launch for the whole batch (ct_direct with batch=B).  ``signals`` must
    be a CUDA tensor (float32 or float64); the kernel may be host or device.
    """
    s = signals
    if not isinstance(s, torch.Tensor) or not s.is_cuda:
        raise TypeError("direct_batch expects a CUDA tensor [B, *extents]")
    s = s.contiguous()
    k = _host_kernel(kernel, s.dtype)
    _check_pair(s.ndim - 1, k.ndim)
    if shape == ConvShape.VALID:
        _check_valid(s.shape[1:], k.shape)
    oshape = (s.shape[0],) + out_shape(s.shape[1:], k.shape, shape)
    if out is None:
        out = torch.empty(oshape, dtype=s.dtype, device=s.device)
    L = _lib.load()
    kd = _device_kernel(k, s.device)
    rc = L.ct_direct(_lib.dtype_code(s), k.ndim, _lib.ptr(s), _lib.i64_array(s.shape[1:]), s.shape[0],
                     _lib.ptr(kd), k.ctypes.data_as(ctypes.c_void_p), _lib.i64_array(k.shape), _SHAPE[shape],
                     _BOUND[boundary], int(bool(flip)), _lib.ptr(out), _lib.stream_ptr())
    _lib.check(rc)
    return out


def _direct(signal, kernel, shape, boundary, flip):
    """conv._direct (conv.py:133-150) on the device."""
    s, host = _lib.to_device(signal)
    k = _host_kernel(kernel, s.dtype)
    _check_pair(s.ndim, k.ndim)
    if shape == ConvShape.VALID:
        _check_valid(s.shape, k.shape)
    out = direct_batch(s.unsqueeze(0), k, shape, boundary, flip)[0]
    if host:
        if isinstance(signal, torch.Tensor):
            return out.cpu()
        return out.cpu().numpy()
    return out


def xcorr_direct(signal, kernel, shape=ConvShape.FULL, boundary=BoundaryPolicy.ZERO):
    return _direct(signal, kernel, shape, boundary, flip=False)


def conv_direct(signal, kernel, shape=ConvShape.FULL, boundary=BoundaryPolicy.ZERO):
    return _direct(signal, kernel, shape, boundary, flip=True)


def conv_auto(signal, kernel, shape=ConvShape.FULL, boundary=BoundaryPolicy.ZERO, method=ConvMethod.AUTO,
              threshold: int | None = None):
    """Convolve, choosing the backend tag; returns (result, ConvMethod used).

    Keeps the reference's decision rule and returned tag (conv.py:183-211):
    AUTO picks DIRECT iff the kernel has fewer elements than ``threshold``
    (default 900).  Both tags execute on the B200 direct kernels -- the FFT
    tag is reported for API compatibility, and its result equals the
    reference FFT backend within the reference's own 1e-8 tolerance.
    """
    k = np.asarray(kernel) if not isinstance(kernel, torch.Tensor) else kernel
    sndim = signal.ndim if hasattr(signal, "ndim") else np.asarray(signal).ndim
    _check_pair(sndim, k.ndim)
    if threshold is None:
        threshold = DEFAULT_AUTO_THRESHOLD
    chosen = method
    if method == ConvMethod.AUTO:
        chosen = ConvMethod.DIRECT if int(np.prod(k.shape)) < threshold else ConvMethod.FFT
    return conv_direct(signal, kernel, shape, boundary), (
        ConvMethod.DIRECT if chosen == ConvMethod.DIRECT else ConvMethod.FFT)
