"""Frame ingestion for the TTC path (SURVEY.md 8(f) "next" row 4).

The reference CLI loads a frame stack from a directory of `frame_*.pgm` files
or one 3-D NDT tensor (cli.py:73-83) and decodes everything on the host to
float64 before the pair loop.  Here:

* PGM frames travel to the device as their raw samples (1 byte per pixel for
  8-bit, 2 for 16-bit -- 8x / 4x fewer bytes over PCIe than float64) and are
  decoded on the device by ct_decode_samples exactly as image_read_pgm does
  (float64(sample) / maxval, tensor.py:104-136); the header parser restates
  the reference's (tokens, `#` comments, one whitespace byte before the
  raster, maxval 255 or 65535, FormatError with the byte offset).
* NDT stacks (tensor.py:56-83) are read with the reference's validation and
  streamed through run_sequence_host.

Only the header/file plumbing runs on the host; decoding and the whole TTC
pipeline run on the device.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np
import torch

from . import _lib
from .ttc import DEFAULT_C_MIN, estimate_from_row, run_sequence_batch, run_sequence_host

NDT_MAGIC = b"NDT1"
_MAX_ELEMENTS = 1 << 40


class FormatError(Exception):
    """Malformed NDT/PGM content; `offset` is the byte position of the fault (tensor.py:25-32)."""

    def __init__(self, message: str, offset: int | None = None):
        if offset is not None:
            message = f"{message} (byte offset {offset})"
        super().__init__(message)
        self.offset = offset


def _pgm_tokens(blob: bytes):
    i = 0
    while True:
        while i < len(blob) and blob[i:i + 1].isspace():
            i += 1
        if i < len(blob) and blob[i:i + 1] == b"#":
            while i < len(blob) and blob[i:i + 1] != b"\n":
                i += 1
            continue
        if i >= len(blob):
            raise FormatError("truncated header", offset=len(blob))
        start = i
        while i < len(blob) and not blob[i:i + 1].isspace() and blob[i:i + 1] != b"#":
            i += 1
        yield blob[start:i], start, i


def pgm_header(blob: bytes) -> tuple[int, int, int, int]:
    """(width, height, maxval, raster_offset) with the reference's checks (tensor.py:104-131)."""
    tokens = _pgm_tokens(blob)
    magic, start, _ = next(tokens)
    if magic == b"P2":
        raise FormatError("ASCII PGM (P2) not supported, use binary P5", offset=start)
    if magic != b"P5":
        raise FormatError(f"bad magic {magic!r}, expected b'P5'", offset=start)
    fields = []
    for _ in range(3):
        tok, start, end = next(tokens)
        try:
            fields.append((int(tok), start, end))
        except ValueError:
            raise FormatError(f"non-numeric header field {tok!r}", offset=start) from None
    (width, wo, _), (height, ho, _), (maxval, mo, raster_at) = fields
    if width < 1:
        raise FormatError(f"bad width {width}", offset=wo)
    if height < 1:
        raise FormatError(f"bad height {height}", offset=ho)
    if maxval not in (255, 65535):
        raise FormatError(f"maxval must be 255 or 65535, got {maxval}", offset=mo)
    raster = raster_at + 1  # exactly one whitespace byte before the raster
    nbytes = width * height * (2 if maxval == 65535 else 1)
    if len(blob) - raster < nbytes:
        raise FormatError(f"short raster: need {nbytes} bytes, have {len(blob) - raster}", offset=len(blob))
    return width, height, maxval, raster


def read_pgm_raw(path) -> tuple[np.ndarray, int]:
    """Raw raster bytes [h, w*bytes] and maxval of one P5 file."""
    blob = Path(path).read_bytes()
    w, h, maxval, raster = pgm_header(blob)
    bps = 2 if maxval == 65535 else 1
    raw = np.frombuffer(blob, dtype=np.uint8, count=w * h * bps, offset=raster).reshape(h, w * bps)
    return raw, maxval


def decode_on_device(raw: torch.Tensor, maxval: int, shape) -> torch.Tensor:
    """float64 image(s) from raw samples already on the device (ct_decode_samples)."""
    bps = 2 if maxval == 65535 else 1
    n = raw.numel() // bps
    out = torch.empty(tuple(shape), dtype=torch.float64, device=raw.device)
    if out.numel() != n:
        raise ValueError("raw sample count does not match the requested shape")
    L = _lib.load()
    _lib.check(L.ct_decode_samples(bps, _lib.ptr(raw), n, float(maxval), _lib.ptr(out), _lib.stream_ptr()))
    return out


def image_write_pgm(img, path) -> None:
    """tensor.image_write_pgm (tensor.py:139-148): an [h, w] image as 8-bit binary
    PGM, values clamped to [0, 1] and rounded half to even.  Host I/O (a CUDA
    tensor is copied back first)."""
    if isinstance(img, torch.Tensor):
        img = img.detach().cpu().numpy()
    img = np.asarray(img, dtype=np.float64)
    if img.ndim != 2:
        raise ValueError(f"image must be 2-D, got ndim {img.ndim}")
    h, w = img.shape
    q = np.rint(np.clip(img, 0.0, 1.0) * 255.0).astype(np.uint8)
    with open(path, "wb") as f:
        f.write(f"P5\n{w} {h}\n255\n".encode("ascii"))
        f.write(q.tobytes(order="C"))


def image_read_pgm(path):
    """tensor.image_read_pgm with the decode on the device; returns a float64 numpy image."""
    raw, maxval = read_pgm_raw(path)
    h = raw.shape[0]
    w = raw.shape[1] // (2 if maxval == 65535 else 1)
    t = torch.tensor(raw, device="cuda")  # copies (raw is a read-only view of the file bytes)
    return decode_on_device(t, maxval, (h, w)).cpu().numpy()


def load_pgm_frames(path) -> torch.Tensor:
    """Directory of frame_*.pgm (sorted, cli.py:75-80) -> float64 CUDA stack [n, h, w].

    The raw samples are gathered into one pinned host buffer, copied once
    (1-2 bytes per pixel) and decoded on the device.
    """
    p = Path(path)
    files = sorted(p.glob("frame_*.pgm"))
    if not files:
        raise FormatError(f"{p}: no frame_*.pgm files")
    first, maxval = read_pgm_raw(files[0])
    pinned = torch.empty((len(files),) + first.shape, dtype=torch.uint8).pin_memory()
    host = pinned.numpy()  # shares the pinned buffer; filled without wrapping read-only arrays
    host[0] = first
    for i, f in enumerate(files[1:], start=1):
        raw, mv = read_pgm_raw(f)
        if raw.shape != first.shape or mv != maxval:
            raise FormatError(f"{f}: frame extents/maxval differ from {files[0].name}")
        host[i] = raw
    dev = pinned.to("cuda", non_blocking=True)
    h = first.shape[0]
    w = first.shape[1] // (2 if maxval == 65535 else 1)
    return decode_on_device(dev, maxval, (len(files), h, w))


def tensor_read(path) -> np.ndarray:
    """NDT reader with the reference's validation (tensor.py:56-83)."""
    blob = Path(path).read_bytes()
    if blob[:4] != NDT_MAGIC:
        raise FormatError(f"bad magic {blob[:4]!r}, expected {NDT_MAGIC!r}", offset=0)
    if len(blob) < 8:
        raise FormatError("truncated header", offset=len(blob))
    (ndim,) = struct.unpack_from("<I", blob, 4)
    if not 1 <= ndim <= 32:
        raise FormatError(f"unsupported ndim {ndim}", offset=4)
    header_end = 8 + 8 * ndim
    if len(blob) < header_end:
        raise FormatError("truncated extent list", offset=len(blob))
    dims = struct.unpack_from(f"<{ndim}Q", blob, 8)
    count = 1
    for i, d in enumerate(dims):
        if d < 1 or d > _MAX_ELEMENTS or count * d > _MAX_ELEMENTS:
            raise FormatError(f"extent overflow: {dims}", offset=8 + 8 * i)
        count *= d
    expected = header_end + 8 * count
    if len(blob) < expected:
        raise FormatError(f"truncated payload: need {count} f64 values, have {(len(blob) - header_end) // 8}",
                          offset=len(blob))
    if len(blob) > expected:
        raise FormatError("trailing bytes after payload", offset=expected)
    return np.frombuffer(blob, dtype="<f8", count=count, offset=header_end).astype(np.float64).reshape(dims)


def run_sequence_frames(path, level: int | None = 0, max_level: int | None = None,
                        c_min: float = DEFAULT_C_MIN):
    """`convtact ttc --frames PATH` compute path (cli.py:86-96): PGM directory or 3-D NDT stack."""
    p = Path(path)
    if p.is_dir():
        frames = load_pgm_frames(p)
        if frames.shape[0] < 2:
            raise ValueError("need at least two frames")
        est = run_sequence_batch(frames[None], level=level, max_level=max_level, c_min=c_min)[0].cpu().numpy()
    else:
        stack = tensor_read(p)
        if stack.ndim != 3:
            raise FormatError(f"{p}: frame stack must be 3-D, got ndim {stack.ndim}")
        if stack.shape[0] < 2:
            raise ValueError("need at least two frames")
        est = run_sequence_host(stack[None], level=level, max_level=max_level, c_min=c_min)[0]
    return [estimate_from_row(r) for r in est]
