"""Frame ingestion: PGM/NDT parsing restated from
tensor.py (CPU tests), raw-sample device decode and the `ttc --frames` compute
path (GPU tests) against the oracle on the same decoded frames."""

import struct

import numpy as np
import pytest

import oracle as O
from paper_1612_08825_b200 import ingest


def write_pgm(img, path, sixteen=False):
    """Writer matching tensor.image_write_pgm (8-bit) plus a 16-bit variant."""
    if sixteen:
        q = np.rint(np.clip(img, 0.0, 1.0) * 65535.0).astype(">u2")
        hdr = f"P5\n# comment line\n{img.shape[1]} {img.shape[0]}\n65535\n"
    else:
        q = np.rint(np.clip(img, 0.0, 1.0) * 255.0).astype(np.uint8)
        hdr = f"P5\n{img.shape[1]} {img.shape[0]}\n255\n"
    with open(path, "wb") as f:
        f.write(hdr.encode("ascii"))
        f.write(q.tobytes())


def write_ndt(t, path):
    t = np.ascontiguousarray(t, dtype=np.float64)
    with open(path, "wb") as f:
        f.write(b"NDT1")
        f.write(struct.pack("<I", t.ndim))
        f.write(struct.pack(f"<{t.ndim}Q", *t.shape))
        f.write(t.tobytes())


def test_pgm_header_and_errors(tmp_path):
    img = np.linspace(0, 1, 35).reshape(5, 7)
    p = tmp_path / "a.pgm"
    write_pgm(img, p, sixteen=True)
    w, h, maxval, raster = ingest.pgm_header(p.read_bytes())
    assert (w, h, maxval) == (7, 5, 65535)
    raw, mv = ingest.read_pgm_raw(p)
    assert raw.shape == (5, 14) and mv == 65535
    for blob, frag in [(b"P2\n1 1\n255\n\x00", "ASCII"), (b"P6\n1 1\n255\n\x00", "bad magic"),
                       (b"P5\n1 x\n255\n\x00", "non-numeric"), (b"P5\n0 1\n255\n\x00", "bad width"),
                       (b"P5\n1 1\n100\n\x00", "maxval"), (b"P5\n4 4\n255\n\x00", "short raster")]:
        with pytest.raises(ingest.FormatError, match=frag):
            ingest.pgm_header(blob)


def test_ndt_reader_and_errors(tmp_path):
    t = np.random.default_rng(0).random((3, 4, 5))
    p = tmp_path / "s.ndt"
    write_ndt(t, p)
    assert np.array_equal(ingest.tensor_read(p), t)
    bad = tmp_path / "b.ndt"
    bad.write_bytes(b"NDT2" + p.read_bytes()[4:])
    with pytest.raises(ingest.FormatError, match="bad magic"):
        ingest.tensor_read(bad)
    bad.write_bytes(p.read_bytes()[:-8])
    with pytest.raises(ingest.FormatError, match="truncated payload"):
        ingest.tensor_read(bad)
    bad.write_bytes(p.read_bytes() + b"\x00")
    with pytest.raises(ingest.FormatError, match="trailing"):
        ingest.tensor_read(bad)


@pytest.mark.gpu
@pytest.mark.parametrize("sixteen", [False, True])
def test_pgm_directory_end_to_end(tmp_path, sixteen):
    frames = O.generate(96, 64, 7, 40.0, (0.5, 0.5), 5, 0.0)
    for i, f in enumerate(frames):
        write_pgm(f, tmp_path / f"frame_{i:06d}.pgm", sixteen)
    # decode exactly as image_read_pgm: float64(sample) / maxval
    raws = [ingest.read_pgm_raw(tmp_path / f"frame_{i:06d}.pgm")[0] for i in range(7)]
    if sixteen:
        dec = np.stack([r.view(">u2").astype(np.float64) / 65535 for r in raws])
    else:
        dec = np.stack([r.astype(np.float64) / 255 for r in raws])
    dev = ingest.load_pgm_frames(tmp_path).cpu().numpy()
    assert np.array_equal(dev, dec)
    assert np.array_equal(ingest.image_read_pgm(tmp_path / "frame_000003.pgm"), dec[3])
    for kw in (dict(level=0), dict(max_level=3)):
        got = ingest.run_sequence_frames(tmp_path, **kw)
        ref = O.run_sequence(dec, **kw)
        for e, r in zip(got, ref):
            assert e.level == int(r[8]) and e.degenerate == bool(r[9])
            assert abs(e.ttc - r[5]) <= 1e-9 * abs(r[5])


@pytest.mark.gpu
def test_ndt_stack_end_to_end(tmp_path):
    frames = O.generate(64, 48, 5, 30.0, (0.45, 0.5), 2, 0.01)
    p = tmp_path / "stack.ndt"
    write_ndt(frames, p)
    got = ingest.run_sequence_frames(p, level=0)
    ref = O.run_sequence(frames, level=0)
    assert [e.level for e in got] == [0] * 4
    assert np.allclose([e.ttc for e in got], ref[:, 5], rtol=1e-9, atol=0)
    write_ndt(frames[0], p)
    with pytest.raises(ingest.FormatError, match="3-D"):
        ingest.run_sequence_frames(p)
