"""Host-only parts of the synth drop-in (no kernel is called): score_mse /
ScoreReport semantics (synth.py:166-208) and the result types of generate
(SyntheticSequence, synth.py:61-65)."""

import numpy as np
import pytest

import paper_1612_08825_b200 as ct


def _csv(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return p


HDR = "frame,ttc,foe_x,foe_y,residual,level,degenerate\n"


def test_score_mse_mean_over_shared_frames(tmp_path):
    pred = _csv(tmp_path, "p.csv", HDR + "0,11.0,0,0,0,0,false\n1,7.0,0,0,0,1,false\n3,1.0,0,0,0,0,false\n")
    truth = _csv(tmp_path, "t.csv", "frame,ttc,foe_x,foe_y\n0,10,5,5\n1,9,5,5\n2,8,5,5\n")
    rep = ct.score_mse(pred, truth)
    assert rep == ct.ScoreReport(mse=pytest.approx(2.5), compared=2, excluded=0)


def test_score_mse_counts_degenerate_and_nonfinite(tmp_path):
    pred = _csv(tmp_path, "p.csv", HDR + "0,12.0,0,0,0,0,false\n1,-inf,nan,nan,0,0,false\n"
                                         "2,3.0,0,0,0,0,true\n")
    truth = _csv(tmp_path, "t.csv", "frame,ttc,foe_x,foe_y\n0,10,5,5\n1,9,5,5\n2,8,5,5\n")
    rep = ct.score_mse(pred, truth)
    assert (rep.compared, rep.excluded) == (1, 2) and rep.mse == pytest.approx(4.0)


@pytest.mark.parametrize("pred_text,truth_text", [
    ("frame,ttc\n4,1.0\n", "frame,ttc\n0,1.0\n"),                 # no shared frame
    ("frame,ttc,degenerate\n0,nan,true\n", "frame,ttc\n0,1.0\n"),  # nothing comparable
    ("x,y\n0,1\n", "frame,ttc\n0,1.0\n"),                          # not a ttc CSV
])
def test_score_mse_errors(tmp_path, pred_text, truth_text):
    with pytest.raises(ValueError):
        ct.score_mse(_csv(tmp_path, "p.csv", pred_text), _csv(tmp_path, "t.csv", truth_text))


def test_synthetic_sequence_fields():
    assert tuple(ct.SyntheticSequence.__dataclass_fields__) == ("frames", "truth", "config")
    seq = ct.SyntheticSequence(frames=np.zeros((2, 16, 16)), truth=np.zeros((2, 4)), config=ct.SynthConfig(frames=2))
    assert seq.config.frames == 2


def test_image_write_pgm_and_write_sequence(tmp_path):
    # tensor.image_write_pgm (tensor.py:139-148) and synth.write_sequence (synth.py:149-162): host I/O
    img = np.array([[0.0, 0.5 / 255, 1.5 / 255, 1.0], [-1.0, 2.0, 0.25, 0.75]])
    ct.image_write_pgm(img, tmp_path / "a.pgm")
    raw = (tmp_path / "a.pgm").read_bytes()
    assert raw.startswith(b"P5\n4 2\n255\n")
    assert list(raw[len(b"P5\n4 2\n255\n"):]) == [0, 0, 2, 255, 0, 255, 64, 191]  # clamp, round half to even
    with pytest.raises(ValueError):
        ct.image_write_pgm(np.zeros(3), tmp_path / "b.pgm")
    cfg = ct.SynthConfig(width=16, height=16, frames=3, t0=10.0)
    frames = np.random.default_rng(1).random((3, 16, 16))
    truth = np.array([(t, 10.0 - t, 6.4, 8.8) for t in range(3)])
    seq = ct.SyntheticSequence(frames=frames, truth=truth, config=cfg)
    ct.write_sequence(seq, tmp_path / "s1")
    ct.write_sequence(seq, tmp_path / "s2")
    names = sorted(p.name for p in (tmp_path / "s1").iterdir())
    assert names == ["frame_000000.pgm", "frame_000001.pgm", "frame_000002.pgm", "truth.csv"]
    for n in names:
        assert (tmp_path / "s1" / n).read_bytes() == (tmp_path / "s2" / n).read_bytes()
    lines = (tmp_path / "s1" / "truth.csv").read_text().splitlines()
    assert lines[0] == "frame,ttc,foe_x,foe_y" and lines[1] == "0,10,6.4000000000000004,8.8000000000000007"
