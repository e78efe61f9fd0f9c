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
