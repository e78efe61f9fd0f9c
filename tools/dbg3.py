import sys, os, numpy as np, torch
sys.path.insert(0, '.')
import paper_1612_08825_b200 as ct
from paper_1612_08825_b200 import _lib
dt = torch.float32 if sys.argv[1] == 'f32' else torch.float64
h, w = int(sys.argv[2]), int(sys.argv[3])
f = torch.rand((1, 3, h, w), dtype=dt, device='cuda')
try:
    e = ct.run_sequence_batch(f, level=0); torch.cuda.synchronize()
    print(sys.argv[1:], os.environ.get('CT_BAND_ROWS'), 'ok', e[0, 0, 5].item())
except Exception as ex:
    print(sys.argv[1:], os.environ.get('CT_BAND_ROWS'), 'FAIL', str(ex)[:80])
