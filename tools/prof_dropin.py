"""Where the time of the drop-in run_sequence(numpy video) call goes (host clock)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1612_08825_b200 as ct
from paper_1612_08825_b200 import ttc

v = torch.rand((64, 256, 256), dtype=torch.float64, device="cuda").cpu().numpy()
vp = torch.from_numpy(v.copy()).pin_memory().numpy()
for _ in range(3):
    ct.run_sequence(v)
torch.cuda.synchronize()


def t(fn, n=20):
    t0 = time.perf_counter()
    for _ in range(n):
        r = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3, r


print("run_sequence(pageable) ms", t(lambda: ct.run_sequence(v))[0])
print("run_sequence(pinned) ms", t(lambda: ct.run_sequence(vp))[0])
print("run_sequence_host(pageable) ms", t(lambda: ttc.run_sequence_host(v[None]))[0])
print("run_sequence_host(pinned) ms", t(lambda: ttc.run_sequence_host(vp[None]))[0])
ms, est = t(lambda: ttc.run_sequence_host(vp[None]))
print("rows -> TtcEstimate ms", t(lambda: [ttc.estimate_from_row(r) for r in est[0]])[0])
d = torch.from_numpy(v).cuda()
print("device run_sequence_batch ms", t(lambda: ct.run_sequence_batch(d[None], level=0))[0])
print("H2D pinned 33.5MB ms", t(lambda: torch.from_numpy(vp).cuda(non_blocking=True))[0])
print("H2D pageable 33.5MB ms", t(lambda: torch.from_numpy(v).cuda())[0])
