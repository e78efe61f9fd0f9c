"""cfg5 multiscale pipeline timing: V approach videos x N frames of 1080x1920 fp32
(seeds 1000+v), run_sequence_batch(max_level=3), CUDA events over REPS calls.
Prints ms per call, us per frame and the fraction of the level-0 HBM roofline
(8,294,400 B per estimate); saves the estimates to $OUT (if set) for A/B checks.
usage: python tools/time_cfg5.py [V] [N] [REPS]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1612_08825_b200 as ct

V = int(sys.argv[1]) if len(sys.argv) > 1 else 2
N = int(sys.argv[2]) if len(sys.argv) > 2 else 256
REPS = int(sys.argv[3]) if len(sys.argv) > 3 else 5
fr = torch.empty((V, N, 1080, 1920), dtype=torch.float32, device="cuda")
for v in range(V):
    ct.approach_stream(N, 1080, 1920, seed=1000 + v, dtype=torch.float32, out=fr[v])
torch.cuda.synchronize()
est = ct.run_sequence_batch(fr, max_level=3)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(REPS):
    est = ct.run_sequence_batch(fr, max_level=3)
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / REPS
npairs = V * (N - 1)
peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
gbs = npairs * 4 * 1080 * 1920 / (ms * 1e-3) / 1e9
print(json.dumps({"V": V, "N": N, "ms": ms, "us_per_frame": ms * 1e3 / npairs, "est_s": npairs / ms * 1e3,
                  "frac": gbs / peak, "env": {k: v for k, v in os.environ.items() if k.startswith("CT_")}}))
if os.environ.get("OUT"):
    np.save(os.environ["OUT"], est.cpu().numpy())
