"""Profiling driver: the cfg2 hot path (fused moments + finalize + solve) on V videos."""
import sys
import torch
sys.path.insert(0, '.')
import paper_1612_08825_b200 as ct
V = int(sys.argv[1]) if len(sys.argv) > 1 else 64
dt = torch.float64 if (len(sys.argv) < 3 or sys.argv[2] == 'f64') else torch.float32
h = int(sys.argv[3]) if len(sys.argv) > 3 else 256
w = int(sys.argv[4]) if len(sys.argv) > 4 else 256
frames = torch.rand((V, 64, h, w), dtype=dt, device='cuda')
for _ in range(3):
    est = ct.run_sequence_batch(frames, level=0)
torch.cuda.synchronize()
print('ok', est.shape)
