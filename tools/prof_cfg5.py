"""Profiling driver: the cfg5 multiscale fp32 pipeline on one 1080x1920 video."""
import sys
import torch
sys.path.insert(0, '.')
import paper_1612_08825_b200 as ct
nf = int(sys.argv[1]) if len(sys.argv) > 1 else 64
fr = torch.empty((1, nf, 1080, 1920), dtype=torch.float32, device='cuda')
ct.approach_stream(nf, 1080, 1920, seed=1000, dtype=torch.float32, out=fr[0])
torch.cuda.synchronize()
for _ in range(3):
    est = ct.run_sequence_batch(fr, max_level=3)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    est = ct.run_sequence_batch(fr, max_level=3)
e1.record(); e1.synchronize()
print('ms per call', e0.elapsed_time(e1) / 10, 'est', est.shape, est[0, :3, 5].tolist(), est[0, :3, 8].tolist())
