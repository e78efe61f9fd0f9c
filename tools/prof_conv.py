"""Profiling driver for the conv configs: python tools/prof_conv.py cfg1|cfg3|cfg4 [reps]."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_1612_08825_b200 as ct
cfg = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if cfg == 'cfg1':
    s = torch.rand((512, 256, 256), dtype=torch.float64, device='cuda')
    k = np.random.Generator(np.random.PCG64(1)).standard_normal((5, 5))
    o = torch.empty((512, 260, 260), dtype=torch.float64, device='cuda')
    work = 512 * 260 * 260
elif cfg == 'cfg3':
    s = torch.rand((8, 128, 128, 128), dtype=torch.float32, device='cuda')
    k = np.random.Generator(np.random.PCG64(1)).standard_normal((7, 7, 7)).astype(np.float32)
    o = torch.empty((8, 134, 134, 134), dtype=torch.float32, device='cuda')
    work = 8 * 134 ** 3
elif cfg == 'w13':  # reference crossover width, fp64, cfg1-sized images
    s = torch.rand((512, 256, 256), dtype=torch.float64, device='cuda')
    k = np.random.Generator(np.random.PCG64(1)).standard_normal((13, 13))
    o = torch.empty((512, 268, 268), dtype=torch.float64, device='cuda')
    work = 512 * 268 * 268
elif cfg == 'w33':  # a width past the tiled instantiations, fp32, cfg4-sized images
    s = torch.rand((2, 2048, 2048), dtype=torch.float32, device='cuda')
    k = np.random.Generator(np.random.PCG64(1)).standard_normal((33, 33)).astype(np.float32)
    o = torch.empty((2, 2080, 2080), dtype=torch.float32, device='cuda')
    work = 2 * 2080 ** 2
else:
    s = torch.rand((2, 2048, 2048), dtype=torch.float32, device='cuda')
    k = np.random.Generator(np.random.PCG64(1)).standard_normal((31, 31)).astype(np.float32)
    o = torch.empty((2, 2078, 2078), dtype=torch.float32, device='cuda')
    work = 2 * 2078 ** 2
for _ in range(2):
    ct.direct_batch(s, k, out=o)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    ct.direct_batch(s, k, out=o)
e1.record(); e1.synchronize()
t = e0.elapsed_time(e1) / reps
flops = {'w13': 512 * 256 * 256 * 169 * 2, 'w33': 2 * 2048 ** 2 * 33 * 33 * 2}.get(cfg)
print(cfg, 'ms', t, 'Gpix/s', work / t / 1e6, '' if flops is None else f'TFLOP/s {flops / t / 1e9:.2f}')
