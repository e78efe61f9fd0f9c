import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle as O, paper_1612_08825_b200 as ct
from paper_1612_08825_b200 import _lib
rng = np.random.default_rng(3)
for h, w in [(37, 50), (33, 257), (300, 29), (5, 5), (64, 511)]:
    fr = O.generate(max(w, 16), max(h, 16), 4, 30.0, (0.4, 0.6), 7, 0.0)[:, :h, :w] + 0.01 * rng.random((4, h, w))
    got = np.array([[getattr(e, f) for f in ("a","b","c","x0","y0","ttc","residual","misfit")] for e in ct.run_sequence(fr, level=0)])
    ref = O.run_sequence(fr, level=0)[:, :8]
    print((h, w), np.nanmax(np.abs(got - ref) / np.abs(ref), axis=0))
f64 = O.generate(480, 270, 4, 300.0, (0.5, 0.5), 11, 0.0)
f32 = torch.from_numpy(f64.astype(np.float32)).cuda()
for lv in range(4):
    try:
        e = ct.run_sequence_batch(f32[None, :2], level=lv); torch.cuda.synchronize()
        print('f32 level', lv, e[0,0,5].item())
    except Exception as ex:
        print('f32 level', lv, 'FAILED', ex); break
