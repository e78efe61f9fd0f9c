import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle as O, paper_1612_08825_b200 as ct
f64 = O.generate(480, 270, 4, 300.0, (0.5, 0.5), 11, 0.0)
f32 = torch.from_numpy(f64.astype(np.float32)).cuda()
for lv in range(4):
    e = ct.run_sequence_batch(f32[None, :2], level=lv); torch.cuda.synchronize()
    print('f32 level', lv, e[0,0,5].item(), O.estimate_fixed(f64[0].astype(np.float32), f64[1].astype(np.float32), level=lv)[5])
