"""One launch of each profiled kernel, for a single ncu --set full capture:
cfg2 moments (f64), cfg3 z-walk conv, cfg4 pair conv, cfg5 level-0 moments (f32) + blur."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_1612_08825_b200 as ct
from paper_1612_08825_b200 import _lib

which = sys.argv[1:] or ['cfg2', 'cfg3', 'cfg4', 'cfg5']
if 'cfg2' in which:
    f = torch.rand((256, 64, 256, 256), dtype=torch.float64, device='cuda')
    L = _lib.load()
    sums = torch.empty((256, 63, 11), dtype=torch.float64, device='cuda')
    nb = L.ct_ttc_moments_workspace_bytes(_lib.CT_F64, 256, 64, 256, 256)
    ws = _lib.workspace(nb, 'cuda')
    _lib.check(L.ct_ttc_moments(_lib.CT_F64, _lib.ptr(f), 256, 64, 256, 256, _lib.ptr(sums), _lib.ptr(ws), nb,
                                torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    del f, ws
if 'cfg3' in which:
    os.environ['CT_CONV_KIND'] = os.environ.get('PROF_CFG3_KIND', '4')
    s = torch.rand((8, 128, 128, 128), dtype=torch.float32, device='cuda')
    k = np.random.Generator(np.random.PCG64(1)).standard_normal((7, 7, 7)).astype(np.float32)
    ct.direct_batch(s, k)
    torch.cuda.synchronize()
if 'cfg4' in which:
    os.environ['CT_CONV_KIND'] = os.environ.get('PROF_CFG4_KIND', '6')
    s = torch.rand((2, 2048, 2048), dtype=torch.float32, device='cuda')
    k = np.random.Generator(np.random.PCG64(1)).standard_normal((31, 31)).astype(np.float32)
    ct.direct_batch(s, k)
    torch.cuda.synchronize()
if 'cfg5' in which:
    os.environ.pop('CT_CONV_KIND', None)
    fr = torch.empty((1, 128, 1080, 1920), dtype=torch.float32, device='cuda')
    ct.approach_stream(128, 1080, 1920, seed=1000, dtype=torch.float32, out=fr[0])
    ct.run_sequence_batch(fr, max_level=3)
    torch.cuda.synchronize()
print('ok')
