"""Time ct_ttc_moments alone on V random cfg2-shaped videos (fraction of HBM roofline)."""
import json, sys
import torch
sys.path.insert(0, '.')
from paper_1612_08825_b200 import _lib
V = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dt = torch.float64 if (len(sys.argv) < 3 or sys.argv[2] == 'f64') else torch.float32
h = int(sys.argv[3]) if len(sys.argv) > 3 else 256
w = int(sys.argv[4]) if len(sys.argv) > 4 else 256
n = int(sys.argv[5]) if len(sys.argv) > 5 else 64
f = torch.rand((V, n, h, w), dtype=dt, device='cuda')
L = _lib.load()
code = _lib.CT_F64 if dt == torch.float64 else _lib.CT_F32
sums = torch.empty((V, n - 1, 11), dtype=torch.float64, device='cuda')
nb = L.ct_ttc_moments_workspace_bytes(code, V, n, h, w)
ws = _lib.workspace(nb, 'cuda')
st = torch.cuda.current_stream()
def go():
    _lib.check(L.ct_ttc_moments(code, _lib.ptr(f), V, n, h, w, _lib.ptr(sums), _lib.ptr(ws), nb, st.cuda_stream))
for _ in range(3): go()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(10): go()
e1.record(st); e1.synchronize()
t = e0.elapsed_time(e1) / 10 * 1e-3
byts = V * (n - 1) * h * w * f.element_size()
peak = json.load(open('MEASURED_PEAKS.json'))['hbm_gbs'] if __import__('os').path.exists('MEASURED_PEAKS.json') else 6550.0
print(f'V={V} {dt} {h}x{w}x{n}: {t*1e3:.3f} ms  {byts/t/1e9:.0f} GB/s  frac {byts/t/1e9/peak:.3f}')
