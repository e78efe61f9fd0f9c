"""Tensor-core ceiling probe for BASELINE config 4 (2048^2 * 31x31 FULL fp32).

The direct conv as a tensor-core contraction: for each kernel row j0, output
rows are a banded Toeplitz product out[y, x0:x0+BX] += S_j0[y, x0:x0+BX+30] @
T_j0 (T_j0 is (BX+30) x BX with the 31 taps of row j0 on its band).  Stacking
the 31 kernel rows along K gives one GEMM per output column tile:
[oy x 31*(BX+30)] @ [31*(BX+30) x BX], of which 961/(31*(BX+30)) of the
K-products are nonzero.  This script measures (1) the cuBLAS TF32 GEMM rate on
that shape (allow_tf32) as the tensor-core ceiling, (2) the parity of 1xTF32
and 3xTF32 (hi/lo split, three TF32 GEMMs) against the float64 reference
(relative inf-norm, north_star fp32 bar 1e-5) on a 256x256 crop, and prints
the useful-TFLOP/s ceiling = GEMM rate * density / passes.
"""
import json
import sys

import numpy as np
import torch

BX = int(sys.argv[1]) if len(sys.argv) > 1 else 128
K1 = 31
OY = 2078
Kd = K1 * (BX + K1 - 1)
torch.backends.cuda.matmul.allow_tf32 = True
try:  # torch >= 2.9 spelling
    torch.backends.cuda.matmul.fp32_precision = "tf32"
except Exception:
    pass
torch.set_float32_matmul_precision("high")
a = torch.rand((OY, Kd), device="cuda")
b = torch.rand((Kd, BX * 16), device="cuda")  # 16 column tiles side by side: N = 16 * BX
for _ in range(3):
    c = a @ b
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
e0.record()
for _ in range(reps):
    c = a @ b
e1.record()
e1.synchronize()
t = e0.elapsed_time(e1) / reps * 1e-3
gemm_tf = 2.0 * OY * Kd * b.shape[1] / t / 1e12
ab, bb = a.bfloat16(), b.bfloat16()
for _ in range(3):
    cb = ab @ bb
torch.cuda.synchronize()
e0.record()
for _ in range(reps):
    cb = ab @ bb
e1.record()
e1.synchronize()
bf16_tf = 2.0 * OY * Kd * b.shape[1] / (e0.elapsed_time(e1) / reps * 1e-3) / 1e12
density = K1 * K1 / Kd


def toeplitz_conv(s, k, split):
    """FULL xcorr of s (m0 x m1) with k (31 x 31) via per-row Toeplitz GEMMs in TF32."""
    m0, m1 = s.shape
    n0, n1 = k.shape
    o0, o1 = m0 + n0 - 1, m1 + n1 - 1
    sp = torch.zeros((m0 + 2 * (n0 - 1), m1 + 2 * (n1 - 1)), device="cuda", dtype=torch.float32)
    sp[n0 - 1:n0 - 1 + m0, n1 - 1:n1 - 1 + m1] = s
    out = torch.zeros((o0, o1), device="cuda", dtype=torch.float32)
    idx = torch.arange(o1, device="cuda")[None, :] + torch.arange(n1, device="cuda")[:, None]  # [n1, o1]
    for j0 in range(n0):
        rows = sp[j0:j0 + o0]                      # [o0, padded cols]
        win = rows[:, idx]                          # [o0, n1, o1]: win[y, j1, x] = s_pad[y + j0, x + j1]
        kk = k[j0][None, :, None]
        def tf32(x):  # the tensor core's TF32 operand rounding (10-bit mantissa, truncation)
            return (x.contiguous().view(torch.int32) & ~0x1FFF).view(torch.float32)
        # products of TF32 operands are exact in fp64; accumulate in fp64 to isolate the operand rounding
        if split == 1:
            out += torch.einsum("yjx,j->yx", tf32(win).double(), tf32(k[j0]).double()).float()
        else:
            wh, kh = tf32(win), tf32(k[j0])
            wl, kl = tf32(win - wh), tf32(k[j0] - kh)
            out += (torch.einsum("yjx,j->yx", wh.double(), kh.double()) +
                    torch.einsum("yjx,j->yx", wl.double(), kh.double()) +
                    torch.einsum("yjx,j->yx", wh.double(), kl.double())).float()
        del kk
    return out


rng = np.random.Generator(np.random.PCG64(0))
s = rng.random((256, 256)).astype(np.float32)
k = np.random.Generator(np.random.PCG64(1)).standard_normal((31, 31)).astype(np.float32)
sys.path.insert(0, ".")
import oracle
ref = oracle.direct(s.astype(np.float64), k.astype(np.float64), "full", "zero", flip=False)
res = {}
for split in (1, 3):
    got = toeplitz_conv(torch.from_numpy(s).cuda(), torch.from_numpy(k).cuda(), split).double().cpu().numpy()
    res[f"{split}xTF32_rel_inf"] = float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
print(json.dumps({"BX": BX, "gemm_shape": [OY, Kd, b.shape[1]], "tf32_gemm_tflops": gemm_tf, "bf16_gemm_tflops_same_shape": bf16_tf, "density": density,
                  "useful_tflops_1xtf32": gemm_tf * density, "useful_tflops_3xtf32": gemm_tf * density / 3, **res}))
