import torch, time
x = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
y = torch.empty(1 << 30, dtype=torch.uint8, device='cuda')
for _ in range(3): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): y.copy_(x, non_blocking=True)
e1.record(); e1.synchronize()
print('H2D GB/s', 5 * (1 << 30) / (e0.elapsed_time(e1) * 1e-3) / 1e9)
# chunked on 2 streams
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
ch = 64 << 20
torch.cuda.synchronize(); t0 = time.perf_counter()
for r in range(5):
    for i in range(0, 1 << 30, ch):
        with torch.cuda.stream(s1 if (i // ch) % 2 == 0 else s2):
            y[i:i + ch].copy_(x[i:i + ch], non_blocking=True)
torch.cuda.synchronize()
print('H2D chunked 2 streams GB/s', 5 * (1 << 30) / (time.perf_counter() - t0) / 1e9)
