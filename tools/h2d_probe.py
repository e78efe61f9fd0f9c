"""Pinned host->device copy bandwidth (the e2e bound): one 1 GiB copy, and 32 MiB
chunks back to back on one stream (the shape of ct_run_sequence_host's copies)."""
import torch
x = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
y = torch.empty(1 << 30, dtype=torch.uint8, device='cuda')
st = torch.cuda.Stream()
for label, ch in (("1 GiB", 1 << 30), ("256 MiB", 256 << 20), ("32 MiB", 32 << 20), ("8 MiB", 8 << 20)):
    with torch.cuda.stream(st):
        for _ in range(2):
            for i in range(0, 1 << 30, ch):
                y[i:i + ch].copy_(x[i:i + ch], non_blocking=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            for i in range(0, 1 << 30, ch):
                y[i:i + ch].copy_(x[i:i + ch], non_blocking=True)
        e1.record()
    e1.synchronize()
    print(f"H2D {label} chunks: {5 * (1 << 30) / (e0.elapsed_time(e1) * 1e-3) / 1e9:.1f} GB/s")
