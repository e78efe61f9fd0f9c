"""Host memcpy bandwidth, pageable -> pinned, over T threads (ctypes.memmove releases the GIL)."""
import ctypes
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

n = 64 << 20
src = np.random.rand(n // 8)
dst = torch.empty(n, dtype=torch.uint8).pin_memory()
sp, dp = src.ctypes.data, dst.data_ptr()
for T in (1, 2, 4, 8, 16):
    per = n // T
    with ThreadPoolExecutor(T) as ex:
        for rep in range(4):
            t0 = time.perf_counter()
            list(ex.map(lambda i: ctypes.memmove(dp + i * per, sp + i * per, per), range(T)))
            dt = time.perf_counter() - t0
        print(T, "threads", round(n / dt / 1e9, 1), "GB/s")
