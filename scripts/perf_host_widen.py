"""Host u8 -> int32 widening throughput into pinned memory (threads)."""
import concurrent.futures as cf
import os
import time

import numpy as np
import torch

N = 60_000_000
src = torch.randint(0, 3, (N,), dtype=torch.uint8).pin_memory().numpy()
dst = torch.empty(N, dtype=torch.int32, pin_memory=True).numpy()
dst[:] = 0
print("cpus", os.cpu_count(), flush=True)
for th in (1, 4, 8, 16, 32):
    pool = cf.ThreadPoolExecutor(th)
    b = np.linspace(0, N, th + 1).astype(np.int64)
    best = 1e9
    for _ in range(5):
        t = time.perf_counter()
        fs = [pool.submit(np.copyto, dst[x:y], src[x:y], "unsafe") for x, y in zip(b[:-1], b[1:])]
        for f in fs:
            f.result()
        best = min(best, time.perf_counter() - t)
    print(f"threads {th}: {best*1e3:.2f} ms  {4*N/best/1e9:.1f} GB/s out", flush=True)
    pool.shutdown()
