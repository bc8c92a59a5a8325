"""Pageable host -> device upload of the c5 CSR arrays (GPU): device.to_device
(pinned staging, threaded host copy) against plain torch copies."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_19703_b200 import device as D

rng = np.random.default_rng(0)
ix = rng.integers(0, 4_000_000, size=47_967_410).astype(np.int32)
ip = np.cumsum(rng.integers(0, 24, size=4_000_001)).astype(np.int64)
dev = torch.device("cuda")


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1e3 * min(ts), 1e3 * sum(ts) / len(ts)


print("to_device (threaded staging) indices+indptr: min %.2f mean %.2f ms" %
      t(lambda: (D.to_device(ix, np.int32, dev), D.to_device(ip, np.int64, dev))))
print("torch .to(dev) pageable:                    min %.2f mean %.2f ms" %
      t(lambda: (torch.from_numpy(ix).to(dev), torch.from_numpy(ip).to(dev))))
for th in (1, 2, 4, 8, 16):
    D._COPY_POOL = None
    os.environ["GU_COPY_THREADS"] = str(th)
    print(f"threads={th}: min %.2f mean %.2f ms" %
          t(lambda: (D.to_device(ix, np.int32, dev), D.to_device(ip, np.int64, dev))))
