"""spectral_init step count and per-step time on a config (GPU)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19703_b200 as gu
from paper_2509_19703_b200 import _lib

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
g = gu.config_graph(name)
gu.spectral_init(gu.synth_graph("scale_free", 2000, seed=1, m0=2), seed=0)
counts = {}
orig = _lib.call


def counting(fn, *a):
    counts[fn] = counts.get(fn, 0) + 1
    return orig(fn, *a)


_lib.call = counting
for rep in range(2):
    counts.clear()
    torch.cuda.synchronize()
    t = time.perf_counter()
    gu.spectral_init(g, seed=0)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    steps = counts.get("gu_lanczos_step", 0)
    print(f"{name}: {dt*1e3:.1f} ms, {steps} Lanczos steps ({dt*1e3/max(steps,1):.3f} ms/step), calls {counts}", flush=True)
