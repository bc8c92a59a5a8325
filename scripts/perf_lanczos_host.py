"""Host-side split of _top_eigvec cycles on c4 (GPU): step enqueue, H read
(sync), restart work."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19703_b200 as gu
from paper_2509_19703_b200 import _lib, layout

g = gu.config_graph(sys.argv[1] if len(sys.argv) > 1 else "c4")
gu.spectral_init(gu.synth_graph("scale_free", 2000, seed=1, m0=2), seed=0)
acc = {"step_calls": 0.0, "n_steps": 0}
orig = _lib.call


def timed(fn, *a):
    if fn == "gu_lanczos_step":
        t = time.perf_counter()
        r = orig(fn, *a)
        acc["step_calls"] += time.perf_counter() - t
        acc["n_steps"] += 1
        return r
    return orig(fn, *a)


_lib.call = timed
orig_cpu = torch.Tensor.cpu
acc["cpu_s"] = 0.0


def cpu(self, *a, **k):
    t = time.perf_counter()
    r = orig_cpu(self, *a, **k)
    acc["cpu_s"] += time.perf_counter() - t
    return r


torch.Tensor.cpu = cpu
for rep in range(2):
    for key in list(acc):
        acc[key] = 0 if key == "n_steps" else 0.0
    torch.cuda.synchronize()
    t = time.perf_counter()
    gu.spectral_init(g, seed=0)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"total {dt*1e3:.1f} ms; {acc['n_steps']} steps, step-call host time {acc['step_calls']*1e3:.1f} ms "
          f"({acc['step_calls']*1e6/max(1,acc['n_steps']):.1f} us each); .cpu() waits {acc['cpu_s']*1e3:.1f} ms", flush=True)
