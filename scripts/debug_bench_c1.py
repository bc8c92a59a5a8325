"""Reproduce bench.py's e2e -> sgd -> c1 sequence on c5 (GPU) and time C1
after each stage, to find what slows the bench's C1 measurement."""
import os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench as B
import paper_2509_19703_b200 as gu

class A:
    steps = 3
    warmup = 3

g, _ = B.build_graph("c5")
dev = torch.device("cuda")
peak = 6545.3
print("c1 fresh:", B._c1_bench(gu, g, A, dev, peak)["ms"], flush=True)
B._e2e_partial(gu, g, A, gteps_te=438660078, dev=dev)
print("c1 after e2e:", B._c1_bench(gu, g, A, dev, peak)["ms"], flush=True)
B._sgd_bench(gu, g, A, dev, peak)
print("c1 after sgd:", B._c1_bench(gu, g, A, dev, peak)["ms"], flush=True)
print("c1 again:", B._c1_bench(gu, g, A, dev, peak)["ms"], flush=True)
import gc; gc.collect()
print("c1 after gc:", B._c1_bench(gu, g, A, dev, peak)["ms"], flush=True)
