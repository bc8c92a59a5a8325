"""Benchmark: BFS-kNN GTEPS (headline), SGD edge-updates/s, end-to-end layout s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (N > 1)

Without a launcher, --gpus N > 1 re-executes itself under
torch.distributed.run with N ranks; under a launcher WORLD_SIZE must equal
--gpus.  --cpu-dry-run rehearses the N-rank record exchange on CPU (gloo).

Workload (BASELINE.json configs[4], the scaling-sweep config): partial-BFS
kNN, k = 15, on a random geometric graph in the unit square, n = 4,000,000,
radius for average degree 12, seed 4, largest component (3,999,956
vertices, 23,983,705 edges).  One step = one pass of the C0 hot path over
every source of this rank's shard (sources sharded across ranks, records
all-gathered over NCCL when N > 1).  The graph CSR (208 MB) is larger than
the 126 MB L2 and L2 is additionally flushed before every timed step,
outside the step's CUDA events: a 256 MB write, then a 256 MB read whose
evictions write the dirty flush lines back before the step starts.

Work unit: TE = adjacency entries the reference algorithm
scans (sum over sources of the degrees of expanded vertices), counted by the
kernel itself; GTEPS = TE / step time.  Roofline: algorithmic bytes per
launch = 8 * expanded + 4 * scanned + 8 * k * sources (two int32 offsets per
expanded vertex, one int32 per scanned entry, k (id, dist) int32 pairs
written) over the measured HBM copy bandwidth (MEASURED_PEAKS.json).

Secondary lines inside the same JSON object:
  sgd         Hogwild fp32 full epochs on the c5 kNN graph (E = sym edges),
              edge-updates/s (one positive visit + 5 negatives), 88 B/update
  layout_e2e  SL-GUMAP on c3 (BA n=100k, 200 epochs, 10% window, random
              init) through the public API from host arrays: seconds
The CPU baseline is the oracle's C port of the reference algorithm
(oracle/oracle.c, all host threads) over the full c5 workload, repeated to
>= 10 s; the reference itself is Python/numba and cannot travel to the GPU
box.
"""

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

K_NN = 15
SEED = 4
WORKLOAD = "c5: partial-BFS kNN k=15 on RGG(n=4M, avg deg 12, seed 4) LCC"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _profile_traffic(kernel):
    """dram bytes per launch from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(kernel)
    except Exception:
        return None


class ClockSampler:
    """SM clocks and throttle reasons sampled through NVML every ~2 ms during
    the timed region (nvidia-smi is too slow for a ~20 ms region); falls back
    to nvidia-smi when NVML is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index=0, period=0.001):
        self.index = index
        self.period = period
        self.samples = []
        self._stop = threading.Event()
        self._th = None

    def _run(self):
        if self._nvml is not None:
            pynvml, h, mx = self._nvml
            while not self._stop.is_set():
                try:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((sm, mx, rs))
                except Exception:  # noqa: BLE001 -- a missed sample, not a failure
                    pass
                self._stop.wait(self.period)
            return
        q = "clocks.sm,clocks.max.sm"
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip().split(",")
                self.samples.append((float(out[0]), float(out[1]), 0))
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        # NVML is initialised here, before the timed region starts, so the
        # sampling thread is live from the region's first microsecond
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            self._nvml = (pynvml, h, mx)
        except Exception:  # noqa: BLE001 -- fall back to nvidia-smi
            self._nvml = None
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._th:
            self._th.join(timeout=10)
        if self._nvml is not None:
            try:
                self._nvml[0].nvmlShutdown()
            except Exception:  # noqa: BLE001
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock samples"],
                    "samples": 0}
        sm = [float(x[0]) for x in self.samples]
        reasons = sorted({name for _, _, r in self.samples for name, bit in self.REASONS.items()
                          if int(r) & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(float(x[1]) for x in self.samples),
                "sm_min_mhz": min(sm), "reasons": reasons, "samples": len(self.samples),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def bench_config(n, m, te, ws):
    """The workload description both arms print, key for key (the driver
    compares the two arms' config objects)."""
    per = -(-n // ws)
    return {"workload": WORKLOAD, "n": n, "m": int(m), "k": K_NN, "seed": SEED,
            "sources_per_rank": per, "te_per_step": int(te),
            "l2": "CSR 208 MB > 126 MB L2; L2 flushed before every timed step (256 MB write, "
                  "then a 256 MB read that writes the dirty lines back outside the step)",
            "parallelism": f"sources sharded over {ws} GPU(s)"
            + (", records all-gathered over NCCL in 4 rounds overlapped with the kernels"
               if ws > 1 else "")}


def build_graph(name="c5"):
    from paper_2509_19703_b200 import fixtures
    t = time.time()
    g = fixtures.config_graph(name)
    return g, time.time() - t


# --------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    ws, rank, local = _dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", torch.cuda.current_device())
    import paper_2509_19703_b200 as gu
    from paper_2509_19703_b200 import _lib
    from paper_2509_19703_b200.device import device_csr, stream_ptr
    from paper_2509_19703_b200.distributed import shard_buffers, shard_range
    from paper_2509_19703_b200.neighbors import partial_bfs_records

    g, gen_s = build_graph("c5")
    n = g.n
    csr = device_csr(g, dev)
    begin, end, per = shard_range(n, rank, ws)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_sum = torch.empty((), dtype=torch.int64, device=dev)

    def flush_l2():
        # write 256 MB (> 126 MB L2), then read it back: the read evicts the
        # write's dirty lines, so their write-back happens here and not inside
        # the next timed step (which then starts from a clean, cold L2)
        flush.fill_(1)
        torch.sum(flush.view(torch.int64), dim=0, out=flush_sum)

    # work units: one counted pass (untimed)
    work = torch.zeros(2, dtype=torch.int64, device=dev)
    partial_bfs_records(csr, K_NN, SEED, begin, end, work=work)
    torch.cuda.synchronize()
    scanned, expanded = (int(x) for x in work.cpu().tolist())

    # records land in the padded shard buffers the all_gather sends as they are
    bufs = shard_buffers(per, K_NN, dev)
    out = (bufs[0][: end - begin], bufs[1][: end - begin], bufs[2][: end - begin])
    # one persistent workspace, as a serving loop would hold it
    from paper_2509_19703_b200.neighbors import _tier2_warps
    from paper_2509_19703_b200.device import workspace
    tw = _tier2_warps(n)
    pws = workspace(_lib.load().gu_partial_bfs_workspace_size(n, end - begin, tw), dev)

    if ws > 1:
        # every rank ends the step holding all n records: interleaved rounds,
        # each round's NCCL all_gather overlapping the next round's kernels
        from paper_2509_19703_b200.distributed import chunk_rows, exchange_records
        xws = workspace(_lib.load().gu_partial_bfs_workspace_size(n, chunk_rows(n, ws, 4), tw), dev)

        def xcompute(b, e, o):
            partial_bfs_records(csr, K_NN, SEED, b, e, out=o, tier2_warps=tw, ws=xws)

    def step():
        if ws > 1:
            return exchange_records(xcompute, n, K_NN, dev, chunks=4)[0]
        partial_bfs_records(csr, K_NN, SEED, begin, end, out=out, tier2_warps=tw, ws=pws)
        return bufs[0]

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    times = []
    st = torch.cuda.current_stream()
    with ClockSampler(local) as clk:
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        # per-step device time (events on the launching stream around each
        # step; the L2 flush sits between steps, outside them); no host sync
        # inside the loop, so Python launch overhead is not in the window
        evs = []
        for _ in range(args.steps):
            flush_l2()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            step()
            e1.record(st)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        times = [a.elapsed_time(b) for a, b in evs]
        if ws > 1:
            dist.barrier()
    my_ms = sum(times) / len(times)
    te_tot = scanned
    if ws > 1:
        t = torch.tensor([my_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        my_ms = float(t.item())
        c = torch.tensor([scanned, expanded], device=dev, dtype=torch.int64)
        dist.all_reduce(c)
        te_tot, exp_tot = (int(x) for x in c.tolist())
    else:
        exp_tot = expanded
    gteps = te_tot / (my_ms / 1e3) / 1e9

    # roofline of the dominant kernel (per-rank launch)
    peak, peak_kind = _peaks()
    nsrc = end - begin
    alg_bytes = 8 * expanded + 4 * scanned + 8 * K_NN * nsrc
    kern_ms = min(times) if ws == 1 else min(times)
    # time the kNN kernel alone (no gather) for the roofline
    kevs = []
    for _ in range(max(3, args.steps)):
        flush_l2()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        partial_bfs_records(csr, K_NN, SEED, begin, end, out=out, tier2_warps=tw, ws=pws)
        e1.record(st)
        kevs.append((e0, e1))
    torch.cuda.synchronize()
    ktimes = [a.elapsed_time(b) for a, b in kevs]
    kern_ms = sum(ktimes) / len(ktimes)
    achieved = alg_bytes / (kern_ms / 1e3) / 1e9
    traffic = _profile_traffic("pbfs_fast")
    result = {
        "metric": "BFS-kNN GTEPS (partial BFS kNN, k=15)",
        "value": round(gteps, 4),
        "unit": "GTEPS",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(my_ms, 4),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "int32",
        "data": "synthetic (seeded RGG fixture, paper datasets absent)",
        "config": bench_config(n, g.m, te_tot, ws),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": traffic, "peak_source": peak_kind,
                     "kernel": "gu_partial_bfs_knn (tier F pbfs_fast<8>: 95% of the call's kernel time, "
                               "profiles/r02_bench_launches_summary.txt)",
                     "alg_bytes_per_launch": alg_bytes, "kernel_ms": round(kern_ms, 4),
                     "limiter": "issue + shared-memory pipe, not HBM: ~535 warp instructions per "
                                "source at 84% of peak issue, LSU wavefronts at 74% of peak (hash "
                                "CAS / atomicMin / clears), DRAM at 26% of peak "
                                "(profiles/r02_ncu_pbfs_fast_final.txt, r02_sass_pbfs_fast.txt, DESIGN.md K3)"},
        # per step: tiers F, 1a, H, C (or 1b), slot clear, tier 2 -- once, or once
        # per exchange round at N > 1 (NCCL and dtype-cast kernels not counted)
        "gpu_launches": 6 * args.steps * (4 if ws > 1 else 1),
        "clocks": clk.summary(),
        "fixture_gen_s": round(gen_s, 2),
    }

    e2e = _e2e_partial(gu, g, args, gteps_te=te_tot, ws=ws, rank=rank, dev=dev)
    if rank == 0:
        result["e2e"] = e2e
        if not args.skip_layout:
            result["c1"] = _c1_bench(gu, g, args, dev, peak)
            result["apsp"] = _apsp_bench(gu, args, peak)
        if not args.skip_sgd:
            result["sgd"] = _sgd_bench(gu, g, args, dev, peak)
        if os.environ.get("GU_BENCH_C1_AGAIN"):
            result["c1_after_sgd"] = _c1_bench(gu, g, args, dev, peak)
        if not args.skip_layout:
            result["layout_e2e"] = _layout_e2e(gu)
            result["full_path"] = _full_path(gu, peak)
        if not args.skip_next:
            result["next_rows"] = _next_rows(gu, g)
        if not args.skip_cpu:
            result["cpu_baseline"] = _cpu_baseline(g)
        print(json.dumps(result), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


def _e2e_partial(gu, g, args, gteps_te, ws=1, rank=0, dev=None):
    """Public API end to end: pinned host Graph arrays in, numpy DirectedKnn
    out, copies timed.  At N > 1 every rank runs the sharded public call
    (distributed.sharded_knn: replicated upload, source shards, NCCL
    all_gather) and rank 0 reads the result back; max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2509_19703_b200.distributed import sharded_knn
    from paper_2509_19703_b200.graph import Graph

    def pinned(a):  # the step's inputs live in pinned host memory (contract)
        t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
        out = t.numpy()
        out[...] = a
        return out

    def fresh():
        return Graph(n=g.n, m=g.m, adj_indptr=pinned(np.asarray(g.adj_indptr)),
                     adj_indices=pinned(np.asarray(g.adj_indices)), edges=g.edges)

    def pageable():
        return Graph(n=g.n, m=g.m, adj_indptr=np.array(g.adj_indptr),
                     adj_indices=np.array(g.adj_indices), edges=g.edges)

    times = []
    first = None
    h2d = d2h = 0
    # at least 5 untimed calls: the first ones also fill torch's pinned-host
    # block cache for the ~0.5 GB of result buffers (cudaHostAlloc is slow);
    # the very first call is reported on its own (cold)
    warm = max(5, args.warmup)
    for i in range(warm + args.steps):
        gg = fresh()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if ws > 1:
            knn = sharded_knn(gg, K_NN, seed=SEED, mode="partial")
        else:
            _, knn = gu.partial_bfs(gg, K_NN, seed=SEED)
        if rank == 0:
            sent = getattr(knn, "_pending_bytes", None)  # the bytes that crossed PCIe
            ip, dst, dd = knn.indptr, knn.dst, knn.dist
            d2h = sent if sent else ip.nbytes + dst.nbytes + dd.nbytes
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if i == 0:
            first = dt
        if i >= warm:
            times.append(dt)
        h2d = ws * (gg.adj_indptr.nbytes + gg.adj_indices.nbytes)
    t = sum(times) / len(times)
    # the reference's own input: a Graph of ordinary (pageable) numpy arrays
    ptimes = []
    for i in range(args.steps + 1):  # the first call warms the staging threads, untimed
        gg = pageable()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if ws > 1:
            knn = sharded_knn(gg, K_NN, seed=SEED, mode="partial")
        else:
            _, knn = gu.partial_bfs(gg, K_NN, seed=SEED)
        if rank == 0:
            knn.indptr, knn.dst, knn.dist
        torch.cuda.synchronize()
        if i:
            ptimes.append(time.perf_counter() - t0)
    tp = statistics.median(ptimes)
    if ws > 1:
        tt = torch.tensor([t, tp, first], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t, tp, first = (float(x) for x in tt.tolist())
    api = ("paper_2509_19703_b200.distributed.sharded_knn(Graph(pinned host arrays), 15, seed=4)"
           if ws > 1 else "paper_2509_19703_b200.partial_bfs(Graph(pinned host arrays), 15, seed=4)")
    return {"value": round(gteps_te / t / 1e9, 4), "unit": "GTEPS", "seconds": round(t, 4),
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "api": api,
            "inputs": "pinned host arrays, warm (5+ untimed calls first)",
            "first_call": {"seconds": round(first, 4), "gteps": round(gteps_te / first / 1e9, 4),
                           "note": "the process's first public call: pinned-buffer "
                                   "allocation and CSR upload included"},
            "pageable": {"value": round(gteps_te / tp / 1e9, 4), "unit": "GTEPS",
                         "seconds": round(tp, 4),
                         "inputs": "ordinary numpy arrays (the reference's Graph), warm, median of steps"}}


def _sgd_bench(gu, g, args, dev, peak):
    import torch
    from paper_2509_19703_b200 import _lib
    from paper_2509_19703_b200.device import stream_ptr
    from paper_2509_19703_b200.layout import INT32_MAX, _plan_for, sgd_concurrency

    _, knn = gu.partial_bfs(g, K_NN, seed=SEED)
    gk = gu.smooth_knn_weights(knn)
    E = gk.edge_count
    a, b = gu.fit_ab(0.1, 1.0)
    torch.cuda.synchronize()
    tp0 = time.perf_counter()
    plan = _plan_for(gk, SEED, dev)
    torch.cuda.synchronize()
    plan_s = time.perf_counter() - tp0
    init = np.random.default_rng(SEED).uniform(-10, 10, size=(g.n, 2)).astype(np.float32)
    xy = torch.from_numpy(init).to(dev)
    div = torch.full((1,), INT32_MAX, dtype=torch.int32, device=dev)
    T = 200
    st = torch.cuda.current_stream()

    def epochs(e0, e1):
        _lib.call("gu_sgd_epochs", plan.n, plan.E, _lib.ptr(xy), _lib.ptr(plan.edges), plan.record_mode,
                  _lib.ptr(plan.nbr_indptr), _lib.ptr(plan.nbr_indices), _lib.ptr(plan.filter), float(a), float(b),
                  1.0, T, e0, e1, 5, E, 0, plan.seed, sgd_concurrency(plan.n), _lib.ptr(div),
                  stream_ptr(dev))

    epochs(0, max(1, args.warmup))
    torch.cuda.synchronize()
    evs = []
    for i in range(args.steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        epochs(3 + i, 4 + i)
        e1.record(st)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    ts = [a.elapsed_time(b) for a, b in evs]
    ms = sum(ts) / len(ts)
    ups = E / (ms / 1e3)
    achieved = 88.0 * E / (ms / 1e3) / 1e9
    return {"metric": "SGD edge-updates/s (full epoch, 5 negatives, fp32 Hogwild)",
            "value": round(ups, 1), "unit": "updates/s", "E": E, "ms_per_epoch": round(ms, 4),
            "records": {0: "16-byte + gathered 64-bit filter", 1: "32-byte with 128-bit filter",
                        2: "32-byte with neighbour-id window (BFS locality order)"}[plan.record_mode],
            "mean_window_frac": getattr(plan, "mean_window", None),
            "plan_seconds": round(plan_s, 4),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": _profile_traffic("sgd_epoch_kernel"),
                         "alg_bytes_per_update": 88,
                         "limiter": "memory latency (long-scoreboard 69% of stall samples, 42% of "
                                    "issue slots, 47% of warp slots at 54 registers; 5 CTAs per SM "
                                    "changed nothing): the warp-pooled first tries took L2 tag "
                                    "lookups from 73% to 52% of peak (612M -> 373M L2 requests per "
                                    "epoch) and consuming them in place removed the per-slot arrays "
                                    "and the cooperative search; DRAM at 10% of peak, the 32 MB "
                                    "coordinates L2-resident (profiles/r02_ncu_sgd_l2.txt, "
                                    "DESIGN.md K7)"},
            "diverged": int(div.item()) != INT32_MAX}


def _c1_bench(gu, g, args, dev, peak):
    """C1 (gu_smooth_knn + gu_symmetrize) on the c5 kNN graph, device-resident
    records in, KnnGraph arrays out, CUDA events.  Compulsory bytes: read the
    kNN CSR (int64 indptr, int32 dst and dist) and write rho, sigma, the
    symmetrised (src, dst, float64 w) and the int64 neighbour indptr; the
    directed weights are an intermediate and not counted."""
    import torch
    _, knn = gu.partial_bfs(g, K_NN, seed=SEED)
    knn.device("indptr", dev)
    n, nnz = g.n, int(knn.device("dst", dev).shape[0])
    gk = gu.smooth_knn_weights(knn)  # warm
    E = gk.edge_count
    st = torch.cuda.current_stream()
    evs = []
    for _ in range(max(3, args.steps)):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        gu.smooth_knn_weights(knn)
        e1.record(st)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in evs) / len(evs)
    alg = 8 * (n + 1) + 8 * nnz + 16 * n + 16 * E + 8 * (n + 1)
    ach = alg / (ms / 1e3) / 1e9
    return {"metric": "C1 smooth kNN weights + fuzzy union (c5 kNN graph)", "ms": round(ms, 4),
            "n": n, "nnz": nnz, "E": E,
            "roofline": {"bound": "hbm", "achieved": round(ach, 2), "peak": peak, "unit": "GB/s",
                         "frac": round(ach / peak, 4), "alg_bytes": alg,
                         "traffic": _profile_traffic("c1_total"),
                         "note": "host syncs of the call (row-length max, E) included"}}


def _apsp_bench(gu, args, peak):
    """A2 all_pairs_bfs rows kernel alone (gu_apsp_rows, 64-source bitset
    BFS writing the int32 n x n matrix to HBM) on c2's G' (n = 20k):
    algorithmic bytes = ceil(n/64) * 2m * 12 (a 4-byte index and an 8-byte
    frontier word per adjacency entry per 64-source batch) + 4 n^2 written."""
    import torch
    from paper_2509_19703_b200 import _lib, fixtures
    from paper_2509_19703_b200.device import device_csr, stream_ptr, workspace

    g = fixtures.config_graph("c2")
    csr = device_csr(g)
    n = g.n
    bif = 148 * 2
    ws = workspace(_lib.load().gu_full_bfs_workspace_size(n, 0, bif), csr.device)
    rows = torch.empty((n, n), dtype=torch.int32, device=csr.device)
    st = torch.cuda.current_stream()

    def once():
        _lib.call("gu_apsp_rows", n, _lib.ptr(csr.indptr), _lib.ptr(csr.indices), 0, n,
                  _lib.ptr(rows), _lib.ptr(ws), ws.numel(), bif, stream_ptr(csr.device))

    once()
    evs = []
    for _ in range(max(3, args.steps)):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        once()
        e1.record(st)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in evs) / len(evs)
    alg = ((n + 63) // 64) * 2 * g.m * 12 + 4 * n * n
    ach = alg / (ms / 1e3) / 1e9
    te = n * 2 * g.m
    del rows
    return {"metric": "A2 all-pairs BFS rows (c2 G', int32 n x n to HBM)", "ms": round(ms, 4),
            "n": n, "m": int(g.m), "gteps": round(te / ms / 1e6, 2),
            "roofline": {"bound": "hbm", "achieved": round(ach, 2), "peak": peak, "unit": "GB/s",
                         "frac": round(ach / peak, 4), "alg_bytes": alg,
                         "traffic": _profile_traffic("msbfs_apsp")}}


def _full_path(gu, peak):
    """Fused full-BFS kNN (GUMAP / SS-GUMAP C0+C1) on c1 and c2: GTEPS over
    the adjacency entries the early-exit bitset BFS actually scans."""
    import torch
    from paper_2509_19703_b200 import fixtures
    from paper_2509_19703_b200.device import device_csr
    from paper_2509_19703_b200.neighbors import full_knn_records

    out = {}
    for name in ("c1", "c2"):
        g = fixtures.config_graph(name)
        csr = device_csr(g)
        work = torch.zeros(2, dtype=torch.int64, device="cuda")
        full_knn_records(csr, K_NN, 0, 0, g.n, work=work)
        torch.cuda.synchronize()
        te = int(work[0])
        ts = []
        for _ in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            full_knn_records(csr, K_NN, 0, 0, g.n)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sum(ts[1:]) / len(ts[1:])
        out[name] = {"n": g.n, "m": int(g.m), "ms": round(ms, 4), "te": te,
                     "gteps": round(te / ms / 1e6, 3)}
    return {"metric": "BFS-kNN GTEPS, full path (bitset BFS, early exit at the k-th distance, "
                      "numpy tie-break)", "configs": out}


def _layout_gumap_c1(gu):
    """GUMAP on c1 (BASELINE configs[0]) through the public API: all-pairs
    BFS kNN -> weights -> 200 full epochs from random init, seconds."""
    import torch
    from paper_2509_19703_b200 import fixtures

    g = fixtures.grid(2500)

    def once():
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        knn = gu.knn_from_full_distances(gu.all_pairs_bfs(g), 15, seed=0)
        gk = gu.smooth_knn_weights(knn)
        lay = gu.optimize_full(gk, gu.random_init(g, 0, 10.0),
                               gu.OptimizerConfig(iterations=200, k=15, seed=0), tag="GUMAP")
        torch.cuda.synchronize()
        return time.perf_counter() - t0

    once()
    return round(min(once() for _ in range(3)), 4)


def _layout_e2e(gu):
    """SL-GUMAP on c3 through the public API, host arrays in / out."""
    import torch
    from paper_2509_19703_b200 import fixtures
    from paper_2509_19703_b200.graph import Graph

    g = fixtures.scale_free(100_000, seed=2, m0=3)

    def once():
        gg = Graph(n=g.n, m=g.m, adj_indptr=np.array(g.adj_indptr),
                   adj_indices=np.array(g.adj_indices), edges=g.edges)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, knn = gu.partial_bfs(gg, 15, seed=2)
        gk = gu.smooth_knn_weights(knn)
        E = gk.edge_count
        samp = math.log(0.1 * E) / math.log(E)
        cfg = gu.OptimizerConfig(iterations=200, k=15, seed=2, samp=samp)
        lay = gu.optimize_sampled(gk, gu.random_init(gg, 2, 10.0), cfg, tag="SL")
        torch.cuda.synchronize()
        return time.perf_counter() - t0, lay

    once()
    ts = [once()[0] for _ in range(3)]
    return {"metric": "end-to-end layout seconds", "config": "c3 SL-GUMAP BA(100k, m0=3), "
            "200 epochs, 10% window, random init, host arrays in/out", "value": round(min(ts), 4),
            "unit": "s", "higher_is_better": False,
            "c1_gumap_seconds": _layout_gumap_c1(gu),
            "configs": _layout_e2e_configs(gu)}


def _layout_e2e_configs(gu):
    """End-to-end layout seconds on BASELINE c2 (SS-GUMAP: the shared G'
    fixture through g_prime=, all-pairs BFS kNN, 200 full epochs) and c4
    (SSSL-GUMAP: SBM 1M, sparsifier identity at this density, partial BFS,
    200 windowed epochs at the default samp=0.9).  Two numbers each: the
    public driver (run_*_gumap, which starts from spectral_init as the
    reference's drivers do) and the C0 -> C1 -> C2 pipeline from random init.
    Graph generation is outside the timing."""
    import torch

    from paper_2509_19703_b200 import fixtures

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        return round(time.perf_counter() - t, 4)

    out = {}
    try:
        g2p = fixtures.config_graph("c2")  # G' of ER(20000, 200)
        cfg2 = gu.OptimizerConfig(iterations=200, k=15, seed=1)

        def c2_pipe():
            knn = gu.knn_from_full_distances(gu.all_pairs_bfs(g2p), 15, seed=1)
            gk = gu.smooth_knn_weights(knn)
            return gu.optimize_full(gk, gu.random_init(g2p, 1, 10.0), cfg2, tag="SS")

        out["c2_ss_gumap"] = {"n": g2p.n, "m_gprime": g2p.m,
                              "driver_s": timed(lambda: gu.run_ss_gumap(g2p, cfg2, g_prime=g2p)),
                              "random_init_pipeline_s": timed(c2_pipe)}
        g4 = fixtures.config_graph("c4")
        cfg4 = gu.OptimizerConfig(iterations=200, k=15, seed=3)

        def c4_pipe():
            _, knn = gu.partial_bfs(g4, 15, seed=3)
            gk = gu.smooth_knn_weights(knn)
            return gu.optimize_sampled(gk, gu.random_init(g4, 3, 10.0), cfg4, tag="SSSL")

        out["c4_sssl_gumap"] = {"n": g4.n, "m": g4.m,
                                "driver_s": timed(lambda: gu.run_sssl_gumap(g4, cfg4)),
                                "random_init_pipeline_s": timed(c4_pipe)}
    except Exception as exc:  # noqa: BLE001 -- report, never fail the headline
        out["error"] = repr(exc)
    return out



def _next_rows(gu, g5):
    """SURVEY 8(f) rows measured on this GPU (seconds, one warm run then the
    best of two): quality metrics on a c3 SL layout, spectral_init on c4, the
    sparsifier on the c2 base graph, build_graph + LCC at c5 scale.  CPU
    comparisons: profiles/r01_{metrics,spectral,sparsify,ingest}_perf.log."""
    import torch

    from paper_2509_19703_b200 import fixtures
    from paper_2509_19703_b200 import graph as G
    from paper_2509_19703_b200 import metrics as M
    from paper_2509_19703_b200 import sparsify as S

    def best(fn, *a):
        fn(*a)
        ts = []
        for _ in range(2):
            torch.cuda.synchronize()
            t = time.perf_counter()
            v = fn(*a)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t)
        return v, round(min(ts), 4)

    out = {}
    try:
        g3 = fixtures.scale_free(100_000, seed=2, m0=3)
        _, knn = gu.partial_bfs(g3, 15, seed=0)
        gk = gu.smooth_knn_weights(knn)
        E = gk.edge_count
        lay = gu.optimize_sampled(gk, gu.random_init(g3, 0, 10.0), gu.OptimizerConfig(
            iterations=200, k=15, seed=0, samp=math.log(0.1 * E) / math.log(E)))
        v1, t1 = best(M.neighborhood_preservation, g3, lay)
        v2, t2 = best(M.stress, g3, lay)
        v3, t3 = best(M.count_crossings, g3, lay)
        out["metrics_c3"] = {"np": v1, "np_s": t1, "stress": v2, "stress_s": t2,
                             "crossings": v3, "crossings_s": t3}
        g4 = fixtures.config_graph("c4")
        _, t = best(gu.spectral_init, g4, 0)
        out["spectral_init_c4_s"] = t
        g2 = fixtures.erdos_renyi(20000, avg_degree=200, seed=1)
        sg, t = best(S.make_sparsifier, g2)
        out["sparsify_c2_base"] = {"m_in": g2.m, "m_out": sg.m, "seconds": t}
        pairs = np.asarray(g5.edges)
        _, tb = best(G.build_graph, pairs)
        out["build_graph_c5_s"] = tb
    except Exception as exc:  # noqa: BLE001 -- report, never fail the headline
        out["error"] = repr(exc)
    return out

def _cpu_full_pass(O, g, thr, src_end=None):
    """One pass of the oracle's C port over sources [0, src_end) of the c5
    graph (all of them by default): (seconds, TE)."""
    end = g.n if src_end is None else src_end
    t0 = time.perf_counter()
    _, _, _, sc, _ = O.partial_bfs_raw(g, K_NN, SEED, 0, end, nthreads=thr, work=True)
    return time.perf_counter() - t0, int(sc.sum())


def _single_core(O, g, min_seconds=4.0):
    """The reference is single-threaded numba (_kernels.py:59-60, no prange;
    BASELINE.md 2 plans 1 core): the same port on ONE host thread, over the
    first quarter of the c5 sources, repeated to >= min_seconds."""
    end = g.n // 4
    tot, te, passes = 0.0, 0, 0
    while tot < min_seconds or passes < 1:
        dt, t = _cpu_full_pass(O, g, 1, end)
        tot, te, passes = tot + dt, te + t, passes + 1
    return {"value": round(te / tot / 1e9, 5), "unit": "GTEPS", "cores": 1, "kind": "port",
            "sample": f"sources 0..{end - 1} of c5 ({te // passes} adjacency entries) x {passes} "
                      "passes on one thread", "seconds": round(tot, 3)}


def _cpu_baseline(g, min_seconds=10.0, max_passes=40):
    """The whole c5 workload on the host cores, repeated until >= min_seconds
    of CPU work (the full workload is ~0.5 s on 16 threads, so no sampling),
    plus the one-thread figure of the single-threaded reference."""
    from oracle import oracle as O
    O.build()
    thr = O.max_threads()
    tot, te, passes = 0.0, 0, 0
    while passes < max_passes and (tot < min_seconds or passes < 2):
        dt, t = _cpu_full_pass(O, g, thr)
        tot, te, passes = tot + dt, te + t, passes + 1
    return {"value": round(te / tot / 1e9, 5), "unit": "GTEPS", "cores": thr, "kind": "port",
            "sample": f"full c5 workload (all {g.n} sources, {te // passes} adjacency entries) x "
                      f"{passes} passes, oracle/oracle.c partial_bfs_all restatement",
            "seconds": round(tot, 3), "single_core": _single_core(O, g)}


# ---------------------------------------------------------- reference arm
def run_reference(args):
    """The reference algorithm's CPU implementation (the oracle's C port of
    _kernels.py:60-131, all host threads); one step = the full c5 workload,
    same metric, unit and config as our arm.  No GPU is touched: CUDA is
    hidden before torch can be imported, so the fixture's largest-component
    pass takes the host path and libgumap.so is never loaded."""
    os.environ["CUDA_VISIBLE_DEVICES"] = ""
    ws, rank, local = _dist_env()
    if rank != 0:
        return
    n_gpus = max(ws, args.gpus)
    from oracle import oracle as O
    O.build()
    g, _ = build_graph("c5")
    thr = O.max_threads()
    for _ in range(args.warmup):
        _cpu_full_pass(O, g, thr)
    ts, te = [], 0
    for _ in range(args.steps):
        dt, t = _cpu_full_pass(O, g, thr)
        ts.append(dt)
        te += t
    tot = sum(ts)
    v = te / tot / 1e9
    out = {"impl": "reference", "metric": "BFS-kNN GTEPS (partial BFS kNN, k=15)",
           "value": round(v, 5), "unit": "GTEPS", "n_gpus": n_gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(1e3 * tot / args.steps, 3),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
           "dtype": "int32", "data": "synthetic (seeded RGG fixture, paper datasets absent)",
           "config": bench_config(g.n, g.m, te // args.steps, n_gpus),
           "cpu_baseline": {"value": round(v, 5), "unit": "GTEPS", "cores": thr, "kind": "port",
                            "sample": f"full c5 workload (all {g.n} sources) per step, "
                                      "oracle/oracle.c partial_bfs_all restatement",
                            "single_core": _single_core(O, g)},
           "e2e": {"value": round(v, 5), "unit": "GTEPS", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------- N-rank launch
def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _spawn_ranks(args):
    """`python bench.py --gpus N` without a torchrun launcher: re-exec this
    script under torch.distributed.run with N ranks (one per GPU) on
    127.0.0.1 and return its exit code; rank 0 prints the JSON line.  NCCL
    prints its communicator-init lines (NCCL_DEBUG=INFO, subsystem INIT) so
    the N-rank communicator is visible in the log."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


def run_cpu_dry_run(args):
    """CPU rehearsal of the N-rank path (gloo; no GPU): each rank fills its
    interleaved source rounds with the oracle's records (the GPU kernels'
    stand-in) through distributed.exchange_records -- the same exchange the
    GPU step runs -- and the gathered records must equal the one-process
    oracle result bit for bit.  Rank 0 prints a JSON line with n_gpus."""
    import torch
    import torch.distributed as dist

    ws, rank, _ = _dist_env()
    dist.init_process_group("gloo")
    from oracle import oracle as O
    from paper_2509_19703_b200 import fixtures as F
    from paper_2509_19703_b200.distributed import exchange_records

    g = F.scale_free(20000, seed=7, m0=3)

    def compute(b, e, out):
        nbr, dd, cnt = O.partial_bfs_raw(g, K_NN, SEED, b, e, nthreads=2)
        out[0].copy_(torch.from_numpy(nbr.reshape(-1, K_NN)))
        out[1].copy_(torch.from_numpy(dd.reshape(-1, K_NN)))
        out[2].copy_(torch.from_numpy(cnt))

    t0 = time.perf_counter()
    nbr, dd, cnt = exchange_records(compute, g.n, K_NN, torch.device("cpu"), chunks=4)
    dt = time.perf_counter() - t0
    on, od, oc = O.partial_bfs_raw(g, K_NN, SEED, nthreads=2)
    same = (np.array_equal(nbr.numpy().reshape(-1), on) and np.array_equal(dd.numpy().reshape(-1), od)
            and np.array_equal(cnt.numpy(), oc))
    flags = torch.tensor([int(same)])
    dist.all_reduce(flags, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(json.dumps({"metric": "cpu dry run of the N-rank record exchange", "n_gpus": ws,
                          "world_size": dist.get_world_size(), "backend": "gloo",
                          "records_identical": bool(flags.item()), "n": g.n,
                          "seconds": round(dt, 3)}), flush=True)
    dist.destroy_process_group()
    if not flags.item():
        sys.exit(1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--skip-sgd", action="store_true")
    ap.add_argument("--skip-layout", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-next", action="store_true")
    ap.add_argument("--cpu-dry-run", action="store_true",
                    help="rehearse the N-rank exchange on CPU (gloo, oracle records)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.impl == "reference":
        run_reference(args)
        return
    launched = "WORLD_SIZE" in os.environ
    if not launched and args.gpus > 1:
        sys.exit(_spawn_ranks(args))
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws != args.gpus:
        print(f"bench.py: WORLD_SIZE={ws} but --gpus {args.gpus}", file=sys.stderr)
        sys.exit(2)
    if args.cpu_dry_run:
        run_cpu_dry_run(args)
    else:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        run_ours(args)


if __name__ == "__main__":
    main()
