#!/usr/bin/env python3
"""Benchmark of the fused-multiloop executor on B200 (driver contract: one JSON line).

Default workload = BASELINE.json's headline: k-means iterations/sec, N=16,777,216 samples,
d=64, k=64, fp64 (config C4), samples sharded contiguously across the ranks; one step = one
k-means iteration = the fused {argmin collect + k*(d+1) predicated reduces} multiloop, the
NCCL allReduce of (counts, sums) across ranks, and the centroid update.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dlx|reference] [--config c4|c1|c2|c3|c5]

--impl reference times the reference's CPU path (the oracle restatement of the reference
loop semantics, oracle/, with all host threads) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (family, params, metric, unit)
    "c4": ("kmeans", dict(n=16_777_216, d=64, k=64),
           "k-means iters/sec (N=16M,d=64,k=64) at 1/2/4/8 B200; fused-op HBM GB/s vs peak", "it/s"),
    "c1": ("kmeans", dict(n=65_536, d=16, k=8), "k-means iters/sec (N=65536,d=16,k=8)", "it/s"),
    # diagnostic: one rank's C4 shard at 8 GPUs (per-iteration fixed costs vs scaling)
    "c4shard8": ("kmeans", dict(n=16_777_216 // 8, d=64, k=64),
                 "k-means iters/sec (N=2M shard of C4 at 8 GPUs, d=64, k=64)", "it/s"),
    "c2": ("logreg", dict(n=1_048_576, d=64), "logistic-regression BGD iters/sec (N=1M,d=64)", "it/s"),
    "l16": ("logreg", dict(n=16_777_216, d=64), "logistic-regression BGD iters/sec (N=16M,d=64)", "it/s"),
    # the fp32-storage opt-in (x rounded to float, fp64 arithmetic): an extension,
    # the reference has no fp32 type
    "l16f32": ("logreg", dict(n=16_777_216, d=64, storage="f32"),
               "logistic-regression BGD iters/sec (N=16M,d=64, fp32 storage of x)", "it/s"),
    "c3": ("gda", dict(n=1_048_576, d=64), "GDA fits/sec (N=1M,d=64)", "fits/s"),
    "c5": ("groupby", dict(n=1_000_000_000, K=64), "GroupBy bucket-count passes/sec (1e9 keys, K=64)", "passes/s"),
    # SURVEY §8 a7 leaves K open and proposes a sweep: 4,096 and 65,536 buckets
    "c5k4096": ("groupby", dict(n=1_000_000_000, K=4096), "GroupBy bucket-count passes/sec (1e9 keys, K=4096)", "passes/s"),
    "c5k65536": ("groupby", dict(n=1_000_000_000, K=65536), "GroupBy bucket-count passes/sec (1e9 keys, K=65536)", "passes/s"),
    "c5k131072": ("groupby", dict(n=1_000_000_000, K=131072), "GroupBy bucket-count passes/sec (1e9 keys, K=131072)", "passes/s"),
    "c5k262144": ("groupby", dict(n=1_000_000_000, K=262144), "GroupBy bucket-count passes/sec (1e9 keys, K=262144)", "passes/s"),
}

# algorithmic bytes per unit: k-means sample d*8 + 4 (int32 assignment write);
# logreg sample 8d + 8; GDA sample 2 * (8d + 8) (two passes); GroupBy key 8.


# fp64 tensor-core (DMMA) peak: not in MEASURED_PEAKS.json (bf16 only) and not in the profiling
# guide, so measured here: scripts/mb/dmma.cu, independent mma.sync f64 chains on every SM,
# best shape 36.9 TFLOP/s (profiles/r75/dmma.txt)
DMMA_PEAK_TFLOPS = 36.9
DMMA_PEAK_KIND = "measured microbench (scripts/mb/dmma.cu, profiles/r75/dmma.txt)"


def algorithmic_bytes(family, p, n_local):
    if family == "kmeans":
        return n_local * (p["d"] * 8 + 4)
    if family == "logreg":
        return n_local * (p["d"] * (4 if p.get("storage") == "f32" else 8) + 8)
    if family == "gda":
        return n_local * (p["d"] * 8 + 8)  # per pass (dominant kernel = one pass)
    if family == "groupby":
        return n_local * 8
    raise ValueError(family)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(config_name):
    """dram bytes per launch of the dominant kernel from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(config_name)
    except Exception:
        return None


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.out = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.out, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.out.close()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [s.strip() for s in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = sorted(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for nm, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": sorted(reasons), "samples": len(rows)}


# ----------------------------------------------------------------------------------------------

def run_reference(args, family, p, metric, unit):
    """The reference CPU path (oracle restatement of the reference multiloop semantics,
    SPEC.md executeDEG chunking, all host threads) on a bounded sample per step."""
    import numpy as np

    import oracle as O
    threads = O.threads()
    t_steps = []
    # every step is the FULL workload (no sampling, no scaling): same config as the GPU arm
    if family == "kmeans":
        n_s = p["n"]
        x = O.rng_units(1, 0, n_s * p["d"]).reshape(n_s, p["d"])
        mu = x[: p["k"]].copy()
        scale = 1.0
        for s in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            a, c, sm = O.kmeans_step(x, p["k"], mu, workers=threads, chunks=4 * threads)
            mu = O.kmeans_update(c, sm)
            dt = time.perf_counter() - t0
            if s >= args.warmup:
                t_steps.append(dt * scale)
        sample = f"full workload: every step is one k-means iteration over all {n_s} samples (d={p['d']}, k={p['k']})"
    elif family == "logreg":
        n_s = p["n"]
        x = O.rng_units(1, 0, n_s * p["d"]).reshape(n_s, p["d"])
        y = O.rng_ints(1, n_s * p["d"], n_s, 2)
        th = np.zeros(p["d"])
        scale = 1.0
        for s in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            th = th - (1.0 / p["n"]) * O.logreg_grad(x, y, th, workers=threads, chunks=4 * threads)
            dt = time.perf_counter() - t0
            if s >= args.warmup:
                t_steps.append(dt * scale)
        sample = f"full workload: every step is one BGD iteration over all {n_s} samples"
    elif family == "gda":
        n_s = p["n"]
        x = O.rng_units(1, 0, n_s * p["d"]).reshape(n_s, p["d"])
        y = O.rng_ints(1, n_s * p["d"], n_s, 2)
        scale = 1.0
        for s in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            n1, s0, s1 = O.gda_pass1(x, y, workers=threads, chunks=4 * threads)
            O.gda_pass2(x, y, s0 / (n_s - n1), s1 / n1, workers=threads, chunks=4 * threads)
            dt = time.perf_counter() - t0
            if s >= args.warmup:
                t_steps.append(dt * scale)
        sample = f"full workload: every step is one GDA fit (pass 1 + pass 2) over all {n_s} samples"
    else:
        n_s = p["n"]
        keys = O.rng_ints(1, 0, n_s, p["K"])
        scale = 1.0
        for s in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            O.groupby_count(keys, p["K"], workers=threads, chunks=4 * threads)
            dt = time.perf_counter() - t0
            if s >= args.warmup:
                t_steps.append(dt * scale)
        sample = f"full workload: every step is one bucket-count pass over all {n_s} keys"
    t = sum(t_steps) / len(t_steps)
    value = 1.0 / t
    return {
        "metric": metric, "value": value, "unit": unit, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64" if family != "groupby" else "int64",
        "data": "synthetic (reference Rng, seed 1)",
        "config": {"workload": args.config, **p},
        "cpu_baseline": {"value": value, "unit": unit, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def cpu_baseline_kmeans(p, budget_s=15.0):
    import oracle as O
    threads = O.threads()
    n_s = p["n"]
    x = O.rng_units(1, 0, n_s * p["d"]).reshape(n_s, p["d"])
    mu = x[: p["k"]].copy()
    times = []
    t_start = time.perf_counter()
    while len(times) < 3 and (time.perf_counter() - t_start) < budget_s:
        t0 = time.perf_counter()
        O.kmeans_step(x, p["k"], mu, workers=threads, chunks=4 * threads)
        times.append(time.perf_counter() - t0)
    t = min(times)
    return {"value": 1.0 / t, "unit": "it/s", "cores": threads, "kind": "port",
            "sample": f"best of {len(times)} k-means iterations over all {n_s} samples (d={p['d']}, k={p['k']}), "
                      f"executeDEG chunking {4 * threads} chunks; not scaled"}


def cpu_baseline_generic(family, p):
    import numpy as np

    import oracle as O
    threads = O.threads()
    n_s = p["n"]   # the full workload, not scaled
    if family == "logreg":
        x = O.rng_units(1, 0, n_s * p["d"]).reshape(n_s, p["d"])
        y = O.rng_ints(1, n_s * p["d"], n_s, 2)
        t0 = time.perf_counter()
        O.logreg_grad(x, y, np.zeros(p["d"]), workers=threads, chunks=4 * threads)
        t = time.perf_counter() - t0
        unit, smp = "it/s", f"1 gradient over all {n_s} samples"
    elif family == "gda":
        x = O.rng_units(1, 0, n_s * p["d"]).reshape(n_s, p["d"])
        y = O.rng_ints(1, n_s * p["d"], n_s, 2)
        t0 = time.perf_counter()
        n1, s0, s1 = O.gda_pass1(x, y, workers=threads, chunks=4 * threads)
        O.gda_pass2(x, y, s0 / (n_s - n1), s1 / n1, workers=threads, chunks=4 * threads)
        t = time.perf_counter() - t0
        unit, smp = "fits/s", f"1 GDA fit (two passes) over all {n_s} samples"
    else:
        keys = O.rng_ints(1, 0, n_s, p["K"])
        t0 = time.perf_counter()
        O.groupby_count(keys, p["K"], workers=threads, chunks=4 * threads)
        t = time.perf_counter() - t0
        unit, smp = "passes/s", f"1 pass over all {n_s} keys"
    return {"value": 1.0 / t, "unit": unit, "cores": threads, "kind": "port", "sample": smp}


def _reduce_dev(dist, dev):
    return "cpu" if dist.get_backend() == "gloo" else dev


def run_dlx(args, family, p, metric, unit, rank, world, local_rank):
    import torch

    from paper_1109_0778_b200 import _lib
    from paper_1109_0778_b200 import multiloops as ml
    from paper_1109_0778_b200.comm import Comm, PeerComm, shard_range
    from paper_1109_0778_b200.programs import KMeansProgram, LogRegProgram

    # DLX_BENCH_SHARED_DEVICE=1 (code-path check only, never a measurement): several ranks on one
    # GPU, gloo for the plumbing and the peer exchange (CUDA IPC works within a device; NCCL
    # refuses duplicate devices)
    shared = os.environ.get("DLX_BENCH_SHARED_DEVICE") == "1"
    if shared and world > 1 and args.comm != "peer":
        raise SystemExit("DLX_BENCH_SHARED_DEVICE needs --comm peer")
    local_dev = local_rank % torch.cuda.device_count() if shared else local_rank
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    dist = None
    comm = None
    if world > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        comm = PeerComm.from_torch_distributed() if args.comm == "peer" else Comm.from_torch_distributed()
    _lib.load()

    def barrier():
        if dist is not None:
            dist.barrier()

    n = p["n"]
    lo, hi = shard_range(n, rank, world)
    n_local = hi - lo
    stream = torch.cuda.current_stream()
    d = p.get("d", 0)

    if family == "kmeans":
        k = p["k"]
        x = ml.rng_units(n_local * d, seed=1, first_draw=lo * d, device=dev).view(n_local, d)
        mu0 = ml.rng_units(k * d, seed=1, first_draw=0, device=dev).view(k, d)  # first k rows of x
        prog = KMeansProgram(x, k, mu0, comm=comm, method=args.method)
        kernel_fn = lambda: ml.kmeans_step(x, prog.mu, prog.assign, prog.counts, prog.sums,  # noqa: E731
                                           method=args.method)
        if comm is None:   # one rank: the update fused into the combine launch (dlx_kmeans_iteration)
            kernel_fn = lambda: ml.kmeans_iteration(x, prog.mu, prog.assign, prog.counts,  # noqa: E731
                                                    prog.sums, method=args.method)

        def rest():   # allreduce + update (one fused launch with --comm peer)
            if comm is None:
                return
            if isinstance(comm, PeerComm):
                comm.kmeans_update_(prog.counts, prog.sums, prog.mu)
                return
            if comm is not None:
                comm.allreduce_many_([prog.counts, prog.sums])
            ml.kmeans_update(prog.counts, prog.sums, prog.mu)

        def step():
            kernel_fn()
            rest()
    elif family == "logreg":
        x = ml.rng_units(n_local * d, seed=1, first_draw=lo * d, device=dev).view(n_local, d)
        if p.get("storage") == "f32":
            x = x.float()   # the fp32-storage opt-in: rounded once, promoted exactly in the kernel
        y = ml.rng_ints(n_local, 2, seed=1, first_draw=n * d + lo, device=dev)
        prog = LogRegProgram(x, y, torch.zeros(d, dtype=torch.float64, device=dev), 1.0 / n, comm=comm)
        kernel_fn = lambda: ml.logreg_grad(x, y, prog.theta, prog.grad)  # noqa: E731

        def rest():
            if isinstance(comm, PeerComm):
                comm.bgd_step_(prog.grad, prog.theta, prog.alpha)
                return
            if comm is not None:
                comm.allreduce_(prog.grad)
            ml.axpy_inplace(prog.theta, prog.grad, prog.alpha)

        def step():
            kernel_fn()
            rest()
    elif family == "gda":
        x = ml.rng_units(n_local * d, seed=1, first_draw=lo * d, device=dev).view(n_local, d)
        y = ml.rng_ints(n_local, 2, seed=1, first_draw=n * d + lo, device=dev)
        holder = {}

        def kernel_fn():
            # one read of x (csrc/gda_dmma.cu single-pass fit); sharded: the ranks' fits pooled
            # through the exchange (gda_combine_ranks_kernel)
            holder["r"] = ml.gda(x, y, comm)

        def step():
            kernel_fn()
    else:
        K = p["K"]
        keys = ml.rng_ints(n_local, K, seed=1, first_draw=lo, device=dev)
        counts = torch.empty(K, dtype=torch.int64, device=dev)
        kernel_fn = lambda: ml.groupby_count(keys, K, counts)  # noqa: E731

        def step():
            kernel_fn()
            if comm is not None:
                comm.allreduce_(counts)

    # warm-up
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()

    sampler = ClockSampler(local_dev)
    sampler.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    L = _lib.load()

    # The step's launches are captured into CUDA graphs (one for the dominant kernel(s), one for
    # the exchange + update), so a launch-bound config (C1, C2) measures the GPU rather than the
    # Python dispatch of each launch.  Multi-rank NCCL exchanges stay eager.
    graphs = {}
    if family == "groupby":
        def rest():
            if comm is not None:
                comm.allreduce_(counts)
    if comm is None or isinstance(comm, PeerComm):
        if family in ("kmeans", "logreg", "groupby", "gda"):
            def cap(fn):
                side = torch.cuda.Stream()
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(side):
                    fn()
                torch.cuda.current_stream().wait_stream(side)
                g = torch.cuda.CUDAGraph()
                c0 = int(L.dlx_launch_count())
                with torch.cuda.graph(g):
                    fn()
                return g, int(L.dlx_launch_count()) - c0
            graphs["kernel"] = cap(kernel_fn)
            if family != "gda" and not (family == "kmeans" and comm is None):
                graphs["rest"] = cap(rest)
            torch.cuda.synchronize()
    run_kernel = (graphs["kernel"][0].replay if "kernel" in graphs else kernel_fn)
    run_rest = (graphs["rest"][0].replay if "rest" in graphs else (rest if family != "gda" else None))
    if family == "kmeans" and comm is None:
        run_rest = rest   # nothing left: the update ran inside the kernel graph's combine
    launches0 = int(L.dlx_launch_count())
    t_start.record(stream)
    for s in range(args.steps):
        ev[s][0].record(stream)
        # dominant kernel timed on its own stream with events around it
        if family in ("kmeans", "logreg", "groupby"):
            run_kernel()
            ev[s][1].record(stream)
            run_rest()   # remainder of the step (allreduce + update)
        else:
            ev2[s][0].record(stream)
            run_kernel()   # the single-pass fit: DMMA scatter + class sums, combines, finalize
            ev2[s][1].record(stream)
            ev[s][1].record(stream)
    t_end.record(stream)
    # this library's kernels in the timed region: counted at launch, or per captured graph
    # (the launches recorded while capturing) times its replays
    launches = int(L.dlx_launch_count()) - launches0 + args.steps * sum(nl for _, nl in graphs.values())
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    total_ms = t_start.elapsed_time(t_end)
    kern_ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    pass2_ms = sum(a.elapsed_time(b) for a, b in ev2) / args.steps if family == "gda" else 0.0
    if dist is not None:
        t = torch.tensor([total_ms, kern_ms, pass2_ms], dtype=torch.float64, device=_reduce_dev(dist, dev))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, kern_ms, pass2_ms = float(t[0]), float(t[1]), float(t[2])
    ms_per_step = total_ms / args.steps
    value = 1000.0 / ms_per_step

    pending = None
    if family == "kmeans" and args.method != 1:
        try:
            pending = ml.kmeans_last_recheck_count(n_local, d, p["k"]) / max(1, n_local)
        except Exception:
            pending = None

    # ---- end to end through the public API with host buffers ----------------------------------
    e2e = None
    e2e_family = None
    if args.no_e2e:
        pass   # A/B runs of kernel variants: the device-timed value only
    elif family == "kmeans":
        e2e_family = e2e_kmeans(args, p, n_local, lo, comm, dist, dev)
        # one GPU: the headline e2e is the reference-facing drop-in (dlx_program_execute) with
        # host buffers; sharded runs keep the family API's (the drop-in runs one device)
        e2e = e2e_dropin_kmeans(args, p, dev) if world == 1 else e2e_family
    elif family == "logreg":
        e2e = e2e_logreg(args, p, n_local, lo, comm, dist, dev)

    result = None
    if rank == 0:
        peak, peak_kind = measured_peaks()
        bytes_launch = algorithmic_bytes(family, p, n_local)
        achieved = bytes_launch / (kern_ms * 1e-3) / 1e9
        result = {
            "metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if family != "groupby" else "int64",
            "data": "synthetic (reference Rng LCG, seed 1, generated on device, bit-identical to host)",
            "config": {"workload": args.config, **p, "parallelism": f"sample-sharded dp{world}",
                       "exchange": None if world == 1 else ("peer-memory fused allreduce+update" if args.comm == "peer"
                                                            else "NCCL allReduce + update kernel"),
                       **({"update": "fused into the combine launch (dlx_kmeans_iteration)" if world == 1
                           else "after the exchange"} if family == "kmeans" else {}),
                       "l2": "inputs larger than L2 (no flush needed)" if bytes_launch > 256e6 else
                             "inputs L2-resident (launch-bound config)",
                       "method": {0: "auto", 1: "direct", 2: "screened"}[args.method],
                       "screen_recheck_fraction": pending},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(args.config),
                         "peak_kind": peak_kind, "kernel_ms": kern_ms,
                         "algorithmic_bytes_per_launch": bytes_launch},
            "e2e": e2e,
            "e2e_family_api": e2e_family,
            "gpu_launches": launches,
            "cuda_graphs": sorted(graphs),
            "clocks": clocks,
        }
        if family == "gda":
            # dominant kernel = the single-pass fit's first pass (pass 2 when sharded).  The int8
            # path (tcgen05 kind::i8 digit products, csrc/gda_dmma.cu gda_fit_i8_kernel) streams x
            # and y once and is HBM-paced: its roofline is the HBM line, with the tensor line in
            # executed int8 ops against the nominal dense int8 peak (not in MEASURED_PEAKS.json).
            # The DMMA path's roofline is the fp64 tensor line on algorithmic symmetric flops.
            nb = (d + 7) // 8
            flops = n_local * d * (d + 1)
            flops_executed = n_local * 2.0 * 64 * nb * (nb + 1) // 2
            hb = algorithmic_bytes(family, p, n_local) / (pass2_ms * 1e-3) / 1e9
            path = ml.gda_fit_path(x, y)
            hbm_line = {"bound": "hbm", "achieved": hb, "peak": peak, "unit": "GB/s",
                        "frac": hb / peak, "kernel_ms": pass2_ms}
            dmma_line = {"bound": "tensor", "achieved": flops / (pass2_ms * 1e-3) / 1e12,
                         "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": flops / (pass2_ms * 1e-3) / 1e12 / DMMA_PEAK_TFLOPS,
                         "peak_kind": DMMA_PEAK_KIND, "kernel_ms": pass2_ms,
                         "algorithmic_flops_per_launch": flops,
                         "executed_flops_per_launch": flops_executed,
                         "executed_frac": flops_executed / (pass2_ms * 1e-3) / 1e12 / DMMA_PEAK_TFLOPS}
            result["config"]["gda_path"] = ("single-pass fit" if comm is None else
                                            "single-pass fit per rank, pooled through the exchange")
            result["config"]["gda_kernel"] = path
            result["config"]["gda_fit_fallback"] = ml.gda_fit_last_fallback(x)
            if path == "int8":
                # 12 MMAs of 128 x 128 x 32 per 96-row tile: four group products x 3 K-steps
                ops = n_local / 96.0 * 12 * 2.0 * 128 * 128 * 32
                result["roofline"] = {**hbm_line, "traffic": ncu_traffic(args.config),
                                      "algorithmic_bytes_per_launch": algorithmic_bytes(family, p, n_local)}
                result["roofline_tensor_int8"] = {"bound": "tensor", "achieved": ops / (pass2_ms * 1e-3) / 1e12,
                                                  "peak": 4500.0, "unit": "TOP/s",
                                                  "frac": ops / (pass2_ms * 1e-3) / 1e12 / 4500.0,
                                                  "peak_kind": "nominal dense int8 = the fp8 figure of B200_PROFILING.md (unmeasured)",
                                                  "executed_ops_per_launch": ops}
                result["roofline_fp64_equivalent"] = dmma_line
            else:
                result["roofline_hbm"] = hbm_line
                result["roofline"] = {**dmma_line, "traffic": ncu_traffic(args.config)}
        if world == 1 and not args.no_cpu_baseline:
            try:
                result["cpu_baseline"] = (cpu_baseline_kmeans(p) if family == "kmeans"
                                          else cpu_baseline_generic(family, p))
            except Exception as exc:  # report, never fake
                result["cpu_baseline"] = {"value": None, "error": str(exc)}
    if comm is not None:
        comm.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return result


def _pipelined_jobs(stream, copy_stream, slots, h2d, compute, jobs):
    """Run `jobs` independent jobs with double-buffered inputs: job j's H2D (copy stream, into
    slot j % 2) overlaps job j-1's iterations; the compute stream waits for its slot's copy and
    the copy stream for the compute of job j-2 (the slot's previous user)."""
    import torch
    ev_in = [torch.cuda.Event() for _ in slots]
    ev_done = [torch.cuda.Event() for _ in slots]
    copy_stream.wait_stream(stream)
    for j in range(jobs):
        b = j % len(slots)
        with torch.cuda.stream(copy_stream):
            if j >= len(slots):
                copy_stream.wait_event(ev_done[b])
            h2d(slots[b])
            ev_in[b].record(copy_stream)
        stream.wait_event(ev_in[b])
        compute(slots[b])
        ev_done[b].record(stream)


def e2e_kmeans(args, p, n_local, lo, comm, dist, dev, iters_per_job=10):
    """One e2e step = one k-means job through the public API from HOST data: H2D of the
    (pinned) sample shard, `iters_per_job` iterations, D2H of assignments + centroids.
    Consecutive jobs are double-buffered on the device (job j+1's H2D overlaps job j's
    iterations), as a streaming caller would run them; every job's copies are in the timed
    region."""
    import torch

    from paper_1109_0778_b200 import multiloops as ml
    from paper_1109_0778_b200.programs import KMeansProgram
    d, k = p["d"], p["k"]
    slots = [torch.empty((n_local, d), dtype=torch.float64, device=dev) for _ in range(2)]
    ml.rng_units(n_local * d, seed=1, first_draw=lo * d, device=dev, out=slots[0].view(-1))
    x_host = torch.empty((n_local, d), dtype=torch.float64, pin_memory=True)
    x_host.copy_(slots[0])
    mu0_dev = ml.rng_units(k * d, seed=1, device=dev).view(k, d)
    a_host = torch.empty(n_local, dtype=torch.int32, pin_memory=True)
    mu_host = torch.empty((k, d), dtype=torch.float64, pin_memory=True)
    stream = torch.cuda.current_stream()
    copy_stream = torch.cuda.Stream(device=dev)
    jobs = max(2, min(4, args.steps // 3 or 1))

    def h2d(xd):
        xd.copy_(x_host, non_blocking=True)

    def compute(xd):
        prog = KMeansProgram(xd, k, mu0_dev, comm=comm, method=args.method)
        prog.run(iters_per_job)
        a_host.copy_(prog.assign, non_blocking=True)
        mu_host.copy_(prog.mu, non_blocking=True)

    _pipelined_jobs(stream, copy_stream, slots, h2d, compute, 2)  # warm-up
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    _pipelined_jobs(stream, copy_stream, slots, h2d, compute, jobs)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device=_reduce_dev(dist, dev))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    it_s = jobs * iters_per_job / (ms * 1e-3)
    del slots, x_host
    torch.cuda.empty_cache()
    return {"value": it_s, "unit": "it/s", "h2d_bytes_per_step": n_local * d * 8,
            "d2h_bytes_per_step": n_local * 4 + k * d * 8,
            "step": f"one job = H2D x shard (pinned) + {iters_per_job} iterations + D2H assignments and "
                    f"centroids; {jobs} jobs, double-buffered (H2D of job j+1 overlaps job j)",
            "iters_per_step": iters_per_job}


def e2e_dropin_kmeans(args, p, dev, iters_per_job=10, jobs=4):
    """e2e through the reference-facing drop-in (include/dlx_program.h): the staged k-means
    program of `iters_per_job` fused iterations (descriptors.kmeans_program, pinned statement by
    statement to the reference's own staging in tests/test_descriptors.py) executed with
    dlx_program_execute, its VectorRand source replaced by caller data in pinned HOST memory
    (dlx_program_input.h_data): every job copies the 8 GiB sample matrix to the device, runs the
    iterations (centroid updates on the device) and returns the printed text (assignment of
    row 0 and counts per iteration, every final centroid).  Two program handles on two host
    threads, as a streaming caller would run them: one job's upload overlaps the other's
    iterations.  Checked against SURVEY App. B (iteration-1 counts prefix)."""
    import threading

    import torch

    from paper_1109_0778_b200 import multiloops as ml
    from paper_1109_0778_b200.descriptors import kmeans_program
    from paper_1109_0778_b200.program import Program
    n, d, k = p["n"], p["d"], p["k"]
    desc = kmeans_program(n, d, k, iters_per_job)
    xsym = next(int(q) for q, st in desc["stmts"].items() if st["op"] == "VectorRand")
    x_host = torch.empty(n * d, dtype=torch.float64, pin_memory=True)
    x_host.copy_(ml.rng_units(n * d, seed=1, device=dev))
    torch.cuda.synchronize()
    progs = [Program(desc), Program(desc)]
    outs = [None, None]
    errs = []

    warm = threading.Barrier(3)
    go = threading.Barrier(3)

    def worker(t, njobs):
        # the warm-up job runs in the same thread as the timed ones: the executor's per-thread
        # streams, pinned staging and the allocator pool's blocks for this thread's streams are
        # set up there (a thread's first run maps its buffers), and every loop gets lowered once
        try:
            torch.cuda.set_device(dev)
            outs[t] = progs[t].run(seed=1, device=dev.index, inputs={xsym: x_host})
            torch.cuda.synchronize()
        except Exception as exc:   # reported, never hidden
            errs.append(repr(exc))
        warm.wait()
        go.wait()
        try:
            for _ in range(njobs):
                outs[t] = progs[t].run(seed=1, device=dev.index, inputs={xsym: x_host})
        except Exception as exc:
            errs.append(repr(exc))

    ths = [threading.Thread(target=worker, args=(t, jobs // 2)) for t in range(2)]
    for th in ths:
        th.start()
    warm.wait()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    go.wait()
    for th in ths:
        th.join()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    if errs:
        return {"value": None, "error": errs[0]}
    with open(os.path.join(ROOT, "tests", "golden", "appendix_b.json")) as f:
        gold = json.load(f)["c4_kmeans"]["counts_prefix"][0]
    lines = outs[0].output.split()
    ok = [int(v) for v in lines[1:5]] == gold if (n, d, k) == (16_777_216, 64, 64) else None
    launch = sorted({e["launch"] for e in outs[0].report})
    del x_host, progs
    torch.cuda.empty_cache()
    return {"value": jobs * iters_per_job / (ms * 1e-3), "unit": "it/s", "h2d_bytes_per_step": n * d * 8,
            "d2h_bytes_per_step": iters_per_job * (k * 8 + 4) + k * d * 8,
            "api": "dlx_program_execute (drop-in for interpret/executeDEG), host-buffer input",
            "step": f"one job = one staged program run: H2D of the pinned sample matrix + {iters_per_job} fused "
                    f"iterations ({', '.join(launch)}, centroid update on the device) + printed results; "
                    f"{jobs} jobs on 2 program handles / host threads (upload of one overlaps the other's iterations)",
            "iters_per_step": iters_per_job, "wall_ms": ms, "appendix_b_counts": ok}


def e2e_logreg(args, p, n_local, lo, comm, dist, dev, iters_per_job=20):
    import torch

    from paper_1109_0778_b200 import multiloops as ml
    from paper_1109_0778_b200.programs import LogRegProgram
    d, n = p["d"], p["n"]
    x0 = ml.rng_units(n_local * d, seed=1, first_draw=lo * d, device=dev).view(n_local, d)
    if p.get("storage") == "f32":
        x0 = x0.float()
    y0 = ml.rng_ints(n_local, 2, seed=1, first_draw=n * d + lo, device=dev)
    x_host = torch.empty_like(x0, device="cpu").pin_memory()
    y_host = torch.empty_like(y0, device="cpu").pin_memory()
    x_host.copy_(x0)
    y_host.copy_(y0)
    slots = [(x0, y0), (torch.empty_like(x0), torch.empty_like(y0))]
    th_host = torch.empty(d, dtype=torch.float64, pin_memory=True)
    stream = torch.cuda.current_stream()
    copy_stream = torch.cuda.Stream(device=dev)
    jobs = max(2, min(4, args.steps // 3 or 1))

    def h2d(xy):
        xy[0].copy_(x_host, non_blocking=True)
        xy[1].copy_(y_host, non_blocking=True)

    def compute(xy):
        prog = LogRegProgram(xy[0], xy[1], torch.zeros(d, dtype=torch.float64, device=dev), 1.0 / n, comm=comm)
        prog.run(iters_per_job)
        th_host.copy_(prog.theta, non_blocking=True)

    _pipelined_jobs(stream, copy_stream, slots, h2d, compute, 2)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    _pipelined_jobs(stream, copy_stream, slots, h2d, compute, jobs)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device=_reduce_dev(dist, dev))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    return {"value": jobs * iters_per_job / (ms * 1e-3), "unit": "it/s",
            "h2d_bytes_per_step": n_local * (d * x0.element_size() + 8), "d2h_bytes_per_step": d * 8,
            "step": f"one job = H2D x,y shard (pinned) + {iters_per_job} BGD iterations + D2H theta; "
                    f"{jobs} jobs, double-buffered (H2D of job j+1 overlaps job j)",
            "iters_per_step": iters_per_job}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="dlx", choices=["dlx", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--method", type=int, default=0, help="k-means: 0 auto, 1 direct fp64, 2 screened")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the e2e legs (kernel A/B runs)")
    ap.add_argument("--comm", default="peer", choices=["peer", "nccl"],
                    help="N>1 exchange: the fused peer-memory allreduce+update kernel (csrc/peer.cu, "
                         "ascending-rank fold), or NCCL allReduce + a separate update kernel")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    family, p, metric, unit = CONFIGS[args.config]
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        if rank != 0:
            return 0
        res = run_reference(args, family, dict(p), metric, unit)
        res["n_gpus"] = world
        print(json.dumps(res), flush=True)
        return 0
    res = run_dlx(args, family, dict(p), metric, unit, rank, world, local_rank)
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
