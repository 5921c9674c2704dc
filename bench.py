#!/usr/bin/env python
"""bench.py — exact kNN + LOF outlier scoring (TOD, arXiv 2110.14007) on B200.

One STEP = one pass of the whole hot path over one
synthetic dataset: prep/quantize -> tcgen05 fused distance + top-K' ->
fp64 re-rank + certificate -> fallback -> kNN scores -> LOF stage.

Default workload: BASELINE.json configs[2] "C3": kNN, n=1,000,000, d=64, k=10,
bf16 provable-quantization path, quoted on 1/2/4/8 B200 (the largest BASELINE
configuration quoted at one GPU).  It scales STRONGLY: the same n at every N,
query rows sharded (256-row aligned), and for N > 1 the sharded library path
(tod_knn_sharded) circulates the quantized reference blocks on an NCCL ring and
all-gathers the scores.  `--gpus N` launches N ranks itself (torch.distributed.run)
when not already under torchrun.  Other configs: --config c1 | c2 (kNN + LOF,
n=100,000, d=32, k=20) | c3f16 | c4 (n=10M, d=64, k=20: each GPU answers one
1/8 query shard, the whole job at N=8) | c5 | c5s | nwr.

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU oracle
(oracle/, the parity reference) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import platform
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (n, d, k, lof, fmt, description)
    "c1": (1_000, 10, 10, True, "auto", "C1: kNN outlier score n=1000 d=10 k=10"),
    "c2": (100_000, 32, 20, True, "auto", "C2: kNN+LOF n=100000 d=32 k=20"),
    "c3": (1_000_000, 64, 10, False, "bf16", "C3: kNN n=1000000 d=64 k=10 bf16 PQ path"),
    "c3f16": (1_000_000, 64, 10, False, "fp16", "C3 shape, fp16 PQ path"),
    "c5": (2_000_000, 512, 50, False, "fp16", "C5: kNN n=2000000 d=512 k=50 (tensor-bound regime)"),
    "c4": (10_000_000, 64, 20, False, "fp16",
           "C4: kNN n=10000000 d=64 k=20 (1/8 query shard per GPU; the whole job on 8 GPUs)"),
    "c5s": (500_000, 512, 50, False, "fp16", "C5 shape at n=500000 (1-GPU sample of C5)"),
    # NEXT-2: NWR on the C2-shaped data; phi = 12 on the squared
    # distance (86 % of rows have no neighbour, mean 39, max ~1900: the paper's
    # "preset distance threshold (usually a small number)")
    "nwr": (100_000, 32, 0, False, "fp16", "NWR (neighbours within range) n=100000 d=32 phi=12"),
}
NWR_PHI = 12.0
METRIC = "kNN/LOF queries/sec & dist-evals/sec at 1/2/4/8 B200; % of distance roofline"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return j.get("bf16_tflops"), j.get("bf16_tflops_sustained"), j.get("hbm_gbs"), "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev = dev
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self, t0, t1):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        inside = [l for ts, l in self.lines if t0 - 0.06 <= ts <= t1 + 0.06] or \
            [l for _, l in self.lines]
        sm, mx, reasons = [], [], set()
        for l in inside:
            parts = [p.strip() for p in l.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist_env():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def _workload(cfg_name, world):
    return CONFIGS[cfg_name]


def run_reference(args):
    """CPU oracle leg: bounded sample of the same workload on the host cores."""
    world, rank, _ = _dist_env()
    if rank != 0:
        return 0
    import datagen
    import oracle
    n, d, k, lof, fmt, desc = _workload(args.config, world)
    X = datagen.gaussian_mixture(n, d, seed=0)
    threads = oracle.num_threads()
    rng = np.random.default_rng(1)
    # calibrate the per-step row sample to ~args.ref_step_s seconds of work
    probe = rng.choice(n, min(n, 2 * threads), replace=False)
    t = time.perf_counter()
    oracle.knn(X, k, rows=probe)
    per_row = (time.perf_counter() - t) / len(probe)
    rows_per_step = int(max(threads, min(n, args.ref_step_s / max(per_row, 1e-9))))
    times = []
    for i in range(args.warmup + args.steps):
        rows = rng.choice(n, rows_per_step, replace=False)
        t = time.perf_counter()
        _, dd = oracle.knn(X, k, rows=rows)
        oracle.scores(dd)
        dt = time.perf_counter() - t
        if i >= args.warmup:
            times.append(dt)
    ms = 1e3 * float(np.mean(times))
    qps = rows_per_step / (ms / 1e3)
    sample = ("oracle kNN+scores on %d seeded query rows of n=%d per step (LOF stage on a full "
              "table is O(nk), excluded)" % (rows_per_step, n))
    line = {
        "impl": "reference", "metric": METRIC, "value": qps, "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak" if args.config == "c4" else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (Gaussian mixture + uniform outliers, seed 0)",
        "config": {"workload": desc, "n": n, "d": d, "k": k, "lof": lof},
        "dist_evals_per_s": qps * n,
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": threads, "kind": "oracle",
                         "sample": sample, "cpu": platform.processor() or platform.machine()},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(n, d, k, X, budget_s):
    import oracle
    threads = oracle.num_threads()
    rng = np.random.default_rng(1)
    probe = rng.choice(n, min(n, 2 * threads), replace=False)
    t = time.perf_counter()
    oracle.knn(X, k, rows=probe)
    per_row = (time.perf_counter() - t) / len(probe)
    rows = int(max(threads, min(n, budget_s / max(per_row, 1e-9))))
    sel = rng.choice(n, rows, replace=False)
    t = time.perf_counter()
    _, dd = oracle.knn(X, k, rows=sel)
    oracle.scores(dd)
    dt = time.perf_counter() - t
    return {"value": rows / dt, "unit": "queries/s", "cores": threads, "kind": "oracle",
            "sample": "oracle kNN+scores (fp64 brute force, full sort) on %d seeded query rows "
                      "of the same n=%d dataset, %.1f s" % (rows, n, dt)}


def _traffic(cfg_name):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get(cfg_name)
    return None


def run_gpu_nwr(args):
    """NWR leg (tod_nwr): one step = counts + CSR neighbour lists of all rows."""
    import torch
    import datagen
    import paper_2110_14007_b200 as tod
    n, d, _, _, fmt, desc = CONFIGS[args.config]
    X = datagen.gaussian_mixture(n, d, seed=0)
    Xd = torch.from_numpy(X).cuda()
    stream = torch.cuda.current_stream()
    ctx = tod.Context(device=torch.cuda.current_device(), fmt=fmt, flags=tod.F_TIMING,
                      stream=stream.cuda_stream)
    c, p, _, st = ctx.nwr(Xd, NWR_PHI, lists=False)
    cap = int(int(p[-1]) * 1.1) + 1024
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    # the clock sampler starts before the warm-up (it keeps only the samples inside
    # the timed window), so the GPU never idles between warm-up and timing
    sampler = ClockSampler(torch.cuda.current_device())
    sampler.start()
    for _ in range(args.warmup):
        ctx.nwr(Xd, NWR_PHI, capacity=cap)
    torch.cuda.synchronize()
    times, kms, stats = [], [], {}
    t0 = time.time()
    for i in range(args.steps):
        flush.fill_(float(i))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        counts, ptr, cols, stats = ctx.nwr(Xd, NWR_PHI, capacity=cap)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        kms.append(stats["ms_main_kernel"])
    t1 = time.time()
    clocks = sampler.stop(t0, t1)
    ms, km = float(np.mean(times)), float(np.mean(kms))
    # e2e: host buffers through the C ABI (H2D of X, D2H of counts/row_ptr/cols)
    Xh = torch.from_numpy(X).pin_memory()
    e2e = []
    for i in range(min(args.steps, 10)):
        flush.fill_(float(i))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ch, ph, lh, _ = ctx.nwr(Xh, NWR_PHI, capacity=cap)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e.append(e0.elapsed_time(e1))
    total = int(ptr[-1])
    peak_b, _, _, peak_src = _peaks()
    flops = 2.0 * n * n * d
    ach = flops / (km * 1e-3) / 1e12
    line = {"metric": "NWR queries/sec (neighbours within range, exact)", "value": n / (ms * 1e-3),
            "unit": "queries/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f16 operands/f32 accumulate (main pass), f64 verification",
            "data": "synthetic (Gaussian mixture + uniform outliers, seed 0)",
            "config": {"workload": desc, "n": n, "d": d, "phi": NWR_PHI, "pairs": total,
                       "l2": "flushed between steps (256 MiB write)"},
            "dist_evals_per_s": n * n / (ms * 1e-3),
            "roofline": {"bound": "tensor", "achieved": ach, "peak": peak_b, "unit": "TFLOP/s",
                         "frac": ach / peak_b, "traffic": None,
                         "kernel": {3: "k_knn_tc3", 4: "k_knn_tc4", 5: "k_knn_tc5"}.get(stats.get("main_kernel"), "?"),
                         "kernel_ms": km, "flops_per_launch": flops,
                         "peak_source": "%s bf16_tflops" % peak_src},
            "fallback_rows": stats.get("fallback_rows"),
            "e2e": {"value": n / (float(np.mean(e2e)) * 1e-3), "unit": "queries/s",
                    "h2d_bytes_per_step": n * d * 4,
                    "d2h_bytes_per_step": n * 8 + (n + 1) * 8 + total * 4},
            "gpu_launches": int(stats.get("kernel_launches", 0)) * args.steps,
            "clocks": clocks}
    print(json.dumps(line), flush=True)
    ctx.close()
    return 0


def _sharding(cfg_name, n, world, rank):
    """(q_begin, q_count, mode) of this rank's work.

    Strong scaling (every config but c4): the n rows are split over the world;
    world > 1 runs the NCCL ring (tod_knn_sharded / tod_lof_sharded).
    c4 (BASELINE configs[3], quoted on 8 GPUs): each rank answers its 1/8 query
    shard of the n = 10M job, so per-GPU work is fixed ("weak") and N=8 is the
    whole job on the ring; N < 8 runs ranks 0..N-1's shards, each against the
    full reference set resident on its GPU (the 1-GPU line measures exactly one
    rank's share of the target)."""
    from paper_2110_14007_b200 import dist as tdist
    if cfg_name == "c4":
        b, c = tdist.shard_rows(n, 8, rank)
        return b, c, ("ring" if world == 8 else "shard8")
    b, c = tdist.shard_rows(n, world, rank)
    return b, c, ("ring" if world > 1 else "single")


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import datagen
    import paper_2110_14007_b200 as tod
    from paper_2110_14007_b200 import dist as tdist

    world, rank, local = _dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.cuda.current_device()
    n, d, k, lof, fmt, desc = CONFIGS[args.config]
    if args.fmt:
        fmt = args.fmt
    if args.config == "c4" and world > 8:
        raise SystemExit("c4 is defined for up to 8 GPUs")
    qb, qc, mode = _sharding(args.config, n, world, rank)
    if args.loopback > 1:
        if world > 1:
            raise SystemExit("--loopback runs on one GPU")
        qb, qc, mode = 0, n, "loopback"
    X = datagen.gaussian_mixture(n, d, seed=0)
    stream = torch.cuda.current_stream()
    ctx = tod.Context(device=dev, fmt=fmt, flags=tod.F_TIMING, stream=stream.cuda_stream)
    if mode == "loopback":
        # the ring schedule of `args.loopback` virtual ranks on this one GPU
        # (collectives and block transfers become device copies): validates the
        # multi-GPU path at full size; NOT a multi-GPU throughput
        ctx.comm_init_loopback(args.loopback)
        Xl = torch.from_numpy(X).cuda()
        Xd = None
    elif mode == "ring":
        r_, w_ = tdist.init_comm(ctx)
        import ctypes
        ver = ctypes.c_int(0)
        try:
            ctypes.CDLL("libnccl.so.2").ncclGetVersion(ctypes.byref(ver))
        except Exception:
            pass
        print("[rank %d] NCCL communicator attached: world=%d, device cuda:%d, NCCL %d" %
              (r_, w_, dev, ver.value), file=sys.stderr, flush=True)
        Xl = torch.from_numpy(X[qb:qb + qc]).cuda()
        Xd = None
    else:
        Xd = torch.from_numpy(X).cuda()
        Xl = None
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    last = {}

    def step():
        if mode in ("ring", "loopback"):
            if lof:
                _, _, _, st = ctx.lof_sharded(Xl, n, qb, k)
            else:
                r, _, _ = ctx.knn_sharded(Xl, n, qb, k, want=())
                st = r.stats
        elif lof:
            _, _, _, st = ctx.lof(Xd, k)
        else:
            st = ctx.knn(Xd, k, qb, qc, want=("score_kth", "score_mean")).stats
        last.clear()
        last.update(st)

    # the clock sampler starts before the warm-up (it keeps only the samples inside
    # the timed window), so the GPU never idles between warm-up and timing
    sampler = ClockSampler(dev)
    sampler.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    main_ms, kern_ms, launches = [], [], []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.time()
    for i in range(args.steps):
        flush.fill_(float(i))               # L2 flush (256 MiB write) between steps, untimed
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
        main_ms.append(last.get("ms_main", 0.0))
        kern_ms.append(last.get("ms_main_kernel", 0.0))
        launches.append(last.get("kernel_launches", 0))
    torch.cuda.synchronize()
    t1 = time.time()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop(t0, t1)
    ms = float(np.mean([a.elapsed_time(b) for a, b in evs]))
    main, kmain = float(np.mean(main_ms)), float(np.mean(kern_ms))
    stats = dict(last)
    if world > 1:  # max over ranks of the device times
        t = torch.tensor([ms, main, kmain], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, main, kmain = float(t[0]), float(t[1]), float(t[2])

    # ---- e2e: the same step through the C ABI with HOST buffers (pinned): the
    # H2D of this rank's X and the D2H of the scores are inside the timed region
    e2e_ms = []
    if mode in ("ring", "loopback"):
        Xh = torch.from_numpy(X[qb:qb + qc]).pin_memory()
        h2d = qc * d * 4
        d2h = n * 4 * 2
    else:
        Xh = torch.from_numpy(X).pin_memory()
        h2d = n * d * 4
        d2h = (n * 4 * 4) if lof else (qc * 4 * 2)
    for i in range(args.warmup + min(args.steps, 10)):
        flush.fill_(float(i))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        if mode in ("ring", "loopback"):
            if lof:
                ctx.lof_sharded(Xh, n, qb, k)
            else:
                ctx.knn_sharded(Xh, n, qb, k, want=())
        elif lof:
            ctx.lof(Xh, k, want_knn=("score_kth", "score_mean"))
        else:
            ctx.knn(Xh, k, qb, qc, want=("score_kth", "score_mean"))
        e1.record(stream)
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e_ms.append(e0.elapsed_time(e1))
    e2e = float(np.mean(e2e_ms))
    if world > 1:
        t = torch.tensor([e2e], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = float(t[0])

    # queries answered by the whole job per step
    if args.config == "c4" and mode != "loopback":
        q_job = sum(tdist.shard_rows(n, 8, r)[1] for r in range(world))
    else:
        q_job = n
    if rank == 0:
        peak_b, peak_s, hbm, peak_src = _peaks()
        # Dominant kernel: the tensor-core main pass (k_knn_tc3 / k_knn_tc5 single-SM
        # or k_knn_tc4 CTA pairs), timed with CUDA events around its launch(es) on
        # the launching stream (the ring: around the W main-pass launches, which
        # also contain any wait for a block transfer).  Algorithmic work per
        # (query, reference) pair = 2d flops of the -2XY^T contraction (DESIGN.md
        # §7); the main pass covers every reference column (key-only sample) or
        # every column outside the sample tiles (list sample, d = 64 in one
        # process), for this rank's rows.
        rows = qc
        mk = stats.get("main_kernel", 0)
        if mk:
            tile = 256
            bt = (n + tile - 1) // tile
            samp_cols = sum(min(tile, n - tile * t) for t in range(0, bt, 8))
            if stats.get("sample_pass") == 2:   # key-only sample: main covers every tile
                samp_cols = 0
            pairs_main = rows * (n - samp_cols)
            kname = {3: "k_knn_tc3 (single-SM tcgen05 main pass)",
                     4: "k_knn_tc4 (CTA-pair tcgen05 cta_group::2 main pass)",
                     5: "k_knn_tc5 (single-SM tcgen05 main pass, 3-deep accumulator ring)"}[mk]
            kms = kmain
        else:
            pairs_main = rows * n
            kname = "k_knn_tc (tcgen05 fused distance + top-K')"
            kms = main
        flops = 2.0 * pairs_main * d          # algorithmic contraction flops per launch (per GPU)
        achieved = flops / (kms * 1e-3) / 1e12
        pass1_tf = 2.0 * rows * n * d / (main * 1e-3) / 1e12
        # peak: the sustained GEMM figure for a kernel that runs tens of ms inside a
        # long step, the burst figure for a short one (B200_PROFILING.md)
        long_kernel = kms >= 20.0
        peak = peak_s if long_kernel else peak_b
        qps = q_job / (ms * 1e-3)
        line = {
            "metric": METRIC, "value": qps, "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "weak" if args.config == "c4" else "strong",
            "vs_baseline": None,
            "dtype": "%s operands/f32 accumulate (pass 1), f64 re-rank" %
                     {1: "f16", 2: "bf16", 3: "f32"}.get(stats.get("format"), "?"),
            "data": "synthetic (Gaussian mixture + uniform outliers, seed 0)",
            "config": {"workload": desc, "n": n, "d": d, "k": k, "lof": lof,
                       "queries_per_step": q_job, "queries_this_rank": qc,
                       "format": stats.get("format"), "kprime": stats.get("kprime"),
                       "chunks": stats.get("chunks"),
                       "l2": "flushed between steps (256 MiB write)",
                       "parallelism": ("query-sharded dp%d, reference blocks on an NCCL ring" % world
                                       if mode == "ring" else
                                       "LOOPBACK: the %d-rank ring schedule run by %d virtual ranks "
                                       "on 1 GPU (validation, not a multi-GPU number)"
                                       % (args.loopback, args.loopback) if mode == "loopback" else
                                       "one rank's 1/8 query shard per GPU, references resident"
                                       if mode == "shard8" else "single GPU")},
            "dist_evals_per_s": qps * n,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak,
                         "frac_of_burst_peak": achieved / peak_b,
                         "traffic": _traffic(args.config),
                         "kernel": kname, "kernel_ms": kms, "flops_per_launch": flops,
                         "pass1": {"kernels": "sample + main", "ms": main,
                                   "achieved_tflops": pass1_tf, "frac": pass1_tf / peak},
                         "peak_source": "%s %s (fp16 dense rate = bf16 on B200)" %
                                        (peak_src, "bf16_tflops_sustained" if long_kernel
                                         else "bf16_tflops")},
            "phase_ms": {kk: stats.get(kk) for kk in
                         ("ms_prep", "ms_main", "ms_main_kernel", "ms_certify", "ms_fallback",
                          "ms_lof")},
            "candidates_per_row": {
                "staged_groups": stats.get("cand_groups", 0) / max(1, rows),
                "visited_groups": stats.get("visited_groups", 0) / max(1, rows),
                "kept_columns": stats.get("cand_columns", 0) / max(1, rows)},
            "certified_rows": stats.get("certified"),
            "fallback_rows": stats.get("fallback_rows"),
            "e2e": {"value": q_job / (e2e * 1e-3),
                    "unit": "queries/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e},
            "gpu_launches": int(sum(launches)),
            "clocks": clocks,
        }
        if not args.no_cpu and world == 1:
            line["cpu_baseline"] = cpu_baseline(n, d, k, X, args.cpu_budget_s)
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def _relaunch_distributed(args):
    """`--gpus N` without torchrun: start N ranks with torch.distributed.run."""
    import random
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node", str(args.gpus), "--master-addr", "127.0.0.1",
           "--master-port", str(random.randint(20000, 40000)), os.path.abspath(__file__)]
    cmd += [a for a in sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--fmt", default=None, choices=[None, "fp16", "bf16", "fp32", "auto"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=15.0)
    ap.add_argument("--ref-step-s", type=float, default=3.0)
    ap.add_argument("--loopback", type=int, default=0,
                    help="run the W-rank ring schedule as W virtual ranks on one GPU (validation)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _relaunch_distributed(args)
    if world != args.gpus and int(os.environ.get("RANK", "0")) == 0:
        print("bench.py: --gpus %d but WORLD_SIZE=%d; using %d ranks" % (args.gpus, world, world),
              file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "nwr":
        return run_gpu_nwr(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
