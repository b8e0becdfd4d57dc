#!/usr/bin/env python
"""Newton steps/s at dimension 1024 (eval + diff + MGS least squares + update)
on B200, per BASELINE.json: F(1024, 1024, 32) random sparse system (SURVEY
8(d)), complex quad double by default (--base d/dd/qd).

One JSON line on rank 0.  `value` is device-resident throughput (inputs in
HBM, CUDA events on the launching stream, max over ranks); `e2e` is the same
step through the C ABI with host buffers (h2d of x, d2h of x_next, f, dx and
the norms inside the timed region).  Multi-GPU runs are independent replicas
(a single system does not shard); `value` sums them.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Newton steps/sec (eval+diff+MGS) at dim 1024 in complex d/dd/qd; quality-up ratio"
R_ADD = {1: 1, 2: 20, 4: 87}   # FP64 instructions of a real add
R_MUL = {1: 1, 2: 9, 4: 185}   # ... of a real multiply with FMA two_prod


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--base", default="qd", choices=["d", "dd", "qd"])
    ap.add_argument("--dim", type=int, default=1024)
    ap.add_argument("--terms", type=int, default=1024)
    ap.add_argument("--k", type=int, default=32)
    ap.add_argument("--rows", type=int, default=None, help="equations m (default = dim)")
    ap.add_argument("--seed", type=int, default=2024)
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of CPU baseline work")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--batch", type=int, default=0,
                    help="config C5: number of homotopy start points (use with --dim 256 --terms 256 --base dd)")
    ap.add_argument("--max-iters", type=int, default=8)
    ap.add_argument("--converge", action="store_true",
                    help="config C4: run_newton to convergence (homotopy start t=0.99 when square; planted "
                         "solution t=1 with x0 = z(1+1e-6u) when --rows > --dim)")
    return ap.parse_args()


def level_costs(nc: int, cplx: bool):
    radd, rmul = R_ADD[nc], R_MUL[nc]
    if cplx:
        return {"add": 2 * radd, "mul": 4 * rmul + 2 * radd, "int": 2 * rmul, "radd": radd, "rmul": rmul}
    return {"add": radd, "mul": rmul, "int": rmul, "radd": radd, "rmul": rmul}


def committed_traffic(kernel: str, workload: str):
    """DRAM bytes per launch of `kernel` on `workload` from the newest
    committed ncu capture (profiles/*/traffic.json), or None."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "traffic.json")), reverse=True):
        try:
            with open(path) as f:
                rec = json.load(f).get(f"{kernel} | {workload}")
        except (OSError, ValueError):
            continue
        if rec:
            return rec["dram_read_bytes"] + rec["dram_write_bytes"]
    return None


def work_counts(stats, nc: int, cplx: bool, m: int, n: int, split: bool = False):
    """Algorithmic FP64 instruction counts and bytes of one step."""
    c = level_costs(nc, cplx)
    w_eval = (stats.mul_ops * c["mul"] + stats.int_mul_ops * c["int"] + stats.add_ops * c["add"]
              + stats.table_mul_ops * c["mul"])
    U = m * n * (n + 1) // 2                      # MGS update elements
    w_factor = (U * (2 * c["mul"] + 2 * c["add"])    # r_kj dot + a -= q r
                + (2 * n + 1) * m * (2 * c["rmul"] + 2 * c["radd"]) // (1 if cplx else 2)  # norms
                + n * m * (2 if cplx else 1) * c["rmul"])                                   # q = a / r
    w_bsub = n * (n - 1) // 2 * (c["mul"] + c["add"])                                       # back-sub
    es = nc * (2 if cplx else 1)
    b_eval = (stats.support * 8 + (stats.monomials + 1) * 4 + stats.monomials * es * 8
              + (n + m) * es * 8 + m * n * es * 8)
    if split:
        return w_eval, w_factor, w_bsub, b_eval
    return w_eval, w_factor + w_bsub, b_eval


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port (oracle/pn_oracle.c) on a bounded sample

def cpu_step_estimate(args, packed, x_planes, budget: float):
    """Seconds of one full Newton step of the oracle, from a timed row sample
    of the evaluation and a smaller MGS (cubic extrapolation)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    threads = os.cpu_count() or 1
    L = oracle.Level(packed.level.base, packed.level.cplx)
    csr = oracle.CSR.from_packed(packed)
    m, n = packed.n_eqs, packed.n_vars
    # evaluation: rows are independent (evaldiff.py:252-265)
    rows = max(1, threads)
    sub = csr.rows(range(rows)).canonical()
    t0 = time.perf_counter()
    oracle.evaluate(L, sub, x_planes, nthreads=threads, canonical=True)
    t_rows = time.perf_counter() - t0
    reps = 1
    if t_rows < budget * 0.3:
        more = int(min(m, rows * max(1, (budget * 0.4) / max(t_rows, 1e-3))))
        if more > rows:
            sub = csr.rows(range(more)).canonical()
            t0 = time.perf_counter()
            oracle.evaluate(L, sub, x_planes, nthreads=threads, canonical=True)
            t_rows = time.perf_counter() - t0
            rows = more
    del reps
    t_eval = t_rows * m / rows
    # MGS: s x s sample, scaled by m n^2
    s = 64
    rng = np.random.default_rng(1)
    while True:
        aug = np.ascontiguousarray(rng.uniform(-1, 1, L.cshape + (s, s + 1)))
        t0 = time.perf_counter()
        oracle.least_squares(L, aug, nthreads=threads)
        t_s = time.perf_counter() - t0
        if t_s > budget * 0.15 or s >= min(m, n):
            break
        s = min(min(m, n), s * 2)
    t_mgs = t_s * (m * n * (n + 1)) / (s * s * (s + 1))
    sample = (f"oracle/pn_oracle.c (-O2, OpenMP {threads} threads): evaluation of {rows} of {m} rows "
              f"({t_rows:.2f} s, scaled x{m / rows:.1f}) + MGS least squares {s}x{s} ({t_s:.2f} s, scaled by "
              f"m*n^2 x{(m * n * (n + 1)) / (s * s * (s + 1)):.0f}); extrapolated")
    return t_eval + t_mgs, threads, sample, {"eval_s": t_eval, "mgs_s": t_mgs}


def quality_up(args, gpu_step_s: float, budget: float = 6.0):
    """SURVEY 8(d) quality-up ratio: seconds of a complex double-double
    Newton step at dimension 512 on the CPU over seconds of this run's
    complex quad-double step at dimension 1024 on the GPU.  The CPU side is
    the oracle port (C, all host threads, sampled and extrapolated like
    cpu_baseline); the reference's own Python path, which the survey timed at
    341.9 s for that step, cannot run on the GPU box."""
    from paper_1402_2626_b200.generators import random_sparse_system
    from paper_1402_2626_b200.xprec import precision_level
    level = precision_level("dd", True)
    packed = random_sparse_system(512, 512, 32, level, seed=args.seed)
    rng = np.random.default_rng(args.seed + 1)
    x = rng.uniform(0.5, 2.0, level.cshape + (512,)) * rng.choice([-1.0, 1.0], level.cshape + (512,))
    x[:, 1:] = 0.0
    t_cpu, cores, sample, parts = cpu_step_estimate(args, packed, np.ascontiguousarray(x), budget)
    return {"value": t_cpu / gpu_step_s, "cpu_s": t_cpu, "gpu_s": gpu_step_s, "cores": cores,
            "definition": "T_cpu(complex dd step, F(512,512,32)) / T_gpu(complex qd step, F(1024,1024,32))",
            "cpu": "oracle port " + sample}


# ---------------------------------------------------------------------------

def build_inputs(args, rank=0):
    from paper_1402_2626_b200.generators import random_sparse_system
    from paper_1402_2626_b200.xprec import precision_level
    level = precision_level(args.base, True)
    m = args.rows or args.dim
    # every rank solves its own system (independent units)
    packed = random_sparse_system(args.dim, args.terms, args.k, level, seed=args.seed + rank, m=m)
    rng = np.random.default_rng(args.seed + 1)
    x = rng.uniform(0.5, 2.0, level.cshape + (args.dim,)) * rng.choice([-1.0, 1.0], level.cshape + (args.dim,))
    x[:, 1:] = 0.0  # level.from_float values (SURVEY 8(d) random_point)
    return level, packed, np.ascontiguousarray(x)


def run_reference(args):
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    level, packed, x = build_inputs(args)
    cfg = {"workload": f"F({args.dim},{args.terms},{args.k}) complex {args.base} Newton step "
                       f"{args.rows or args.dim}x{args.dim}", "m": args.rows or args.dim, "n": args.dim,
           "terms_per_poly": args.terms, "k": args.k, "precision": f"complex {args.base}"}
    per_step_budget = max(3.0, args.cpu_budget / max(1, args.steps + args.warmup))
    times = []
    for i in range(args.warmup + args.steps):
        t, cores, sample, parts = cpu_step_estimate(args, packed, x, per_step_budget)
        if i >= args.warmup:
            times.append(t)
    t = statistics.median(times)
    v = 1.0 / t
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "steps/s", "n_gpus": 0, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": v, "unit": "steps/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "phases_s": parts}))


def run_ours(args):
    import torch
    world, rank, local = dist_setup()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    from paper_1402_2626_b200 import _lib
    from paper_1402_2626_b200.evaldiff import PreparedSystem

    lib = _lib.load()
    _lib.require_gpu()
    level, packed, x_host = build_inputs(args, rank)
    m, n = packed.n_eqs, packed.n_vars
    es, nc = level.es, level.ncomp
    t_prep = time.perf_counter()
    prep = PreparedSystem(packed)
    t_prep = time.perf_counter() - t_prep
    stats = prep.stats()
    w_eval, w_factor, w_bsub, b_eval = work_counts(stats, nc, level.cplx, m, n, split=True)
    w_mgs = w_factor + w_bsub

    dev = torch.device("cuda", torch.cuda.current_device())
    x_d = torch.from_numpy(x_host).to(dev)
    outs = {k: torch.empty(s, dtype=torch.float64, device=dev) for k, s in
            [("xn", (es, n)), ("f", (es, m)), ("dx", (es, n)), ("fm", (nc, m)), ("dm", (nc, n)), ("xm", (nc, n))]}
    info = _lib.NumInfo()
    stream = torch.cuda.current_stream().cuda_stream

    def step():
        rc = lib.pn_newton_step(prep.handle, _lib.ptr(x_d), _lib.ptr(outs["xn"]), _lib.ptr(outs["f"]),
                                _lib.ptr(outs["dx"]), _lib.ptr(outs["fm"]), _lib.ptr(outs["dm"]),
                                _lib.ptr(outs["xm"]), ctypes.byref(info), ctypes.c_void_p(stream))
        _lib.check(rc, info)
        return info.t_evaluate, info.t_solve, info.t_update, info.t_factor

    peak = ctypes.c_double(0)
    _lib.check(lib.pn_fp64_peak(ctypes.byref(peak), ctypes.c_void_p(stream)))
    fp64_peak = peak.value

    for _ in range(args.warmup):
        step()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev.index)
    clocks.start()
    launches0 = _lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    phases = []
    e0.record()
    for _ in range(args.steps):
        phases.append(step())
    e1.record()
    torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    clk = clocks.stop()
    elapsed = e0.elapsed_time(e1) / 1e3
    gather_s = None
    if world > 1:
        t = torch.tensor([elapsed], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        elapsed = float(t.item())
        # the one collective of the batched path: gather every system's x_next
        g0 = time.perf_counter()
        gathered = [torch.empty_like(outs["xn"]) for _ in range(world)]
        torch.distributed.all_gather(gathered, outs["xn"])
        torch.cuda.synchronize()
        gather_s = time.perf_counter() - g0
        torch.distributed.barrier()
    sec_step = elapsed / args.steps
    value = world * args.steps / elapsed

    # end to end through the C ABI with host buffers (pinned)
    ke = args.e2e_steps or max(2, min(args.steps, 5))
    pin = lambda shape: torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()
    xh = pin((es, n))
    xh[...] = x_host.reshape(es, n)
    ho = {k: pin(tuple(v.shape)) for k, v in outs.items()}

    def step_host():
        rc = lib.pn_newton_step(prep.handle, _lib.ptr(xh), _lib.ptr(ho["xn"]), _lib.ptr(ho["f"]),
                                _lib.ptr(ho["dx"]), _lib.ptr(ho["fm"]), _lib.ptr(ho["dm"]), _lib.ptr(ho["xm"]),
                                ctypes.byref(info), ctypes.c_void_p(stream))
        _lib.check(rc, info)

    step_host()
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record()
    for _ in range(ke):
        step_host()
    e3.record()
    torch.cuda.synchronize()
    e2e_elapsed = e2.elapsed_time(e3) / 1e3
    if world > 1:
        t = torch.tensor([e2e_elapsed], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_elapsed = float(t.item())
    h2d = xh.nbytes
    d2h = sum(v.nbytes for v in ho.values())

    t_eval = statistics.median(p[0] for p in phases)
    t_solve = statistics.median(p[1] for p in phases)
    t_upd = statistics.median(p[2] for p in phases)
    t_fac = statistics.median(p[3] for p in phases)
    mgs_rate = w_factor / t_fac
    workload = f"F({args.dim},{args.terms},{args.k}) complex {args.base} {m}x{n}"
    # the schedule mgs.cu's mgs_mode picks by default for this shape
    mgs_kernel = ("k_mgs_flow" if nc == 4 else
                  "k_mgs_pipe" if m % 256 == 0 and m <= 1024 else "k_mgs_dataflow")
    roofline = {"bound": "fp64", "kernel": f"{mgs_kernel} (MGS factorisation of [J | -f], one launch per step)",
                "achieved": mgs_rate / 1e12, "peak": fp64_peak / 1e12, "unit": "T FP64-instr/s",
                "frac": mgs_rate / fp64_peak, "traffic": committed_traffic(mgs_kernel, workload),
                "peak_source": "measured in-run DFMA probe (pn_fp64_peak); MEASURED_PEAKS.json has no FP64 entry",
                "work_fp64_instr": w_factor, "seconds": t_fac,
                "arithmetic_ceiling_frac": {4: 0.76, 2: 0.95}.get(nc)}
    bsub = {"kernel": "k_backsub_look" if nc == 4 else "k_backsub_blocked_look", "seconds": t_solve - t_fac,
            "work_fp64_instr": w_bsub, "bound": "latency (n dependent divisions)"}
    evalr = {"kernel": "k_mono_tree + k_segments (eval+diff phase)", "seconds": t_eval,
             "achieved_fp64": w_eval / t_eval / 1e12, "frac_fp64": w_eval / t_eval / fp64_peak,
             "achieved_gbs": b_eval / t_eval / 1e9, "work_fp64_instr": w_eval, "bytes": b_eval}

    cpu = None
    quality = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        t_cpu, cores, sample, parts = cpu_step_estimate(args, packed, x_host, args.cpu_budget)
        cpu = {"value": 1.0 / t_cpu, "unit": "steps/s", "cores": cores, "kind": "port", "sample": sample,
               "phases_s": parts}
        if args.base == "qd" and args.dim == 1024 and args.rows is None:
            quality = quality_up(args, sec_step)

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": sec_step * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"F({args.dim},{args.terms},{args.k}) complex {args.base} Newton step "
                                   f"{m}x{n} (eval+diff+MGS+update), x fixed per step",
                       "m": m, "n": n, "terms_per_poly": args.terms, "k": args.k,
                       "precision": f"complex {args.base}", "parallelism": f"replicas{world}",
                       "l2": "inputs larger than L2 (supports + contributions > 126 MB per step)"},
            "e2e": {"value": world * ke / e2e_elapsed, "unit": "steps/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "roofline": roofline,
            "eval_roofline": evalr,
            "backsub": bsub,
            "phases_ms": {"evaluate": t_eval * 1e3, "solve": t_solve * 1e3, "update": t_upd * 1e3},
            "cpu_baseline": cpu,
            "clocks": clk,
            "prepare_s": t_prep,
            "gather_s": gather_s,
        }
        if cpu:
            out["quality_up_same_precision"] = value / cpu["value"]
        if quality:
            out["quality_up"] = quality
        print(json.dumps(out))
    if world > 1:
        torch.distributed.destroy_process_group()


def run_batched(args):
    """Config C5: B independent homotopy Newton runs of one F(dim, terms, k)
    system sharded across ranks (no collective on the data path), one
    all_gather of status / iterations / final x at the end."""
    import torch
    world, rank, local = dist_setup()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method="tcp://127.0.0.1:29512", rank=0, world_size=1)
    from paper_1402_2626_b200 import _lib
    from paper_1402_2626_b200.batch import gather_batch, homotopy_batch, run_newton_batch, shard_range
    from paper_1402_2626_b200.evaldiff import PreparedSystem
    from paper_1402_2626_b200.generators import random_sparse_system
    from paper_1402_2626_b200.xprec import precision_level

    level = precision_level(args.base, True)
    B = args.batch
    packed = random_sparse_system(args.dim, args.terms, args.k, level, seed=args.seed)
    rng = np.random.default_rng(args.seed + 7)
    theta = rng.uniform(0.0, 2.0 * math.pi, (B, args.dim))
    Z = np.zeros(level.cshape + (B, args.dim))
    Z[0, 0] = np.cos(theta)
    Z[1, 0] = np.sin(theta)
    lo, hi = shard_range(B, world, rank)
    Zs = np.ascontiguousarray(Z[..., lo:hi, :])
    t = level.from_float(0.99)
    system, consts = homotopy_batch(packed, Zs, t)
    prep = PreparedSystem(system)
    lib = _lib.load()
    import ctypes
    peak = ctypes.c_double(0)
    _lib.check(lib.pn_fp64_peak(ctypes.byref(peak), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    # warm-up: one iteration of the whole shard (sizes every slot buffer), then the timed run
    for _ in range(max(1, args.warmup)):
        run_newton_batch(prep, Zs, consts, max_iters=1)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    launches0 = _lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = run_newton_batch(prep, Zs, consts, max_iters=args.max_iters)
    e1.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = _lib.launch_count() - launches0
    elapsed = e0.elapsed_time(e1) / 1e3
    it_local = int(res.iters.sum())
    tt = torch.tensor([elapsed, float(it_local)], dtype=torch.float64,
                      device="cuda" if world > 1 else "cpu")
    if world > 1:
        mx = tt.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = tt.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        elapsed, total_iters = float(mx[0]), int(sm[1])
    else:
        total_iters = it_local
    g0 = time.perf_counter()
    full = gather_batch(res, B)
    gather_s = time.perf_counter() - g0
    # FP64 roofline of the whole run: every start-iteration is one evaluation
    # plus one MGS least-squares solve of the (m x n) system
    w_eval, w_mgs, _ = work_counts(prep.stats(), level.ncomp, level.cplx, system.n_eqs, system.n_vars)
    achieved = total_iters * (w_eval + w_mgs) / elapsed / 1e12
    fp64_peak = peak.value / 1e12
    if rank == 0:
        counts = {name: int((full.status == code).sum()) for code, name in
                  [(0, "converged"), (1, "max_iters"), (2, "breakdown"), (3, "singular")]}
        print(json.dumps({
            "metric": "batched Newton iterations/sec (start-iterations, eval+diff+MGS), config C5",
            "value": total_iters / elapsed, "unit": "start-iterations/s", "n_gpus": world, "steps": 1,
            "warmup": 1, "ms_per_step": elapsed * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C5: {B} homotopy starts of F({args.dim},{args.terms},{args.k}) complex "
                                   f"{args.base}, t=0.99, max_iters={args.max_iters}",
                       "starts": B, "starts_per_gpu": hi - lo, "parallelism": f"start-sharded x{world}",
                       "collective": "one all_gather (status, iterations, x) after the run"},
            "status": counts, "mean_iters": float(full.iters.mean()) if B else 0.0,
            "gather_s": gather_s, "gpu_launches": launches, "clocks": clk,
            "roofline": {"bound": "fp64", "kernel": "k_solve_batch + k_mono_tree + k_segments (whole run)",
                         "achieved": achieved, "peak": fp64_peak * world, "unit": "T FP64-instr/s",
                         "frac": achieved / (fp64_peak * world), "traffic": None,
                         "peak_source": "measured in-run DFMA probe (pn_fp64_peak), per GPU x n_gpus",
                         "work_fp64_instr_per_start_iteration": w_eval + w_mgs}}))
    dist.destroy_process_group()


def run_converge(args):
    """Config C4: full Gauss-Newton (run_newton, newton.py:106-132) on the
    device-resident step until the reference's tolerance is met."""
    import torch
    torch.cuda.set_device(0)
    from paper_1402_2626_b200 import _lib
    from paper_1402_2626_b200.batch import homotopy_batch
    from paper_1402_2626_b200.evaldiff import PreparedSystem
    from paper_1402_2626_b200.generators import random_sparse_system
    from paper_1402_2626_b200.newton import NewtonConfig, run_newton
    from paper_1402_2626_b200.xprec import precision_level

    _lib.require_gpu()
    level = precision_level(args.base, True)
    n = args.dim
    m = args.rows or n
    packed = random_sparse_system(n, args.terms, args.k, level, seed=args.seed, m=m)
    rng = np.random.default_rng(args.seed + 3)
    theta = rng.uniform(0.0, 2.0 * math.pi, n)
    z = np.zeros(level.cshape + (n,))
    z[0, 0], z[1, 0] = np.cos(theta), np.sin(theta)
    planted = m > n
    t = level.from_float(1.0 if planted else 0.99)
    t0 = time.perf_counter()
    system, consts = homotopy_batch(packed, z[..., None, :], t)
    # bake the start's constants into the system (B = 1 batch helper does the shift on the GPU)
    from paper_1402_2626_b200.polyrep import PackedSystem
    coef = system.coeffs.reshape(level.es, -1).copy()
    ks = np.diff(system.mon_ptr)
    for i in range(m):
        lo, hi = system.poly_ptr[i], system.poly_ptr[i + 1]
        c = lo + int(np.nonzero(ks[lo:hi] == 0)[0][0])
        coef[:, c] = consts.reshape(level.es, m)[:, i]
    shifted = PackedSystem(level, n, system.poly_ptr, system.mon_ptr, system.var_idx, system.exps,
                           np.ascontiguousarray(coef.reshape(system.coeffs.shape)))
    del packed, system
    prep = PreparedSystem(shifted)
    t_setup = time.perf_counter() - t0
    x0 = z.copy()
    if planted:
        x0[0, 0] *= 1.0 + 1e-6 * rng.uniform(-1, 1, n)
        x0[1, 0] *= 1.0 + 1e-6 * rng.uniform(-1, 1, n)
    cfg = NewtonConfig(level=level, max_iters=args.max_iters)
    run_newton(prep, x0, NewtonConfig(level=level, max_iters=1))  # warm-up (first-touch allocations)
    torch.cuda.synchronize()
    clocks = ClockSampler(0)
    clocks.start()
    w0 = time.perf_counter()
    tr = run_newton(prep, x0, cfg)
    wall = time.perf_counter() - w0
    clk = clocks.stop()
    gpu_s = tr.timings["evaluate"] + tr.timings["solve"] + tr.timings["update"]
    print(json.dumps({
        "metric": "Gauss-Newton run to convergence (config C4)", "value": wall, "unit": "s",
        "higher_is_better": False, "n_gpus": 1, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"F({n},{args.terms},{args.k}) complex {args.base}, {m}x{n}, "
                               + ("planted solution t=1, x0=z(1+1e-6u)" if planted else "homotopy start t=0.99, x0=z"),
                   "m": m, "n": n},
        "iterations": len(tr.entries), "converged": tr.converged,
        "f_norm": [e.f_norm for e in tr.entries], "dx_norm": [e.dx_norm for e in tr.entries],
        "gpu_seconds": gpu_s, "ms_per_step": 1e3 * gpu_s / max(1, len(tr.entries)),
        "phases_s": tr.timings, "setup_s": t_setup, "clocks": clk}))


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.converge:
        run_converge(args)
    elif args.batch:
        run_batched(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
