#!/usr/bin/env python
"""bench.py -- S_k(A) evals/s and TFLOP/s at d=4096 (BASELINE.json metric, configs[2]).

One step = one evaluation of S_k(A) through the C ABI (nseries_eval) on the headline plan:
config 3 (d=4096, fp64, spectrum [0, 0.995]), radix-15 x3 in the residual framework
(k=3375, 18 products in the paper's counting).  The same run also times the radix-9 x4
(k=6561) and binary x12 (k=4096) plans ("per_plan") for the wall-time ratio targets.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]

N > 1 (under torchrun): the single-matrix path does not shard (DESIGN.md "Multi-GPU:
replicas only"); each rank evaluates its own replica, value = all ranks' evals / max time.
--impl reference times the oracle (oracle/, long double, host cores) on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "S_k(A) evals/sec and TFLOP/s (% of FP64/TF32 tensor peak) at d=4096, per radix plan"
D = 4096
HEADLINE = ([15, 15, 15], 3375)
PLANS = {"x15^3": ([15, 15, 15], 3375), "x9^4": ([9, 9, 9, 9], 6561), "x2^12": ([2] * 12, 4096)}
# Roofline denominator for the FP64 tensor pipe: measured DMMA.8x8x4 register-loop peak on
# this pool's B200 (tools/peak_fp64.cu -> profiles/peaks_r01_fp64_microbench.json).
FP64_PEAK_TFLOPS = 37.161
FP64_PEAK_SOURCE = "measured: DMMA m8n8k4 register loop, tools/peak_fp64.cu (profiles/peaks_r01_fp64_microbench.json)"
# TF32 dense peak: measured bf16 burst (MEASURED_PEAKS.json, 1631.3 TF) x the guide's nominal
# tf32/bf16 ratio (1.1 / 2.25 PFLOP/s, B200_PROFILING.md) -- "of measured x nominal ratio"
TF32_PEAK_TFLOPS = 1631.3 * 1.1 / 2.25
# tcgen05 .kind::tf32 measured on this pool (tools/tcgen05_peak.cu, 4 s sustained, 148 CTAs x
# M128 N256 K8 from SMEM: 128.0 clk per MMA = the cycle floor; profiles/peaks_r02_tcgen05_tf32.json):
# 1116 TF/s with all-zero operands (1842 MHz), 916 TF/s with random operands -- the board's power
# cap holds the SM clock at ~1510 MHz when the tensor cores switch real data.  The random-operand
# figure is the sustained peak a real 3xTF32 GEMM can reach.
TCGEN05_TF32_PEAK_TFLOPS = 1116.4
TCGEN05_TF32_PEAK_RANDOM_TFLOPS = 916.4
# Legacy-path (mma.sync m16n8k8 .tf32) peak used by the batched small-matrix kernel: measured
# register loop, tools/mma_issue.cu (profiles/peaks_r01_mma_sync.txt)
MMA_SYNC_TF32_PEAK_TFLOPS = 275.7
REASONS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-per-plan", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the configs 1/2/4 side lines")
    ap.add_argument("--sharded-direct", action="store_true",
                    help="with --sharded: read right factors in place from the peers' arenas (CUDA IPC "
                         "over NVLink, NSERIES_SHARDED_DIRECT) instead of an allgather per product")
    ap.add_argument("--sharded", action="store_true",
                    help="NEXT-3: config 5 (d = 8192, k = 10000) row-sharded across the N ranks "
                         "(strong scaling; not the headline line)")
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = "clocks.sm,clocks.max.sm," + ",".join(f"clocks_event_reasons.{r}" for r in REASONS)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 2 + len(REASONS):
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max(float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit())
        reasons = sorted({REASONS[i] for r in self.rows for i in range(len(REASONS))
                          if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


from paper_2602_11843_b200 import replicas as R  # noqa: E402  (host plumbing, no method arithmetic)


def dist_setup(n):
    return R.setup(n)


def barrier(world):
    R.barrier(world)


def max_over_ranks(x, world):
    return R.max_over_ranks(x, world)


# ------------------------------------------------------------------ oracle (CPU) legs

def oracle_sample(A_np, steps, n_cols=1):
    """Time the oracle (as it stands) on n_cols probe columns of the workload; returns
    (seconds per column, threads)."""
    import numpy as np
    from oracle import oracle as O
    from paper_2602_11843_b200 import inputs
    V, _ = inputs.probe_block(A_np.shape[0], 2, n_unit=n_cols, n_gauss=0)
    t0 = time.perf_counter()
    if 15 in steps:
        O.plan_apply(A_np, steps, V)
    else:
        k = 1
        for s in steps:
            k = k + 1 if s == 1 else k * s
        O.series_sum(A_np, k, V)
    return (time.perf_counter() - t0) / n_cols, O.num_threads()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np
    from paper_2602_11843_b200 import inputs
    A_np = inputs.cfg3(D, device="cpu")[0] if not _cuda_ok() else inputs.cfg3(D, device="cuda")[0].cpu().numpy()
    steps, k = HEADLINE
    for _ in range(args.warmup):
        oracle_sample(A_np, steps)
    times = []
    threads = 1
    for _ in range(args.steps):
        t, threads = oracle_sample(A_np, steps)
        times.append(t)
    per_col = sum(times) / len(times)
    per_eval = per_col * D
    value = 1.0 / per_eval
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_col * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f80 (x87 long double)",
        "data": "synthetic",
        "config": {"workload": "cfg3 d=4096 spectrum[0,0.995] radix-15x3 k=3375", "d": D, "k": k, "plan": "x15^3"},
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads, "kind": "oracle",
                         "sample": "per step: oracle C-2 (compositional Horner, 4912 long-double matvecs) on 1 of "
                                   "4096 columns; evals/s = 1/(seconds per column x 4096)"},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


# ------------------------------------------------------------------ native leg

def time_plan(P, h, A, S, steps, k, n_steps, n_warm, flags, stream, world):
    import torch
    plan = P.nseries_plan_finalize(steps, k, flags)
    for _ in range(n_warm):
        P.nseries_eval(h, A, D, k, plan=plan, S=S, flags=flags, stream=stream)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(n_steps):
        P.nseries_eval(h, A, D, k, plan=plan, S=S, flags=flags, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    ms = e0.elapsed_time(e1)
    st = P.nseries_last_stats(h)
    return max_over_ranks(ms, world), plan, st


def run_native(args):
    import numpy as np
    import torch
    rank, world, local = dist_setup(args.gpus)
    import paper_2602_11843_b200 as P
    P.load_library()
    from paper_2602_11843_b200 import inputs
    torch.cuda.set_device(local)
    h = P.nseries_create(local)
    A, _, _ = inputs.cfg3(D, seed=2, device="cuda")
    A = A.contiguous()
    S = torch.empty_like(A)
    stream = torch.cuda.current_stream()
    steps, k = HEADLINE
    flags = P.NSERIES_ALLOW_APPROX
    flop_per_product = 2.0 * D ** 3

    with ClockSampler(local) as clk:
        ms, plan, st = time_plan(P, h, A, S, steps, k, args.steps, max(args.warmup, 3), flags, stream, world)
    clocks = clk.summary()
    ms_step = ms / args.steps
    evals_per_s = R.aggregate_rate(args.steps, ms, world)
    tflops = plan.products * flop_per_product / (ms_step * 1e-3) / 1e12

    per_plan = {}
    if not args.no_per_plan:
        for name, (stp, kk) in PLANS.items():
            fl = P.NSERIES_ALLOW_APPROX if 15 in stp else 0
            n = max(2, args.steps // 2)
            pms, pplan, _ = time_plan(P, h, A, S, stp, kk, n, 2, fl, stream, world)
            pstep = pms / n
            per_plan[name] = {"k": kk, "products": pplan.products, "ms_per_eval": pstep,
                              "evals_per_s": world * 1e3 / pstep,
                              "tflops": pplan.products * flop_per_product / (pstep * 1e-3) / 1e12}
        # NSERIES_SYMMETRIC (config 3's A is symmetric): same products, upper-triangle tiles only
        for name, (stp, kk) in PLANS.items():
            fl = (P.NSERIES_ALLOW_APPROX if 15 in stp else 0) | P.NSERIES_SYMMETRIC
            n = max(2, args.steps // 2)
            pms, pplan, _ = time_plan(P, h, A, S, stp, kk, n, 2, fl, stream, world)
            pstep = pms / n
            per_plan[name + " fp64 symmetric"] = {
                "k": kk, "products": pplan.products, "ms_per_eval": pstep, "evals_per_s": world * 1e3 / pstep,
                "tflops_dense_equivalent": pplan.products * flop_per_product / (pstep * 1e-3) / 1e12,
                "tflops_executed": pplan.products * flop_per_product * _sym_fraction(D) / (pstep * 1e-3) / 1e12}
        b = per_plan["x2^12"]
        for name in ("x15^3", "x9^4"):
            p = per_plan[name]
            p["time_ratio_vs_binary"] = p["ms_per_eval"] / b["ms_per_eval"]
            p["target_ratio"] = (p["products"] / b["products"]) / 0.95
        # fp32 (3xTF32 on tcgen05) on fl32(A): same plans, tensor-pipe rate = 3 x algorithmic
        A32 = A.float().contiguous()
        S32 = torch.empty_like(A32)
        # The fp32 plans run under the board power cap, whose state drifts over seconds: the three
        # plans are timed in 3 interleaved rounds (x15^3, x9^4, x2^12, x15^3, ...) and each plan
        # reports the median round, so the ratios compare plans under the same power state.
        n = max(2, args.steps // 2)
        rounds = {name: [] for name in PLANS}
        with ClockSampler(local) as fclk:
            for _ in range(3):
                for name, (stp, kk) in PLANS.items():
                    fl = P.NSERIES_ALLOW_APPROX if 15 in stp else 0
                    pms, pplan, _ = time_plan(P, h, A32, S32, stp, kk, n, 2, fl, stream, world)
                    rounds[name].append((pms / n, pplan.products))
        fclocks = fclk.summary()
        for name, (stp, kk) in PLANS.items():
            fl = P.NSERIES_ALLOW_APPROX if 15 in stp else 0
            times = sorted(t for t, _ in rounds[name])
            pstep, products = times[len(times) // 2], rounds[name][0][1]
            alg = products * flop_per_product / (pstep * 1e-3) / 1e12
            per_plan[name + " fp32"] = {"k": kk, "products": products, "ms_per_eval": pstep,
                                        "ms_per_eval_rounds": [t for t, _ in rounds[name]],
                                        "timing": f"median of 3 interleaved rounds of {n} evals",
                                        "evals_per_s": world * 1e3 / pstep, "tflops": alg,
                                        "tf32_tensor_tflops": 3 * alg,
                                        "tf32_frac_of_peak": 3 * alg / TF32_PEAK_TFLOPS,
                                        "tf32_frac_of_measured_tcgen05_peak": 3 * alg / TCGEN05_TF32_PEAK_TFLOPS,
                                        "tf32_frac_of_measured_tcgen05_peak_random_operands":
                                            3 * alg / TCGEN05_TF32_PEAK_RANDOM_TFLOPS,
                                        "clocks": fclocks}
            with ClockSampler(local) as sclk:
                sms, _, _ = time_plan(P, h, A32, S32, stp, kk, max(4, args.steps), 2, fl | P.NSERIES_SYMMETRIC,
                                      stream, world)
            sstep = sms / max(4, args.steps)
            per_plan[name + " fp32 symmetric"] = {
                "k": kk, "products": products, "ms_per_eval": sstep, "evals_per_s": world * 1e3 / sstep,
                "tflops_dense_equivalent": products * flop_per_product / (sstep * 1e-3) / 1e12,
                "clocks": sclk.summary()}
        bf = per_plan["x2^12 fp32"]
        for name in ("x15^3", "x9^4"):
            p = per_plan[name + " fp32"]
            p["time_ratio_vs_binary"] = p["ms_per_eval"] / bf["ms_per_eval"]
            p["target_ratio"] = (p["products"] / bf["products"]) / 0.95
        del A32, S32

    configs = None
    if world == 1 and not args.no_configs:
        configs = other_configs(P, h, stream)
    batch_slices = batched_slice_leg(P, h, stream, rank, world, args)

    # e2e: same metric through the C ABI with HOST buffers (pinned), copies inside the timed region
    # (NSERIES_HOST_ASYNC: the calls are pipelined -- matrix i+1's copy-in overlaps evaluation
    # i, S_i's copy-out overlaps the trailing product -- every step still moves its A in and
    # its S out; two host buffer pairs alternate as a streaming caller would use them)
    A_hosts = [A.cpu().pin_memory() for _ in range(2)]
    S_hosts = [torch.empty_like(A_hosts[0]).pin_memory() for _ in range(2)]
    plan = P.nseries_plan_finalize(steps, k, flags)
    hflags = flags | P.NSERIES_HOST_ASYNC
    for i in range(2):
        P.nseries_eval_host(h, A_hosts[i], D, k, plan=plan, S=S_hosts[i], flags=hflags, stream=stream)
    P.nseries_host_sync(h)
    barrier(world)
    n_e2e = max(2, args.steps // 2)
    t0 = time.perf_counter()
    for i in range(n_e2e):
        P.nseries_eval_host(h, A_hosts[i % 2], D, k, plan=plan, S=S_hosts[i % 2], flags=hflags, stream=stream)
    P.nseries_host_sync(h)
    e2e_s = max_over_ranks(time.perf_counter() - t0, world)
    e2e_val = world * n_e2e / e2e_s

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        A_np = A.cpu().numpy()
        n_cols = 2   # ~10-20 s of CPU work
        per_col, threads = oracle_sample(A_np, steps, n_cols=n_cols)
        cpu = {"value": 1.0 / (per_col * D), "unit": "evals/s", "cores": threads, "kind": "oracle",
               "sample": f"oracle C-2 (compositional Horner, 4912 long-double matvecs) on {n_cols} of {D} columns "
                         f"({per_col * n_cols:.1f} s); evals/s = 1/(s per column x {D})"}

    roof = {"bound": "tensor", "achieved": tflops, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": tflops / FP64_PEAK_TFLOPS, "traffic": _traffic(),
            "kernel": "gemm_f64_kernel<128,128,16,64,32,4> (DMMA.8x8x4)",
            "algorithmic_flops_per_launch": flop_per_product,
            "note": "achieved = 2 d^3 per GEMM launch / average launch duration over the timed region "
                    "(every launch in the step is this kernel); peak " + FP64_PEAK_SOURCE}
    line = {
        "metric": METRIC, "value": evals_per_s, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg3 d=4096 fp64, A = Q diag(1-lam) Q^T, lam~U[0.005,1] (seed 2); radix-15x3 residual plan k=3375",
                   "d": D, "k": k, "plan": "x15^3", "products": plan.products,
                   "parallelism": "replicas" if world > 1 else "single",
                   "l2": "inputs larger than L2 (A 128 MiB + ~1 GiB workspace per eval > 126 MB L2)"},
        "tflops": tflops, "products": plan.products,
        "roofline": roof, "cpu_baseline": cpu,
        "e2e": {"value": e2e_val, "unit": "evals/s", "h2d_bytes_per_step": D * D * 8,
                "d2h_bytes_per_step": D * D * 8, "api": "nseries_eval_host (NSERIES_HOST_ASYNC, pinned host buffers)"},
        "gpu_launches": st["launches"] * args.steps,
        "clocks": clocks,
        "per_plan": per_plan,
        "configs": configs,
        "cfg4_batch_slices": batch_slices,
    }
    P.nseries_destroy(h)
    if rank == 0:
        print(json.dumps(line), flush=True)
    R.teardown(world)
    return 0


def _sym_fraction(d, bm=128):
    """Fraction of the dense tile work the symmetric mode executes (tiles on/above the diagonal)."""
    nt = -(-d // bm)
    return (nt * (nt + 1) / 2) / (nt * nt)


def _time_evals(fn, n, n_warm, stream):
    import torch
    for _ in range(n_warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(n):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def other_configs(P, h, stream):
    """Side measurements on BASELINE.json configs 1, 2 and 4 (device-resident inputs, CUDA events
    on the launching stream).  Not the headline; parity for each is in tests/."""
    import torch
    from paper_2602_11843_b200 import inputs
    out = {}
    # config 1: d = 64 fp64 single matrix (latency; whole plan in one single-CTA launch)
    A = torch.from_numpy(inputs.cfg1()).cuda()
    S = torch.empty_like(A)
    for name, (stp, kk) in {"x9^2": ([9, 9], 81), "x2^6": ([2] * 6, 64), "x5^3": ([5] * 3, 125)}.items():
        plan = P.nseries_plan_finalize(stp, kk, 0)
        ms = _time_evals(lambda: P.nseries_eval(h, A, 64, kk, plan=plan, S=S, stream=stream), 200, 20, stream)
        out.setdefault("cfg1_d64_fp64", {})[name] = {"k": kk, "products": plan.products, "us_per_eval": ms * 1e3,
                                                   "launches": P.nseries_last_stats(h)["launches"]}
    # config 2: d = 1024 fp64
    A = torch.from_numpy(inputs.cfg2()).cuda()
    S = torch.empty_like(A)
    for name, (stp, kk) in {"x9^3": ([9] * 3, 729), "x5^4": ([5] * 4, 625), "x2^9": ([2] * 9, 512),
                            "x2^10": ([2] * 10, 1024)}.items():
        plan = P.nseries_plan_finalize(stp, kk, 0)
        ms = _time_evals(lambda: P.nseries_eval(h, A, 1024, kk, plan=plan, S=S, stream=stream), 20, 3, stream)
        out.setdefault("cfg2_d1024_fp64", {})[name] = {
            "k": kk, "products": plan.products, "ms_per_eval": ms,
            "tflops": plan.products * 2.0 * 1024 ** 3 / (ms * 1e-3) / 1e12,
            "frac_of_fp64_peak": plan.products * 2.0 * 1024 ** 3 / (ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS}
    # config 4: 16384 x 32^2 fp32 batched (one launch per batch)
    Ab = torch.from_numpy(inputs.cfg4()).cuda()
    Sb = torch.empty_like(Ab)
    B, d = Ab.shape[0], Ab.shape[1]
    for name, (stp, kk) in {"x9^2": ([9, 9], 81), "x5^2": ([5, 5], 25)}.items():
        plan = P.nseries_plan_finalize(stp, kk, 0)
        ms = _time_evals(lambda: P.nseries_eval_batched_strided(h, Ab, d * d, B, d, kk, plan=plan, S=Sb,
                                                                stream=stream), 20, 3, stream)
        alg = plan.products * 2.0 * d ** 3 * B / (ms * 1e-3) / 1e12
        out.setdefault("cfg4_batched_16384x32x32_fp32", {})[name] = {
            "k": kk, "products_per_matrix": plan.products, "us_per_batch": ms * 1e3,
            "matrices_per_s": B / (ms * 1e-3), "hbm_gbs": 2 * B * d * d * 4 / (ms * 1e-3) / 1e9,
            "hbm_frac": 2 * B * d * d * 4 / (ms * 1e-3) / 1e9 / 6533.5,
            "alg_tflops": alg, "tf32_tensor_tflops": 3 * alg,
            "frac_of_mma_sync_tf32_peak": 3 * alg / MMA_SYNC_TF32_PEAK_TFLOPS}
    # config 5: d = 8192 fp64, arbitrary k = 10000 through the AUTO mixed-radix plan
    A = inputs.cfg5(device="cuda")
    S = torch.empty_like(A)
    fl = P.NSERIES_ALLOW_APPROX
    plan = P.nseries_plan_build(10000, P.NSERIES_PLAN_AUTO, [15, 9, 5, 2], fl)
    ms = _time_evals(lambda: P.nseries_eval(h, A, 8192, 10000, plan=plan, S=S, flags=fl, stream=stream), 2, 1, stream)
    tf = plan.products * 2.0 * 8192 ** 3 / (ms * 1e-3) / 1e12
    out["cfg5_d8192_fp64_k10000"] = {"plan": list(plan.step[:plan.n_steps]),
                                      "products": plan.products, "ms_per_eval": ms, "tflops": tf,
                                      "frac_of_fp64_peak": tf / FP64_PEAK_TFLOPS}
    # the paper's own Table 3 workload (d = 500, normal A, fp64): ms per method
    # on this GPU beside the paper's CPU times (context only) and the normal
    # residual ||I - (I - A) S||_F of the returned S (the paper's accuracy column)
    import numpy as np
    A3, _, _ = inputs.table3_matrix()
    A3t = torch.from_numpy(A3).cuda()
    S3 = torch.empty_like(A3t)
    rows3 = [("binary", [2] * 7, 128, 8), ("binary", [2] * 9, 512, 10), ("quinary", [5] * 3, 125, 8),
             ("quinary", [5] * 4, 625, 10), ("radix-9", [9, 9], 81, 9), ("radix-9", [9] * 3, 729, 13),
             ("radix-15", [15, 15], 225, 18), ("radix-15", [15] * 3, 3375, 25)]
    t3 = []
    for meth, stp, kk, paper_ms in rows3:
        fl = P.NSERIES_ALLOW_APPROX if 15 in stp else 0
        plan3 = P.nseries_plan_finalize(stp, kk, fl)
        ms3 = _time_evals(lambda: P.nseries_eval(h, A3t, 500, kk, plan=plan3, S=S3, flags=fl, stream=stream), 50, 5,
                          stream)
        Sn = S3.cpu().numpy()
        res = float(np.linalg.norm(np.eye(500) - Sn + A3 @ Sn))
        t3.append({"method": meth, "k": kk, "products": plan3.products, "ms": ms3, "paper_cpu_ms": paper_ms,
                   "normal_residual": res})
    out["paper_table3_d500_fp64"] = t3
    del A3t, S3
    # NEXT-3 row-sharded chain, config 5 in 8 row blocks, all on this GPU (device-copy gathers):
    # the per-rank kernels of an 8-GPU run (1024 x 8192 x 8192 GEMMs) executed back to back
    n = 8
    blocks = [P.nseries_shard_rows(8192, n, s) for s in range(n)]
    As = [A[r0:r0 + m].contiguous() for r0, m in blocks]
    del S
    Ss = [torch.empty_like(a) for a in As]
    ms8 = _time_evals(lambda: P.nseries_eval_sharded(h, As, 0, n, 8192, 10000, plan=plan, S_shards=Ss, flags=fl,
                                                     stream=stream), 1, 1, stream)
    st = P.nseries_last_stats(h)
    out["next3_sharded_cfg5_8blocks_1gpu"] = {
        "blocks": n, "rows_per_block": blocks[0][1], "ms_per_eval": ms8, "gathers": st["gathers"],
        "gathers_prefetched": st["gathers_prefetched"],
        "gathered_bytes_per_eval": st["gathers"] * 8192 * 8192 * 8,
        "overhead_vs_dense": ms8 / ms - 1.0,
        "note": "all row blocks on one GPU; an 8-rank run executes 1/8 of these launches per GPU plus "
                "NCCL allgather-v gathers (not measurable on this 1-GPU box)"}
    # the same with NSERIES_SHARDED_DIRECT: right factors read in place from the 8 row blocks
    msd = _time_evals(lambda: P.nseries_eval_sharded(h, As, 0, n, 8192, 10000, plan=plan, S_shards=Ss,
                                                     flags=fl | P.NSERIES_SHARDED_DIRECT, stream=stream),
                      1, 1, stream)
    st = P.nseries_last_stats(h)
    out["next3_sharded_cfg5_8blocks_1gpu_direct"] = {
        "blocks": n, "ms_per_eval": msd, "gathers": st["gathers"], "overhead_vs_dense": msd / ms - 1.0,
        "note": "NSERIES_SHARDED_DIRECT: each GEMM's k-tile loads read the right factor's row blocks in "
                "place (no gather, no full copy)"}
    del A, As, Ss
    return out


def batched_slice_leg(P, h, stream, rank, world, args):
    """Config 4 across the ranks: the 16384 matrices split into contiguous
    batch slices, one per rank, each evaluated by one nseries_eval_batched_strided launch; no
    collective on the data path (barrier + max-over-ranks timing only).  Strong scaling: the
    batch is fixed, value = 16384 matrices / the slowest rank's time per batch."""
    import torch
    from paper_2602_11843_b200 import inputs
    Ab = inputs.cfg4()                                   # same seeded batch on every rank
    n, d = Ab.shape[0], Ab.shape[1]
    b0, b1 = R.batch_slice(n, world, rank)
    A = torch.from_numpy(Ab[b0:b1]).cuda()
    S = torch.empty_like(A)
    plan = P.nseries_plan_finalize([9, 9], 81, 0)
    m = b1 - b0
    run = lambda: P.nseries_eval_batched_strided(h, A, d * d, m, d, 81, plan=plan, S=S, stream=stream)
    for _ in range(max(args.warmup, 3)):
        run()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    n_it = max(10, args.steps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(n_it):
        run()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    ms = max_over_ranks(e0.elapsed_time(e1) / n_it, world)
    counts = R.gather_counts(m, world, device="cuda" if world > 1 else "cpu")
    return {"metric": "matrices/s", "value": n / (ms * 1e-3), "unit": "matrices/s", "n_gpus": world,
            "scaling": "strong", "ms_per_batch": ms, "plan": "x9^2 k=81 fp32", "batch": n,
            "matrices_per_rank": counts, "collectives_on_data_path": 0,
            "hbm_gbs_aggregate": 2 * n * d * d * 4 / (ms * 1e-3) / 1e9,
            "note": "contiguous batch slices per rank (replicas.batch_slice), one launch per rank per batch"}


def _traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu capture (or None)."""
    p = os.path.join(ROOT, "profiles", "ncu_gemm_f64_traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p)).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


def run_sharded(args):
    """One A (config 5) split into N row blocks, one per rank, gathers over NCCL (NEXT-3)."""
    import torch
    import torch.distributed as dist
    # NCCL's own per-rank INIT lines (rank, channels, ring / NVLS / P2P transport choice) are
    # printed to stderr: file descriptor 1 points at stderr until the one JSON line is printed
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    sys.stdout.flush()
    saved_stdout = os.dup(1)
    os.dup2(2, 1)
    rank, world, local = dist_setup(args.gpus)
    import paper_2602_11843_b200 as P
    from paper_2602_11843_b200 import inputs
    torch.cuda.set_device(local)
    h = P.nseries_create(local)
    d, k = 8192, 10000
    uid = [P.nseries_comm_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0)
    P.nseries_comm_init(h, uid[0], world, rank)
    A = inputs.cfg5(device="cuda")
    r0, rows = P.nseries_shard_rows(d, world, rank)
    A_blk = A[r0:r0 + rows].contiguous()
    del A
    S_blk = torch.empty_like(A_blk)
    fl = P.NSERIES_ALLOW_APPROX
    plan = P.nseries_plan_build(k, P.NSERIES_PLAN_AUTO, [15, 9, 5, 2], fl)
    if args.sharded_direct:
        # right factors read in place from the owners' arenas over NVLink (CUDA IPC), one-int
        # all-reduce barrier per op, instead of an allgather per product
        from paper_2602_11843_b200 import replicas
        fl |= P.NSERIES_SHARDED_DIRECT
        need = P.nseries_sharded_arena_bytes(d, world, 1, k, plan, flags=fl)
        P.nseries_peer_import(h, replicas.exchange_blobs(P.nseries_peer_export(h, need), world))
    stream = torch.cuda.current_stream()
    run = lambda: P.nseries_eval_sharded(h, [A_blk], rank, world, d, k, plan=plan, S_shards=[S_blk], flags=fl,
                                         stream=stream)
    for _ in range(max(args.warmup, 1)):
        run()
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = max(1, args.steps // 5)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(n):
        run()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1), world) / n
    st = P.nseries_last_stats(h)
    sys.stdout.flush()
    os.dup2(saved_stdout, 1)
    os.close(saved_stdout)
    if rank == 0:
        tf = plan.products * 2.0 * d ** 3 / (ms * 1e-3) / 1e12
        print(json.dumps({
            "metric": "S_k(A) evals/sec, one config-5 matrix row-sharded over the ranks (NEXT-3)",
            "value": 1e3 / ms, "unit": "evals/s", "n_gpus": world, "steps": n, "warmup": max(args.warmup, 1),
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": "cfg5 d=8192 k=10000 AUTO plan, row-sharded",
                                           "d": d, "k": k, "plan": list(plan.step[:plan.n_steps]),
                                           "products": plan.products, "parallelism": f"row-shard{world}"},
            "tflops": tf, "frac_of_fp64_peak_per_gpu": tf / world / FP64_PEAK_TFLOPS,
            "gathers": st["gathers"], "gathers_prefetched": st["gathers_prefetched"],
            "right_factors": "in place over NVLink (NSERIES_SHARDED_DIRECT)" if args.sharded_direct
            else "NCCL allgather-v per product",
            "nccl_log": "stderr (NCCL_DEBUG=INFO, SUBSYS=INIT)"}))
    P.nseries_destroy(h)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.sharded:
        return run_sharded(args)
    return run_native(args)


if __name__ == "__main__":
    sys.exit(main())
