#!/usr/bin/env python
"""bench.py -- QMC paths/s with price+delta+vega+gamma (d=64) on 1..8 B200.

Contract (task statement + BASELINE.json):
  python bench.py --gpus N --steps K --warmup W            (N > 1 under torchrun)
  python bench.py --impl reference ...                     (the oracle on host cores)
prints ONE JSON line on rank 0.

Workload: BASELINE.json configs[3] = SURVEY.md C4 -- arithmetic Asian, binary
Asian and lookback calls fused on the same paths, S0 = K = 100, sigma = 0.2,
r = 0.1, T = 1, d = 64, Brownian bridge + W(t_1) conditioning (the paper's
QMC+BB-CPW), 2^20 Sobol' points x 64 randomisations PER GPU (weak scaling: N
GPUs price 64 N replicates; rank g owns replicates [64 g, 64 g + 64)).

A step = one full estimator run: randomisation tables, the fused path kernel
over every cell, per-replicate reduction, one NCCL all-reduce (N > 1), the
device->host read of the replicate sums and the host finalize.  value =
underlying QMC paths (points x replicates, each delivering the 4 outputs of
all 3 options) per second over all ranks, timed with CUDA events on the
launching stream, max over ranks; L2 is flushed (256 MiB write) before every
timed step, outside the events.
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "QMC paths/sec with price+delta+vega+gamma (d=64) at 1/2/4/8 B200; % FP64 roof"
UNIT = "paths/s"
SM_COUNT = 148
FP64_LANES_PER_SM = 64          # FP64 FMA lanes per SM per clock (B200)
SM_MAX_MHZ_FALLBACK = 1965.0    # B200_PROFILING.md / MEASURED_PEAKS.json sm_max_mhz


def fp64_model_per_path(d, constr, cond, n_opt, arith_x1=0, n_lookback_x1=0):
    """Algorithmic FP64 lane-instructions per underlying path (SURVEY.md 8(d)
    planning model, fixed constants -- independent of how the kernel is written):
    c_icdf = 50 (branch-light FP64 inverse normal), c_exp = 17, c_tail = 160
    per option (log + 2 erfc + exp + ~30 FMA), c_W = 1 (STD) / 2 (BB) / d (PCA).
    X1: 4 Newton passes per arithmetic / binary option (SURVEY's count); under STD all
    dates share one slope, so the threshold is closed-form and one pass replaces the four
    (reading 19); a lookback under X1 has a closed-form threshold and one
    envelope pass instead (row f1)."""
    c_icdf, c_exp, c_tail = 50, 17, 160
    c_w = {0: 1, 1: 2, 2: d, 3: d}[constr]  # GPCA: a rotated PCA matrix, same dense contraction
    d_icdf = d - 1 if (cond == 1 or constr == 0) else d
    if cond == 0:
        return d_icdf * c_icdf + d * (c_exp + c_w + 6) + n_opt * c_tail
    newton = (1 if constr == 0 else 4) * d * (c_exp + 3)
    n_newton = n_opt - n_lookback_x1
    return (d_icdf * c_icdf + d * c_w + n_newton * (newton + d * (c_exp + 3) + c_tail)
            + n_lookback_x1 * (d * (c_exp + 3) + c_tail) + arith_x1 * d * (c_exp + 60 + 4))


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """SM clocks + throttle reasons sampled in-process through NVML every 100 ms
    during the timed region (no nvidia-smi subprocesses: they contend for the
    driver lock and would perturb the timed launches)."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._th = None
        self.nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None

    def _run(self):
        while not self._stop.is_set():
            try:
                sm = self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM)
                rs = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, rs))
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        if self.nvml is not None:
            self._th = threading.Thread(target=self._run, daemon=True)
            self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._th:
            self._th.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        reasons = sorted({n for _, rs in self.samples for n, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median([s for s, _ in self.samples]), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "source": "nvml"}


def cpu_baseline_oracle(options, d, constr, cond, budget_s=12.0):
    """The oracle (plain C, never tuned) on this host's cores, on a bounded
    sample of the same workload: replicates 0..R-1 x the first n points."""
    import oracle as O
    cores = os.cpu_count() or 1
    opts = [(t, 100.0) for t in options]
    mk = O.market(W.S0, W.R, W.SIGMA, W.T, d)
    cfg = O.config(construction=constr, conditioning=cond, seed=W.SEED)
    reps = max(1, min(64, cores))
    t0 = time.perf_counter()
    O.price_greeks(opts, mk, 256, reps, cfg, n_threads=cores)
    pilot = (time.perf_counter() - t0) / (256 * reps)
    n = int(max(256, min(1 << 20, budget_s / max(pilot, 1e-9) / reps)))
    t0 = time.perf_counter()
    O.price_greeks(opts, mk, n, reps, cfg, n_threads=cores)
    dt = time.perf_counter() - t0
    return {"value": n * reps / dt, "unit": UNIT, "cores": min(cores, reps), "kind": "oracle",
            "sample": f"C4 replicates 0..{reps - 1} x first {n} Sobol' points, {len(options)} options fused, "
                      f"d={d}, {dt:.1f} s wall on {min(cores, reps)} threads"}


def run_reference(args):
    """--impl reference: the oracle as it stands, on the host cores, same metric/config."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle as O
    c = W.CONFIGS[W.HEADLINE]
    options, d = c["options"], c["d"]
    cores = os.cpu_count() or 1
    reps = max(1, min(64, cores))
    opts = [(t, 100.0) for t in options]
    mk = O.market(W.S0, W.R, W.SIGMA, W.T, d)
    cfg = O.config(construction=W.BB, conditioning=W.W1, seed=W.SEED)
    n = 4096
    for _ in range(args.warmup):
        O.price_greeks(opts, mk, 512, reps, cfg, n_threads=cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.price_greeks(opts, mk, n, reps, cfg, n_threads=cores)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = n * reps * args.steps / tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Sobol'/Philox; no datasets)",
            "config": {"workload": "C4: arith+binary+lookback Asian calls fused, d=64, BB-W1 (QMC+BB-CPW)",
                       "sample_per_step": f"{reps} replicates x {n} points", "global_batch": n * reps,
                       "seq_len": d, "parallelism": "host threads"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": min(cores, reps), "kind": "oracle",
                             "sample": f"{reps} replicates x {n} points per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--construction", type=int, default=W.BB)
    ap.add_argument("--conditioning", type=int, default=W.W1)
    ap.add_argument("--randomization", type=int, default=0,
                    help="0 LMS + digital shift (default), 1 shift, 3 none, 4 nested Owen scrambling (row f4)")
    ap.add_argument("--workload", default="C4", choices=["C4", "C5"],
                    help="C4: 3 exotics fused, d=64 (the BASELINE metric); C5: 1024-option portfolio, d=128")
    ap.add_argument("--method", type=int, default=0,
                    help="0 QMC-CPW (default), 1 LR+MC (STD), 2 MC-CPW, 3 MC+AV-CPW (STD/BB, W1; row f2)")
    ap.add_argument("--options", default=None, help="comma-separated option types (0 arith, 1 binary, 2 lookback)")
    ap.add_argument("--points", type=int, default=None)
    ap.add_argument("--reps-per-gpu", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2209_11337_b200 as q
    from paper_2209_11337_b200.distributed import DistributedPricer

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    if args.workload == "C5":
        port = W.c5_portfolio()
        options, d = [o["type"] for o in port], 128
        args.construction, args.conditioning = W.PCA, W.W1
        N = args.points or (1 << 18)
        L = (args.reps_per_gpu or 16) * world
        plist = [q.params(S0=o["S0"], K=o["K"], r=o["r"], sigma=o["sigma"], T=o["T"], d=d) for o in port]
    else:
        c = W.CONFIGS[W.HEADLINE]
        options, d = c["options"], c["d"]
        if args.conditioning == W.X1:
            options = [W.ARITH, W.BINARY]  # the DMMA Newton-threshold kernel; --options 0,1,2 adds the lookback (f1)
        if args.options:
            options = [int(t) for t in args.options.split(",")]
        N = args.points or c["n_points"]
        L = (args.reps_per_gpu or c["n_replicates"]) * world
        plist = [q.params(S0=W.S0, K=100.0, r=W.R, sigma=W.SIGMA, T=W.T, d=d) for _ in options]
    ckw = dict(method=args.method, construction=args.construction, conditioning=args.conditioning,
               randomization=args.randomization, seed=W.SEED, device=local)
    cfg = q.config(**ckw)
    pricer = DistributedPricer(options, plist, N, L, cfg, dev, rank, world)

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    q.qmccpw_launch_count(reset=True)
    for _ in range(args.warmup):
        pricer.step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    q.qmccpw_launch_count(reset=True)
    step_ms, kern_ms = [], []
    stream = torch.cuda.current_stream(dev)
    results = None
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            pricer.enqueue_device_work((k0, k1))
            pricer.all_reduce()
            e1.record(stream)
            results = pricer.fetch_and_finalize()
            step_ms.append(e0.elapsed_time(e1))
            kern_ms.append(k0.elapsed_time(k1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = q.qmccpw_launch_count(reset=True)
    total_ms = sum(step_ms)
    kernel_avg_ms = sum(kern_ms) / len(kern_ms)
    if world > 1:
        t = torch.tensor([total_ms, kernel_avg_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, kernel_avg_ms = t.tolist()
    paths = N * L * args.steps
    value = paths / (total_ms / 1e3)

    # e2e: the public host API call per step (host buffers in, host results out)
    e2e_steps = args.e2e_steps or args.steps
    # clean e2e measurement (host wall time around each public call, max over ranks);
    # one untimed call first so the library's scratch allocation is not inside the timing
    if world == 1:
        q.qmccpw_price_greeks_batch(options, plist, N, L, q.config(**ckw))
    else:
        pricer.step()
    e2e_total = 0.0
    for _ in range(e2e_steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t1 = time.perf_counter()
        if world == 1:
            q.qmccpw_price_greeks_batch(options, plist, N, L, q.config(**ckw))
        else:
            pricer.step()
        e2e_total += time.perf_counter() - t1
    if world > 1:
        t = torch.tensor([e2e_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = t.item()
    e2e_value = N * L * e2e_steps / e2e_total

    # roofline of the dominant kernel (tables + fused path kernel), FP64-ALU bound
    peaks = measured_peaks()
    sm_max = float(peaks.get("sm_max_mhz", SM_MAX_MHZ_FALLBACK))
    peak_tflops = SM_COUNT * FP64_LANES_PER_SM * 2 * sm_max * 1e6 / 1e12
    if args.workload == "C5":
        # phase A per point: d inverse normals, the d x d contraction, 8 families x d exps;
        # phase B: the 1024 option tails (160 each, SURVEY 8(d) c_tail)
        per_path = d * 50 + d * d + 8 * d * (17 + 6) + len(options) * 160
    else:
        per_path = fp64_model_per_path(d, args.construction, args.conditioning, len(options),
                                       arith_x1=int(args.conditioning == W.X1 and W.ARITH in options),
                                       n_lookback_x1=sum(1 for t in options if t == W.LOOKBACK)
                                       if args.conditioning == W.X1 else 0)
        if args.method == 3:  # MC+AV-CPW: the antithetic path's exps, accumulators and tails as well
            per_path += d * (17 + 6) + len(options) * 160
    launch_paths = N * (L // world)
    achieved = 2.0 * per_path * launch_paths / (kernel_avg_ms / 1e3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if (os.path.exists(tpath) and args.workload == "C4" and args.randomization == 0
            and (args.construction, args.conditioning) == (W.BB, W.W1)):
        try:
            traffic = json.load(open(tpath)).get("bytes_per_launch")
        except Exception:
            traffic = None

    metric, unit = METRIC, UNIT
    if args.workload == "C5":
        metric = "C5 portfolio option-paths/sec (1024 options, d=128) with price+delta+vega+gamma; % FP64 roof"
        unit = "option-paths/s"
        value *= len(options)
        e2e_value *= len(options)
    if rank == 0:
        line = {
            "metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Sobol'/Philox; no datasets or weights)",
            "config": {
                "workload": ("C5: 1024 options (8 sigma/T families x 128; K 70..130; arith/binary/lookback), S0=100, "
                             "r=0.1, d=128, PCA-W1 (portfolio kernel)") if args.workload == "C5" else
                            ("C4: arithmetic+binary+lookback Asian calls fused on shared paths, S0=K=100, sigma=0.2, "
                             "r=0.1, T=1, d=64, " + {(1, 0): "BB-W1 (QMC+BB-CPW)", (0, 0): "STD-W1 (QMC-CPW)",
                                                     (2, 0): "PCA-W1", (2, 1): "PCA-X1 (Halley threshold)",
                                                     (0, 1): "STD-X1 (closed-form threshold)", (1, 1): "BB-X1 (Halley threshold)",
                                                     (3, 0): "GPCA-W1 (f3)", (3, 1): "GPCA-X1 (Halley threshold, f3)"}.get(
                                 (args.construction, args.conditioning), "custom"))
                            + {1: ", digital shift only", 3: ", plain Sobol'", 4: ", nested Owen scrambling (f4)"}.get(
                                args.randomization, "")
                            + (f", options {args.options}" if args.options else "")
                            + {1: ", LR+MC", 2: ", MC-CPW (Philox)", 3: ", MC+AV-CPW (Philox, antithetic)"}.get(
                                args.method, ""),
                "points_per_replicate": N, "replicates_per_gpu": L // world, "replicates_total": L,
                "global_batch": N * L, "seq_len": d, "parallelism": f"dp{world} (replicate-partitioned)",
                "option_paths_per_s": value * len(options), "greek_sets_per_s": value * len(options),
                "l2": "flushed (256 MiB write) before every timed step",
                "kernel_ms_avg": kernel_avg_ms,
            },
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak_tflops, "unit": "TFLOP/s",
                         "frac": achieved / peak_tflops, "traffic": traffic,
                         "note": f"FP64 pipe: {SM_COUNT} SMs x {FP64_LANES_PER_SM} FMA lanes x 2 x {sm_max:.0f} MHz; "
                                 f"algorithmic work {per_path} FP64 lane-instr/path (SURVEY 8(d) model)"},
            "clocks": clk.summary(),
            "e2e": {"value": e2e_value, "unit": unit, "h2d_bytes_per_step": pricer.h2d_bytes,
                    "d2h_bytes_per_step": pricer.d2h_bytes},
            "gpu_launches": int(launches),
            "results_sample": {"price": [r.mean[0] for r in results[:3]], "delta": [r.mean[1] for r in results[:3]],
                               "vega": [r.mean[2] for r in results[:3]], "gamma": [r.mean[3] for r in results[:3]]},
        }
        if world == 1 and not args.no_cpu_baseline and args.workload == "C4":
            line["cpu_baseline"] = cpu_baseline_oracle(options, d, args.construction, args.conditioning)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
