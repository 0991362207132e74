#!/usr/bin/env python
"""bench.py -- QMC paths/s with price+delta+vega+gamma (d=64) on 1..8 B200.

Contract (task statement + BASELINE.json):
  python bench.py --gpus N --steps K --warmup W       (N > 1: under torchrun, or spawned by itself)
  python bench.py --impl reference ...                (the oracle on host cores)
prints ONE JSON line on rank 0.

Workload: BASELINE.json configs[3] = SURVEY.md C4 -- arithmetic Asian, binary
Asian and lookback calls fused on the same paths, S0 = K = 100, sigma = 0.2,
r = 0.1, T = 1, d = 64, Brownian bridge + W(t_1) conditioning (the paper's
QMC+BB-CPW), 2^20 Sobol' points x 64 randomisations.

Scaling:
  --scaling strong (default)  the SAME input on every N: the 2^20 x 64 grid of
                              cells (replicate, block of 4096 Sobol' indices) is
                              split over the N ranks by distributed.cell_range;
                              --points 8388608 is the x8 variant that amortises
                              fixed costs.  C5: the fixed 2^18 x 16 = 2^22 points
                              of the 1024-option portfolio, partitioned.
  --scaling weak              64 replicates PER GPU (N GPUs price 64 N).
--gpus N without torchrun re-launches itself under torch.distributed.run with
N ranks (127.0.0.1); a run whose world size differs from --gpus fails loudly.

A timed step = one full estimator run on the device: randomisation tables,
the fused path kernel over this rank's cells, per-replicate reduction, one
NCCL all-reduce (N > 1) and the device->host copy of the replicate sums, all
on the launching stream between two CUDA events.  The host finalize that
follows (tens of microseconds, reported as config.finalize_us) is outside the
events; `e2e` covers it.  value = underlying QMC paths (points x replicates,
each delivering the 4 outputs of all 3 options) per second over all ranks, at
the MEDIAN step time, max over ranks.  L2 is flushed (256 MiB write) before
every timed step, outside the events.
"""
import argparse
import json
import os
import socket
import statistics
import subprocess
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
MODE_NAMES = {(0, 0): "STD-W1", (1, 0): "BB-W1", (2, 0): "PCA-W1", (3, 0): "GPCA-W1",
              (0, 1): "STD-X1", (1, 1): "BB-X1", (2, 1): "PCA-X1", (3, 1): "GPCA-X1"}


def fp64_model_per_path(d, constr, cond, types, strikes):
    """Algorithmic FP64 lane-instructions per underlying path: SURVEY.md 8(d)'s planning model
    with its fixed constants (independent of how the kernel is written):

        W_path = d_icdf c_icdf + d (c_exp + c_W + 6) + n_solve d (c_exp + 3) + n_opt c_tail

    c_icdf = 50, c_exp = 17, c_tail = 160, c_W = 1 (STD) / 2 (BB) / d (PCA, GPCA).  d_icdf = d - 1
    where x_1 is not needed (STD-W1, every X1 mode), else d.  W1: n_solve = 0 (closed-form psi_d).
    X1 (reading 29): for each distinct-strike group of arithmetic / binary options one
    threshold solve of 4 passes (SURVEY's count); a lookback under X1 (row f1) adds one envelope
    pass.  Under STD (equal slopes) the threshold is in closed form and the envelope is a single
    line, both from the sums the path's own exponentials already give: no extra pass is charged.
    The per-date Phi-bar of the arithmetic X1 sums (App. A.4) is NOT in 8(d)'s model and is not
    credited here."""
    c_icdf, c_exp, c_tail = 50, 17, 160
    c_w = {0: 1, 1: 2, 2: d, 3: d}[constr]
    n_opt = len(types)
    d_icdf = d - 1 if (cond == 1 or constr == 0) else d
    w = d_icdf * c_icdf + d * (c_exp + c_w + 6) + n_opt * c_tail
    if cond == 1 and constr != 0:
        nonlb = [(t, K) for t, K in zip(types, strikes) if t != W.LOOKBACK]
        n_groups = len({K for _, K in nonlb})
        n_lb = sum(1 for t in types if t == W.LOOKBACK)
        w += (n_groups * 4 + n_lb) * d * (c_exp + 3)
    return w


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def ncu_counters(key):
    """ncu --set full counters of this mode's dominant kernel, from the committed
    profiles/ncu_metrics.json (scripts/ncu_to_json.py): FP64 pipe, issue, SFU (xu) utilisation,
    DRAM bytes per launch.  None if this mode has not been captured."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_metrics.json"))).get(key)
    except Exception:
        return None


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


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline_oracle(options, d, constr, cond, method=0, budget_1t_s=10.0):
    """The oracle (plain C, never tuned) on this host: ONE thread and ALL cores on the same
    bounded sample of the workload: replicates 0..R-1 x the
    first n Sobol' points, R = min(64, cores), n sized for ~budget_1t_s on one thread."""
    import oracle as O
    cores = os.cpu_count() or 1
    opts = [(t, 100.0) for t in options]
    mk = O.market(W.S0, W.R, W.SIGMA, W.T, d)
    cfg = O.config(method=method, construction=constr, conditioning=cond, seed=W.SEED)
    reps = max(1, min(64, cores))
    t0 = time.perf_counter()
    O.price_greeks(opts, mk, 64, reps, cfg, n_threads=1)
    pilot = (time.perf_counter() - t0) / (64 * reps)
    n = int(max(64, min(1 << 20, budget_1t_s / max(pilot, 1e-9) / reps)))
    t0 = time.perf_counter()
    O.price_greeks(opts, mk, n, reps, cfg, n_threads=1)
    dt1 = time.perf_counter() - t0
    t0 = time.perf_counter()
    O.price_greeks(opts, mk, n, reps, cfg, n_threads=cores)
    dtn = time.perf_counter() - t0
    sample = (f"C4 replicates 0..{reps - 1} x first {n} Sobol' points ({n * reps} paths), {len(options)} options "
              f"fused, d={d}, {MODE_NAMES.get((constr, cond), '?')}")
    return {"value": n * reps / dtn, "unit": UNIT, "cores": min(cores, reps), "kind": "oracle", "sample": sample,
            "seconds": dtn, "one_thread": {"value": n * reps / dt1, "unit": UNIT, "cores": 1, "seconds": dt1},
            "nproc": cores, "cpu_model": cpu_model()}


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
    med = statistics.median(times)
    value = n * reps / med
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * med,
            "ms_per_step_mean": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Sobol'/Philox; no datasets)",
            "config": {"workload": "C4: arith+binary+lookback Asian calls fused, d=64, BB-W1 (QMC+BB-CPW)",
                       "sample_per_step": f"{reps} replicates x {n} points", "global_batch": n * reps,
                       "seq_len": d, "parallelism": "host threads"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": min(cores, reps), "kind": "oracle",
                             "sample": f"{reps} replicates x {n} points per step", "nproc": cores,
                             "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(args):
    """--gpus N > 1 without a torchrun environment: re-launch this script under
    torch.distributed.run with N ranks, one per GPU.  Fails loudly without N GPUs."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible CUDA devices, found {have}\n")
        return 3
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the same input split over the ranks (default); weak: 64 replicates per GPU")
    ap.add_argument("--construction", type=int, default=W.BB)
    ap.add_argument("--conditioning", type=int, default=W.W1)
    ap.add_argument("--randomization", type=int, default=0,
                    help="0 LMS + digital shift (default), 1 shift, 3 none, 4 nested Owen scrambling (row f4)")
    ap.add_argument("--workload", default="C4", choices=["C4", "C5"],
                    help="C4: 3 exotics fused, d=64 (the BASELINE metric); C5: 1024-option portfolio, d=128")
    ap.add_argument("--method", type=int, default=0,
                    help="0 QMC-CPW (default), 1 LR+MC (STD), 2 MC-CPW, 3 MC+AV-CPW (STD/BB, W1; row f2)")
    ap.add_argument("--options", default=None, help="comma-separated option types (0 arith, 1 binary, 2 lookback)")
    ap.add_argument("--points", type=int, default=None, help="points per replicate (C4 default 2^20; x8: 8388608)")
    ap.add_argument("--replicates", type=int, default=None,
                    help="replicates (strong: in total; weak: per GPU); C4 default 64, C5 16")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    return ap.parse_args(argv)


def main():
    args = parse_args()
    if args.gpus < 1:
        sys.exit("bench.py: --gpus must be >= 1")
    if args.impl == "reference":
        return run_reference(args)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: world size {world} != --gpus {args.gpus}; refusing to report a mislabelled run")

    import torch
    import torch.distributed as dist

    import paper_2209_11337_b200 as q
    from paper_2209_11337_b200.distributed import DistributedPricer

    if not torch.cuda.is_available() or torch.cuda.device_count() <= local:
        sys.exit(f"bench.py: rank {rank} needs cuda:{local}; no CUDA device (there is no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    strong = args.scaling == "strong"
    if args.workload == "C5":
        port = W.c5_portfolio()
        options, d = [o["type"] for o in port], 128
        strikes = [o["K"] for o in port]
        args.construction, args.conditioning = W.PCA, W.W1
        N = args.points or (1 << 18)
        reps = args.replicates or 16
        plist = [q.params(S0=o["S0"], K=o["K"], r=o["r"], sigma=o["sigma"], T=o["T"], d=d) for o in port]
    else:
        c = W.CONFIGS[W.HEADLINE]
        options, d = c["options"], c["d"]
        if args.conditioning == W.X1:
            options = [W.ARITH, W.BINARY]  # the DMMA Newton-threshold kernel; --options 0,1,2 adds the lookback (f1)
        if args.options:
            options = [int(t) for t in args.options.split(",")]
        strikes = [100.0] * len(options)
        N = args.points or c["n_points"]
        reps = args.replicates or c["n_replicates"]
        plist = [q.params(S0=W.S0, K=100.0, r=W.R, sigma=W.SIGMA, T=W.T, d=d) for _ in options]
    L = reps if strong else reps * world
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
    step_ms, kern_ms, fin_s = [], [], []
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
            pricer.enqueue_fetch()
            e1.record(stream)
            stream.synchronize()
            t0 = time.perf_counter()
            results = pricer.finalize()
            fin_s.append(time.perf_counter() - t0)
            step_ms.append(e0.elapsed_time(e1))
            kern_ms.append(k0.elapsed_time(k1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = q.qmccpw_launch_count(reset=True)
    med_ms = statistics.median(step_ms)
    mean_ms = sum(step_ms) / len(step_ms)
    kernel_avg_ms = sum(kern_ms) / len(kern_ms)
    if world > 1:
        t = torch.tensor([med_ms, mean_ms, kernel_avg_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        med_ms, mean_ms, kernel_avg_ms = t.tolist()
    value = N * L / (med_ms / 1e3)

    # e2e: the public host API per step (host buffers in, host results out): one process prices
    # through qmccpw_price_greeks_batch; N ranks through DistributedPricer.step (partials, replicate
    # sums, NCCL all-reduce, D2H, finalize).  One untimed call first (scratch allocation).
    e2e_steps = args.e2e_steps or args.steps

    def public_call():
        if world == 1:
            return q.qmccpw_price_greeks_batch(options, plist, N, L, q.config(**ckw))
        return pricer.step()

    public_call()
    e2e_times = []
    for _ in range(e2e_steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t1 = time.perf_counter()
        public_call()
        e2e_times.append(time.perf_counter() - t1)
    e2e_med = statistics.median(e2e_times)
    if world > 1:
        t = torch.tensor([e2e_med], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_med = t.item()
    e2e_value = N * L / e2e_med

    # roofline of the dominant kernel (the fused path kernel over this rank's cells), FP64-ALU bound
    peaks = measured_peaks()
    sm_max = float(peaks.get("sm_max_mhz", SM_MAX_MHZ_FALLBACK))
    peak_tflops = SM_COUNT * FP64_LANES_PER_SM * 2 * sm_max * 1e6 / 1e12
    if args.workload == "C5":
        # phase A per point: d inverse normals, the d x d contraction, 8 families x d exps;
        # phase B: the 1024 option tails (160 each, SURVEY 8(d) c_tail)
        per_path = d * 50 + d * d + 8 * d * (17 + 6) + len(options) * 160
        mode_key = "C5"
    else:
        per_path = fp64_model_per_path(d, args.construction, args.conditioning, options, strikes)
        if args.method == 3:  # MC+AV-CPW: the antithetic path's exps, accumulators and tails as well
            per_path += d * (17 + 6) + len(options) * 160
        mode_key = MODE_NAMES.get((args.construction, args.conditioning), "custom")
        if args.options or args.method or args.randomization:
            mode_key += f"/o{','.join(map(str, options))}/m{args.method}/r{args.randomization}"
    launch_paths = pricer.points_owned()
    achieved = 2.0 * per_path * launch_paths / (kernel_avg_ms / 1e3) / 1e12
    default_size = (N, reps) == ((1 << 18, 16) if args.workload == "C5" else (1 << 20, 64))
    ncu = ncu_counters(mode_key) if (world == 1 and default_size) else None  # captured on one GPU at this size

    metric, unit = METRIC, UNIT
    if args.workload == "C5":
        metric = "C5 portfolio option-paths/sec (1024 options, d=128) with price+delta+vega+gamma; % FP64 roof"
        unit = "option-paths/s"
        value *= len(options)
        e2e_value *= len(options)
    if rank == 0:
        mode_txt = {(1, 0): "BB-W1 (QMC+BB-CPW)", (0, 0): "STD-W1 (QMC-CPW)", (2, 0): "PCA-W1",
                    (2, 1): "PCA-X1 (Halley threshold)", (0, 1): "STD-X1 (closed-form threshold)",
                    (1, 1): "BB-X1 (Halley threshold)", (3, 0): "GPCA-W1 (f3)",
                    (3, 1): "GPCA-X1 (Halley threshold, f3)"}.get((args.construction, args.conditioning), "custom")
        workload = (("C5: 1024 options (8 sigma/T families x 128; K 70..130; arith/binary/lookback), S0=100, "
                     "r=0.1, d=128, PCA-W1 (portfolio kernel)") if args.workload == "C5" else
                    ("C4: arithmetic+binary+lookback Asian calls fused on shared paths, S0=K=100, sigma=0.2, "
                     "r=0.1, T=1, d=64, " + mode_txt)
                    + {1: ", digital shift only", 3: ", plain Sobol'", 4: ", nested Owen scrambling (f4)"}.get(
                        args.randomization, "")
                    + (f", options {args.options}" if args.options else "")
                    + {1: ", LR+MC", 2: ", MC-CPW (Philox)", 3: ", MC+AV-CPW (Philox, antithetic)"}.get(
                        args.method, ""))
        roof = {"bound": "alu", "achieved": achieved, "peak": peak_tflops, "unit": "TFLOP/s",
                "frac": achieved / peak_tflops, "traffic": ncu.get("dram_bytes_per_launch") if ncu else None,
                "work_per_path": per_path,
                "note": f"FP64 pipe: {SM_COUNT} SMs x {FP64_LANES_PER_SM} FMA lanes x 2 x {sm_max:.0f} MHz "
                        f"(spec at sm_max_mhz; DESIGN.md 5); algorithmic work {per_path} FP64 lane-instr/path "
                        f"(SURVEY 8(d) model) x {launch_paths} paths per launch / kernel time (CUDA events)"}
        try:  # the FP64 roof measured on this GPU now (context; the denominator stays the spec figure)
            mb = q.qmccpw_fp64_roof(local)
            roof["measured_roof"] = {k: mb[k] for k in ("dfma_tflops", "dmma_tflops", "sm_clock_mhz",
                                                        "dfma_latency_cycles")}
            roof["measured_roof"]["dfma_frac_of_spec_at_run_clock"] = mb["dfma_tflops"] / (
                SM_COUNT * FP64_LANES_PER_SM * 2 * mb["sm_clock_mhz"] * 1e6 / 1e12)
        except Exception as e:  # noqa: BLE001 -- context only
            roof["measured_roof"] = {"error": str(e)}
        if ncu:
            roof["ncu"] = {k: ncu[k] for k in ("fp64_pipe_pct", "dmma_pipe_pct", "fp64_plus_dmma_pct",
                                               "issue_active_pct", "xu_pipe_pct", "warps_active",
                                               "registers", "build", "source") if k in ncu}
        line = {
            "metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": med_ms, "ms_per_step_mean": mean_ms, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Sobol'/Philox; no datasets or weights)",
            "config": {
                "workload": workload,
                "points_per_replicate": N, "replicates_total": L, "replicates_per_gpu": L / world,
                "global_batch": N * L, "seq_len": d,
                "parallelism": f"dp{world} (cell-range partitioned: Sobol' index blocks x replicates; "
                               f"one NCCL all-reduce)" if world > 1 else "dp1",
                "option_paths_per_s": value * (1 if args.workload == "C5" else len(options)),
                "greek_sets_per_s": value * (1 if args.workload == "C5" else len(options)),
                "l2": "flushed (256 MiB write) before every timed step",
                "timed_region": "tables + path kernel + replicate sums + all-reduce + D2H (CUDA events); "
                                "median of the steps",
                "kernel_ms_avg": kernel_avg_ms, "finalize_us": 1e6 * statistics.median(fin_s),
            },
            "roofline": roof,
            "clocks": clk.summary(),
            "e2e": {"value": e2e_value, "unit": unit, "h2d_bytes_per_step": pricer.h2d_bytes,
                    "d2h_bytes_per_step": pricer.d2h_bytes,
                    "api": "qmccpw_price_greeks_batch" if world == 1 else "DistributedPricer.step"},
            "gpu_launches": int(launches),
            "results_sample": {"price": [r.mean[0] for r in results[:3]], "delta": [r.mean[1] for r in results[:3]],
                               "vega": [r.mean[2] for r in results[:3]], "gamma": [r.mean[3] for r in results[:3]]},
        }
        if world == 1 and not args.no_cpu_baseline and args.workload == "C4":
            line["cpu_baseline"] = cpu_baseline_oracle(options, d, args.construction, args.conditioning,
                                                       args.method)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
