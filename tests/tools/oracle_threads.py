"""Oracle (plain C, FP64) throughput on C4 with 1 thread and with all host cores: the
CPU side of the paper's GPU-vs-sequential-CPU comparison."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))  # repo root
import oracle as O  # noqa: E402
import workloads as W  # noqa: E402

mk = O.market(W.S0, W.R, W.SIGMA, W.T, 64)
opts = [(t, 100.0) for t in (0, 1, 2)]
cfg = O.config(construction=W.BB, conditioning=W.W1, seed=W.SEED)
cores = os.cpu_count() or 1
for threads, n, reps in ((1, 4096, 1), (cores, 8192, cores)):
    O.price_greeks(opts, mk, 256, reps, cfg, n_threads=threads)
    t0 = time.perf_counter()
    O.price_greeks(opts, mk, n, reps, cfg, n_threads=threads)
    dt = time.perf_counter() - t0
    print(f"threads={threads} paths={n * reps} seconds={dt:.2f} paths_per_s={n * reps / dt:.4g}")
print("cpu:", open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": \t"))
