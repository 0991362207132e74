"""A fixed list of C-ABI calls touching every kernel (the sanitize_run.py set at smaller sizes),
results saved to an .npy: run once normally and once with QMCCPW_POISON=1 and/or
QMCCPW_LIB=<checked build> by tests/test_memory_safety.py."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2209_11337_b200 as q  # noqa: E402
import workloads as W  # noqa: E402


def cfg(constr, cond, method=0, rand=0):
    return q.config(method=method, construction=constr, conditioning=cond, randomization=rand, device=0)


def main(out):
    N, L = 4096 + 77, 2
    vals = []
    runs = []
    for constr, cond in ((0, 0), (1, 0), (2, 0), (3, 0), (0, 1), (1, 1), (2, 1), (3, 1)):
        for d in (16, 64):
            runs.append(([0, 1, 2], d, cfg(constr, cond)))
        if cond == 1:
            runs.append(([0, 1], 64, cfg(constr, cond)))
    runs += [([0, 1, 2], 200, cfg(2, 0)), ([0, 1, 2], 200, cfg(2, 1)), ([0, 1, 2], 64, cfg(2, 1, rand=4)),
             ([0, 1, 2], 64, cfg(1, 0, rand=4)), ([0, 1, 2], 64, cfg(0, 0, 1)), ([0, 1, 2], 64, cfg(0, 0, 2)),
             ([0, 1, 2], 64, cfg(1, 0, 2)), ([0, 1, 2], 64, cfg(0, 0, 3)), ([0, 1, 2], 64, cfg(1, 0, 3))]
    for opts, d, c in runs:
        for r in q.qmccpw_price_greeks_batch(opts, [q.params(K=95.0, d=d)] * len(opts), N, L, c):
            vals.append(np.concatenate([r.mean[:], r.se[:], r.within_var[:]]))
    port = W.c5_portfolio()
    for d in (16, 128):
        sel = [port[i] for i in range(0, 1024, 37)]
        ps = [q.params(S0=o["S0"], K=o["K"], r=o["r"], sigma=o["sigma"], T=o["T"], d=d) for o in sel]
        for r in q.qmccpw_price_greeks_batch([o["type"] for o in sel], ps, N, L, cfg(2, 0)):
            vals.append(np.concatenate([r.mean[:], r.se[:], r.within_var[:]]))
        vals.append(q.qmccpw_portfolio_path_values([o["type"] for o in sel], ps, 1, 5, 5 + 300, cfg(2, 0)).ravel())
    for rand in (0, 2, 4):
        vals.append(q.qmccpw_sobol_u32(1, 0, 64, 1000, 3000, cfg(0, 0, rand=rand)).astype(np.float64).ravel())
    vals.append(q.qmccpw_normals(1, 64, 0, 2000, cfg(0, 0)).ravel())
    for constr, cond in ((0, 0), (1, 0), (2, 0), (2, 1), (1, 1)):
        for t in (0, 1, 2):
            vals.append(q.qmccpw_path_values(t, q.params(d=64), 1, 10, 10 + 500, cfg(constr, cond)).ravel())
    np.save(out, np.concatenate(vals))
    print("launches", q.qmccpw_launch_count())


if __name__ == "__main__":
    main(sys.argv[1])
