"""Locate the BB-X1 means deviation (parity_report: gamma 2.7e-9 of max(|C|, mean|f|)) down to
single paths: means per (K, option), then per-path values of the worst (K, option) over every
point of every replicate, worst paths printed with both sides' values."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import paper_2209_11337_b200 as q  # noqa: E402

constr, cond, d = int(sys.argv[1]) if len(sys.argv) > 1 else 1, 1, 64
N, L = 2 * 4096 + 77, 4
worst = (0, None)
for K in (90.0, 100.0, 110.0):
    for t in (0, 1, 2):
        g = q.qmccpw_price_greeks(t, q.params(K=K, d=d), N, L, q.config(construction=constr, conditioning=cond, device=0))
        o, _ = O.price_greeks([(t, K)], O.market(d=d), N, L, O.config(construction=constr, conditioning=cond))
        scale = np.maximum(np.abs(o[0]["mean"]), o[0]["mean_abs"])
        dev = np.abs(np.array(g.mean[:]) - o[0]["mean"]) / scale
        print(f"K={K} type={t} dev={dev} ties g/o {g.argmax_near_ties}/{o[0]['argmax_near_ties']}", flush=True)
        if dev.max() > worst[0]:
            worst = (dev.max(), (K, t))
K, t = worst[1]
print("worst", worst, flush=True)
mk = O.market(d=d)
piv = np.abs(O.pivots(t, K, mk))
for rep in range(L):
    gv = q.qmccpw_path_values(t, q.params(K=K, d=d), rep, 0, N, q.config(construction=constr, conditioning=cond, device=0))
    ov = O.path_values(t, K, mk, O.config(construction=constr, conditioning=cond), rep, 0, N)
    err = np.abs(gv - ov) / (np.abs(ov) + piv)
    idx = np.argsort(err.max(axis=1))[-3:]
    for i in idx:
        print(f"rep {rep} k {i} err {err[i]} gpu {gv[i]} oracle {ov[i]}", flush=True)
