"""Diagnostic: dump worst per-path disagreements GPU vs oracle for one case."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))  # repo root
import numpy as np
import oracle as O
import paper_2209_11337_b200 as q

def run(otype, K, d, constr, cond, rep=3, k0=1000, k1=1700):
    p = q.params(K=K, d=d)
    g = q.qmccpw_path_values(otype, p, rep, k0, k1, q.config(construction=constr, conditioning=cond, device=0))
    mk = O.market(d=d)
    o = O.path_values(otype, K, mk, O.config(construction=constr, conditioning=cond), rep, k0, k1)
    piv = np.abs(O.pivots(otype, K, mk))
    err = np.abs(g - o) / (np.abs(o) + piv)
    print(f"case type={otype} K={K} d={d} constr={constr} cond={cond}: max err per q", err.max(axis=0))
    idx = np.argsort(-err.max(axis=1))[:5]
    for i in idx:
        print("  k", k0 + i, "gpu", g[i], "ora", o[i], "err", err[i])
    if cond == 1:
        x = O.normals(rep, d, k0 + idx[0], k0 + idx[0] + 1, O.config(construction=constr))[0]
        print("  x", x)

if __name__ == "__main__":
    for K in (90.0, 100.0, 110.0):
        for constr in (0, 1, 2):
            run(1, K, 16, constr, 1)
            run(0, K, 16, constr, 1)
