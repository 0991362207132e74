import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))  # repo root
import numpy as np
import oracle as O
import paper_2209_11337_b200 as q

def run(otype, K, d, constr, cond, rep=3, k0=1000, k1=3000):
    p = q.params(K=K, d=d)
    g = q.qmccpw_path_values(otype, p, rep, k0, k1, q.config(construction=constr, conditioning=cond, device=0))
    mk = O.market(d=d)
    o = O.path_values(otype, K, mk, O.config(construction=constr, conditioning=cond), rep, k0, k1)
    piv = np.abs(O.pivots(otype, K, mk))
    err = np.abs(g - o) / (np.abs(o) + piv)
    s = 0.2 * (1.0 / d) ** 0.5
    print(f"type={otype} K={K} d={d} constr={constr} cond={cond}: max err/q {np.array2string(err.max(axis=0), precision=2)}"
          f"  gamma_err*s^2 {err[:,3].max()*s*s:.2e}  gamma_err*s {err[:,3].max()*s:.2e}")

for d in (16, 64, 256):
    for K in (90.0, 100.0, 110.0):
        for constr, cond in ((0, 0), (1, 0), (2, 0), (0, 1), (1, 1), (2, 1)):
            for t in (0, 1, 2):
                if cond == 1 and t == 2: continue
                if d == 256 and K != 100.0: continue
                run(t, K, d, constr, cond)
