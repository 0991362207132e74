import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))  # repo root
import numpy as np
import oracle as O
import paper_2209_11337_b200 as q
for d in (16, 32, 48, 64, 96, 128):
    for (k0, k1) in ((0, 128), (50, 350), (0, 4096)):
        for cond in (0, 1):
            p = q.params(K=100.0, d=d)
            g = q.qmccpw_path_values(0, p, 2, k0, k1, q.config(construction=2, conditioning=cond, device=0))
            o = O.path_values(0, 100.0, O.market(d=d), O.config(construction=2, conditioning=cond), 2, k0, k1)
            err = np.abs(g - o) / (np.abs(o) + np.abs(O.pivots(0, 100.0, O.market(d=d))))
            bad = np.where(err.max(axis=1) > 1e-10)[0]
            print(d, (k0, k1), cond, "max err", err.max(), "bad rows", len(bad), bad[:12])
