import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))  # repo root
import numpy as np
import oracle as O
import paper_2209_11337_b200 as q
N = 3 * 4096 + 1234
for rep in range(4):
    g = q.qmccpw_path_values(2, q.params(K=90.0, d=64), rep, 0, N, q.config(construction=1, device=0))
    bad = np.where(~np.isfinite(g).all(axis=1) | (np.abs(g) > 1e6).any(axis=1))[0]
    print("rep", rep, "bad", len(bad), bad[:10])
    if len(bad):
        k = int(bad[0])
        o = O.path_values(2, 90.0, O.market(d=64), O.config(construction=1), rep, k, k + 1)
        print("  gpu", g[k], "ora", o[0])
        x = q.qmccpw_normals(rep, 64, k, k + 1, q.config(device=0))[0]
        xo = O.normals(rep, 64, k, k + 1, O.config())[0]
        print("  normals max diff", np.max(np.abs(x - xo)), "argmax", np.argmax(np.abs(x - xo)), x[np.argmax(np.abs(x-xo))], xo[np.argmax(np.abs(x-xo))])
        ys = q.qmccpw_sobol_u32(rep, 0, 64, k, k + 1, q.config(device=0))[:, 0]
        j = int(np.argmax(np.abs(x - xo)))
        print("  y", hex(int(ys[j])))
