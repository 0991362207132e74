import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))  # repo root
import numpy as np
import oracle as O
import paper_2209_11337_b200 as q
np.set_printoptions(linewidth=200, precision=6)
for d in (64, 96):
    p = q.params(K=100.0, d=d)
    g = q.qmccpw_path_values(0, p, 2, 0, 8, q.config(construction=2, conditioning=0, device=0))
    o = O.path_values(0, 100.0, O.market(d=d), O.config(construction=2, conditioning=0), 2, 0, 8)
    print(d); print(g); print(o)
    # lookback: W1 stats path with max tracking
    g = q.qmccpw_path_values(2, p, 2, 0, 8, q.config(construction=2, conditioning=0, device=0))
    o = O.path_values(2, 100.0, O.market(d=d), O.config(construction=2, conditioning=0), 2, 0, 8)
    print(g); print(o)
