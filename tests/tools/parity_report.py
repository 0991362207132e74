"""Measured GPU-vs-oracle deviations per mode, written to
gpurun_out/parity_report.json.  Per-path: max |df| / (|f| + |pivot_K|) per
output (gamma also scaled by sigma^2 t_1, the conditioning factor); full runs:
max |dC| / max(|C|, mean|f|) (SURVEY.md 8(c)'s scales)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import paper_2209_11337_b200 as q  # noqa: E402
import workloads as W  # noqa: E402

NAMES = {(0, 0): "STD-W1", (1, 0): "BB-W1", (2, 0): "PCA-W1", (3, 0): "GPCA-W1",
         (0, 1): "STD-X1", (1, 1): "BB-X1", (2, 1): "PCA-X1", (3, 1): "GPCA-X1"}


def main():
    out = {"per_path": {}, "means": {}}
    for (constr, cond), name in NAMES.items():
        for method in ((0, 1, 2, 3) if (cond == 0 and constr in (0, 1)) else (0,)):
            if method == 1 and constr != 0:
                continue
            worst = np.zeros(4)
            worst_g = 0.0
            for d in (1, 4, 16, 64, 128):
                if constr == 1 and d & (d - 1):
                    continue
                for otype in (0, 1, 2):
                    for K in W.STRIKES:
                        p = q.params(K=K, d=d)
                        cfg = q.config(method=method, construction=constr, conditioning=cond, device=0)
                        g = q.qmccpw_path_values(otype, p, 3, 1000, 1000 + 512, cfg)
                        mk = O.market(d=d)
                        o = O.path_values(otype, K, mk, O.config(method=method, construction=constr,
                                                                 conditioning=cond), 3, 1000, 1000 + 512)
                        piv = np.abs(O.pivots(otype, K, mk))
                        err = (np.abs(g - o) / (np.abs(o) + piv)).max(axis=0)
                        worst = np.maximum(worst, err)
                        worst_g = max(worst_g, err[3] * W.SIGMA ** 2 * W.T / d)
            key = name + ("" if method == 0 else f"/m{method}")
            out["per_path"][key] = {"price": worst[0], "delta": worst[1], "vega": worst[2], "gamma": worst[3],
                                    "gamma_x_sigma2_t1": worst_g}
            print(key, out["per_path"][key], flush=True)
            N, L = 2 * 4096 + 77, 4
            opts = [0, 1, 2]
            dev = np.zeros(4)
            for K in W.STRIKES:
                res = q.qmccpw_price_greeks_batch(opts, [q.params(K=K, d=64)] * 3, N, L,
                                                  q.config(method=method, construction=constr, conditioning=cond,
                                                           device=0))
                ref, _ = O.price_greeks([(t, K) for t in opts], O.market(d=64), N, L,
                                        O.config(method=method, construction=constr, conditioning=cond))
                for r, o in zip(res, ref):
                    scale = np.maximum(np.abs(o["mean"]), o["mean_abs"])
                    dev = np.maximum(dev, np.abs(np.array(r.mean[:]) - o["mean"]) / scale)
            out["means"][key] = dict(zip(("price", "delta", "vega", "gamma"), dev.tolist()))
            print(key, "means", out["means"][key], flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "parity_report.json"), "w"), indent=1,
              default=float)


if __name__ == "__main__":
    main()
