"""Reproduce the paper's experiments on one B200.

Tables 1-3: VRF = sigma_LR^2 / sigma_method^2 of delta,
vega, gamma for LR+MC, MC-CPW, MC+AV-CPW, QMC-CPW (STD) and QMC+BB-CPW (BB),
P = 2^15 paths, L = 500 runs (sigma with divisor L), S0 = 100,
sigma = 0.2, r = 0.1, T = 1, K in {90, 100, 110}, d in {64, 256};
plus this build's rows (marked "ours", d = 64): Owen scrambling (f4), PCA-W1, PCA-X1
and GPCA-X1 (f3; the paper's stated future work).

Figures 3-11: the run-to-run error sigma of each Greek against
P = 2^12 .. 2^19 at d = 256, L = 500.

Writes results/paper_tables.md and results/paper_figures.json.  The paper's
randomisation of its L runs is unknown (reading 10), so agreement is
expected in magnitude, not digit for digit.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2209_11337_b200 as q  # noqa: E402

PAPER = {  # (option, K, d) -> {method: (delta, vega, gamma)}; Tables 1-3
    "arith": {
        (90, 64): {"MC-CPW": (623, 471, 20393), "MC+AV-CPW": (3209, 1566, 49141), "QMC-CPW": (5784, 14603, 28067), "QMC+BB-CPW": (154860, 442513, 271351)},
        (90, 256): {"MC-CPW": (2159, 1595, 108667), "MC+AV-CPW": (9527, 5424, 275370), "QMC-CPW": (11976, 30894, 134644), "QMC+BB-CPW": (106806, 340858, 487940)},
        (100, 64): {"MC-CPW": (106, 294, 3814), "MC+AV-CPW": (963, 759, 9433), "QMC-CPW": (903, 7770, 5427), "QMC+BB-CPW": (52689, 376285, 75020)},
        (100, 256): {"MC-CPW": (353, 967, 20967), "MC+AV-CPW": (2702, 2540, 49834), "QMC-CPW": (1735, 18162, 21116), "QMC+BB-CPW": (34478, 633051, 72558)},
        (110, 64): {"MC-CPW": (35, 113, 1101), "MC+AV-CPW": (172, 289, 2468), "QMC-CPW": (207, 3195, 1477), "QMC+BB-CPW": (13226, 119816, 23085)},
        (110, 256): {"MC-CPW": (103, 330, 5977), "MC+AV-CPW": (423, 917, 13770), "QMC-CPW": (445, 6701, 6147), "QMC+BB-CPW": (7645, 294813, 25695)},
    },
    "binary": {
        (90, 64): {"MC-CPW": (109, 326, 363), "MC+AV-CPW": (247, 733, 713), "QMC-CPW": (150, 447, 376), "QMC+BB-CPW": (1447, 4227, 999)},
        (90, 256): {"MC-CPW": (159, 481, 691), "MC+AV-CPW": (389, 1168, 1446), "QMC-CPW": (197, 593, 673), "QMC+BB-CPW": (714, 2114, 883)},
        (100, 64): {"MC-CPW": (43, 771, 136), "MC+AV-CPW": (123, 2078, 201), "QMC-CPW": (58, 1176, 126), "QMC+BB-CPW": (830, 12571, 784)},
        (100, 256): {"MC-CPW": (64, 1419, 201), "MC+AV-CPW": (150, 3405, 415), "QMC-CPW": (64, 1502, 212), "QMC+BB-CPW": (221, 5111, 392)},
        (110, 64): {"MC-CPW": (23, 839, 79), "MC+AV-CPW": (69, 1965, 137), "QMC-CPW": (32, 1167, 67), "QMC+BB-CPW": (497, 9232, 355)},
        (110, 256): {"MC-CPW": (35, 1976, 116), "MC+AV-CPW": (89, 4617, 237), "QMC-CPW": (36, 1950, 117), "QMC+BB-CPW": (150, 7803, 179)},
    },
    "lookback": {
        (90, 64): {"MC-CPW": (7020, 501, 55102633), "MC+AV-CPW": (58906, 2333, 113383607), "QMC-CPW": (382145, 10667, 113193362), "QMC+BB-CPW": (2631721, 51816, 129220281)},
        (90, 256): {"MC-CPW": (26665, 1855, 1.2e17), "MC+AV-CPW": (187898, 7492, 4.2e17), "QMC-CPW": (1135848, 33043, 6.2e16), "QMC+BB-CPW": (7737083, 165179, 1.0e18)},
        (100, 64): {"MC-CPW": (1635, 311, 27235), "MC+AV-CPW": (12183, 1420, 72792), "QMC-CPW": (21857, 6580, 89333), "QMC+BB-CPW": (40682, 35370, 212928)},
        (100, 256): {"MC-CPW": (8323, 1138, 175073), "MC+AV-CPW": (58180, 4569, 393763), "QMC-CPW": (79683, 20418, 434423), "QMC+BB-CPW": (171880, 103536, 604285)},
        (110, 64): {"MC-CPW": (233, 178, 9787), "MC+AV-CPW": (1899, 870, 24450), "QMC-CPW": (1896, 4601, 13755), "QMC+BB-CPW": (13181, 26065, 42199)},
        (110, 256): {"MC-CPW": (920, 657, 51687), "MC+AV-CPW": (5594, 2876, 123922), "QMC-CPW": (4264, 13739, 60037), "QMC+BB-CPW": (23354, 69210, 112398)},
    },
}
OPT = {"arith": 0, "binary": 1, "lookback": 2}
METHODS = {  # name -> (method, construction, conditioning, randomization)
    "LR+MC": (1, 0, 0, 0), "MC-CPW": (2, 0, 0, 0), "MC+AV-CPW": (3, 0, 0, 0), "QMC-CPW": (0, 0, 0, 0),
    "QMC+BB-CPW": (0, 1, 0, 0),
    "QMC+BB-CPW Owen (ours)": (0, 1, 0, 4), "PCA-W1 (ours)": (0, 2, 0, 0), "PCA-X1 (ours)": (0, 2, 1, 0),
    "PCA-X1 Owen (ours)": (0, 2, 1, 4), "GPCA-X1 (ours)": (0, 3, 1, 0),
}


def sigma_run(option, K, d, P, L, method):
    m, c, k, rz = METHODS[method]
    cfg = q.config(method=m, construction=c, conditioning=k, randomization=rz, device=0)
    r = q.qmccpw_price_greeks(OPT[option], q.params(K=float(K), d=d), P, L, cfg)
    return np.array(r.sigma_run[:]), np.array(r.mean[:])


def tables(P=1 << 15, L=500, log=None):
    rows, raw = [], {}
    for option in ("arith", "binary", "lookback"):
        for (K, d) in PAPER[option]:
            s0, m0 = sigma_run(option, K, d, P, L, "LR+MC")
            for method in METHODS:
                if method == "LR+MC" or ("ours" in method and d > 128):
                    continue  # our PCA rows at d = 64 only (d = 256 PCA uses the slow shared-memory fallback)
                t0 = time.time()
                s, mm = sigma_run(option, K, d, P, L, method)
                with np.errstate(divide="ignore"):
                    vrf = (s0[1:] / s[1:]) ** 2
                if log:
                    log.write(f"{option} {K} {d} {method} {time.time() - t0:.2f}s vrf {vrf.tolist()}\n")
                    log.flush()
                paper = PAPER[option][(K, d)].get(method)
                raw[f"{option},{K},{d},{method}"] = dict(vrf=vrf.tolist(), sigma=s.tolist(), mean=mm.tolist(),
                                                         paper=paper)
                rows.append((option, K, d, method, vrf, paper))
    return rows, raw


def figures(L=500, d=256):
    out = {}
    for option in ("arith", "binary", "lookback"):
        for K in (90, 100, 110):
            for method in METHODS:
                if "ours" in method:
                    continue
                key = f"{option},{K},{method}"
                out[key] = {}
                for lp in range(12, 20):
                    s, _ = sigma_run(option, K, d, 1 << lp, L, method)
                    out[key][lp] = s.tolist()
    return out


def fmt(v):
    return f"{v:.2e}" if (v >= 1e6 or v < 1) else f"{v:,.0f}"


def main():
    os.makedirs(os.path.join(ROOT, "results"), exist_ok=True)
    t0 = time.time()
    with open(os.path.join(ROOT, "results", "tables_progress.log"), "w") as log:
        rows, raw = tables(log=log)
    t_tab = time.time() - t0
    lines = ["# Paper Tables 1-3 reproduced on one B200 (P = 2^15, L = 500)", "",
             "VRF = sigma_LR^2 / sigma^2 for delta / vega / gamma (PAPER.md P:637-652).  `paper` = the printed",
             "value (P:667-769).  Randomisation of the L runs differs from the paper's (unspecified) one, so",
             "magnitudes, not digits, are comparable.  Generated by `scripts/reproduce_tables.py` "
             f"({t_tab:.1f} s of GPU time for all {len(rows)} rows).", "",
             "| option | K | d | method | VRF delta (ours / paper) | VRF vega | VRF gamma |", "|---|---|---|---|---|---|---|"]
    for option, K, d, method, vrf, paper in rows:
        cells = []
        for i in range(3):
            cells.append(fmt(vrf[i]) + (" / " + fmt(paper[i]) if paper else ""))
        lines.append(f"| {option} | {K} | {d} | {method} | " + " | ".join(cells) + " |")
    open(os.path.join(ROOT, "results", "paper_tables.md"), "w").write("\n".join(lines) + "\n")
    json.dump({"tables": raw}, open(os.path.join(ROOT, "results", "paper_tables.json"), "w"))
    if "--figures" in sys.argv:
        t1 = time.time()
        figs = figures()
        json.dump({"figures": figs, "seconds": time.time() - t1},
                  open(os.path.join(ROOT, "results", "paper_figures.json"), "w"))
    print("\n".join(lines[:12]))


if __name__ == "__main__":
    main()
