"""Small runs that touch every kernel of libqmccpw.so, for compute-sanitizer
(SURVEY.md 4.3 T7): memcheck, racecheck, synccheck, initcheck.

    compute-sanitizer --tool memcheck python scripts/sanitize_run.py

Sizes are C1/C2-like (a few cells) so the instrumented run finishes in minutes.
Each call goes through the C ABI exactly as the tests and bench do.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2209_11337_b200 as q  # noqa: E402
import workloads as W  # noqa: E402


def cfg(constr, cond, method=0, rand=0):
    return q.config(method=method, construction=constr, conditioning=cond, randomization=rand, device=0)


def main():
    import torch
    torch.cuda.init()
    N, L = 4096 + 77, 2                                     # one full cell + a ragged one
    opts3 = [0, 1, 2]
    runs = []
    for constr, cond in ((0, 0), (1, 0), (2, 0), (3, 0), (0, 1), (1, 1), (2, 1), (3, 1)):
        # three options fused; X1 with a lookback also takes the envelope kernels (row f1)
        for d in (16, 64):
            runs.append((opts3, d, cfg(constr, cond)))
        if cond == 1:
            runs.append(([0, 1], 64, cfg(constr, cond)))     # X1 without a lookback (the Halley-only kernel)
    runs.append((opts3, 200, cfg(2, 0)))                    # PCA beyond the DMMA tile range
    runs.append((opts3, 200, cfg(2, 1)))
    runs.append((opts3, 64, cfg(2, 1, rand=4)))             # Owen + PCA-X1 instantiation
    runs.append((opts3, 64, cfg(1, 0, rand=4)))
    for method in (1, 2, 3):                                # LR+MC, MC-CPW, MC+AV-CPW (a9, f2)
        for constr in ((0,) if method == 1 else (0, 1)):
            runs.append((opts3, 64, cfg(constr, 0, method)))
    for opts, d, c in runs:
        res = q.qmccpw_price_greeks_batch(opts, [q.params(d=d)] * len(opts), N, L, c)
        print(f"batch d={d} constr={c.construction} cond={c.conditioning} method={c.method} "
              f"rand={c.randomization}: price {res[0].mean[0]:.6f}", flush=True)
    # C5-style portfolio kernel (several families), d = 16 and 128
    port = W.c5_portfolio()
    for d in (16, 128):
        sel = [port[i] for i in range(0, 1024, 37)]
        ps = [q.params(S0=o["S0"], K=o["K"], r=o["r"], sigma=o["sigma"], T=o["T"], d=d) for o in sel]
        res = q.qmccpw_price_greeks_batch([o["type"] for o in sel], ps, N, L, cfg(2, 0))
        print(f"portfolio d={d}: {len(sel)} options, price[0] {res[0].mean[0]:.6f}", flush=True)
        q.qmccpw_portfolio_path_values([o["type"] for o in sel], ps, 1, 5, 5 + 300, cfg(2, 0))
    # multi-GPU building blocks: partials over a cell range, replicate sums, device finalize
    ps = [q.params(d=64)] * 3
    n_cells, per = q.qmccpw_cell_count(ps[0], 3, N, L, cfg(1, 0))
    buf = torch.zeros(n_cells * per, dtype=torch.float64, device="cuda:0")
    rs = torch.zeros(L * per, dtype=torch.float64, device="cuda:0")
    c = cfg(1, 0)
    c.stream = torch.cuda.current_stream().cuda_stream
    q.qmccpw_partials(opts3, ps, N, L, c, 0, n_cells, buf.data_ptr())
    q.qmccpw_replicate_sums(buf.data_ptr(), ps[0], 3, N, L, c, 0, L, rs.data_ptr())
    torch.cuda.synchronize()
    q.qmccpw_finalize(rs.cpu().numpy(), opts3, ps, N, L, c)
    q.qmccpw_finalize_device(buf.data_ptr(), opts3, ps, N, L, cfg(1, 0))
    # parity hooks
    for rand in (0, 2, 4):
        q.qmccpw_sobol_u32(1, 0, 64, 1000, 3000, cfg(0, 0, rand=rand))
    q.qmccpw_normals(1, 64, 0, 2000, cfg(0, 0))
    q.qmccpw_normals(1, 64, 0, 2000, cfg(0, 0, method=1))
    for constr, cond in ((0, 0), (1, 0), (2, 0), (2, 1), (1, 1)):
        for t in (0, 1, 2):
            q.qmccpw_path_values(t, q.params(d=64), 1, 10, 10 + 500, cfg(constr, cond))
    torch.cuda.synchronize()
    print("sanitize_run: launches", q.qmccpw_launch_count(), flush=True)


if __name__ == "__main__":
    main()
