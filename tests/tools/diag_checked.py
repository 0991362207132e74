"""Run each call of the every-kernel list in its own process against the checked build and
report which ones trap (a trap poisons the CUDA context, so one call per process)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CODE = """
import sys; sys.path.insert(0, {root!r})
import paper_2209_11337_b200 as q
c = q.config(method={m}, construction={c}, conditioning={k}, randomization={r}, device=0)
res = q.qmccpw_price_greeks_batch({opts}, [q.params(K=95.0, d={d})] * {n}, {N}, 2, c)
print('ok', res[0].mean[0])
"""
cases = []
for c, k in ((0, 0), (1, 0), (2, 0), (3, 0), (0, 1), (1, 1), (2, 1), (3, 1)):
    for d in (1, 4, 16, 64, 200):
        if c == 1 and d & (d - 1):
            continue
        cases.append((0, c, k, 0, [0, 1, 2], d))
for m in (1, 2, 3):
    cases.append((m, 0, 0, 0, [0, 1, 2], 64))
cases.append((0, 1, 0, 4, [0, 1, 2], 64))
cases.append((0, 2, 1, 4, [0, 1, 2], 64))
for N in (4096 + 77, 100):
    for m, c, k, r, opts, d in cases:
        code = CODE.format(root=ROOT, m=m, c=c, k=k, r=r, opts=opts, n=len(opts), d=d, N=N)
        p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=dict(os.environ))
        status = "ok" if p.returncode == 0 else ("TRAP " + (p.stderr.strip().splitlines() or ["?"])[-1][:100])
        print(f"N={N} method={m} constr={c} cond={k} rand={r} d={d}: {status}", flush=True)
