"""Markdown table of a bench_all_modes.jsonl (one bench.py line per mode):

    python scripts/modes_table.py profiles/r02/r02z3_bench_all_modes.jsonl
"""
import json
import sys


def mode_name(j):
    w = j["config"]["workload"]
    if w.startswith("C5"):
        return "C5 portfolio (1024 options, d = 128)"
    tail = w.split("d=64, ", 1)[-1]
    n = j["config"].get("points_per_replicate", 0) * j["config"].get("replicates_total", 0)
    if n and n != 67108864:
        tail += f", {n / 2**20:.0f} Mi paths"
    if j.get("scaling") == "weak":
        tail += ", weak scaling"
    return tail


def main(path):
    print("| Mode | ms/step | paths/s | model frac | ncu FP64 (+DMMA) |")
    print("|---|---|---|---|---|")
    for line in open(path):
        if not line.startswith("{"):
            continue
        j = json.loads(line)
        r = j.get("roofline", {})
        ncu = r.get("ncu") or {}
        pct = ncu.get("fp64_plus_dmma_pct")
        pct_s = f"{pct:.1f} %" if pct is not None else "—"
        print(f"| {mode_name(j)} | {j['ms_per_step']:.2f} | {j['value']:.3g} | {r.get('frac', float('nan')):.2f} | {pct_s} |")


if __name__ == "__main__":
    main(sys.argv[1])
