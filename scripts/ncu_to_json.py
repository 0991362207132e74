"""Summarise one ncu --set full capture (.ncu-rep) of a dominant kernel:

    python scripts/ncu_to_json.py REPORT.ncu-rep KEY PATHS_PER_LAUNCH [--build TEXT] [--out profiles/x.txt]

* writes the headline counters into profiles/ncu_metrics.json under KEY (the bench mode key
  bench.py looks up: "BB-W1", "PCA-W1", "PCA-X1", "C5", ...): FP64 pipe, issue, SFU (xu)
  utilisation, warps active, registers, DRAM bytes per launch -- bench.py copies them into
  the JSON line's roofline object;
* prints (and with --out writes) a text summary: counters, the stall mix, the SASS opcode mix
  per path and the top stalled source lines (scripts/ncu_summary.py's format).
"""
import argparse
import collections
import csv
import io
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COUNTERS = ['gpu__time_duration.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
            'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.per_cycle_active',
            'launch__registers_per_thread', 'smsp__inst_executed.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
            'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
            'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
            'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
            'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
            'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
            'sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active',
            'launch__occupancy_limit_registers', 'launch__shared_mem_per_block_dynamic', 'launch__block_size',
            'smsp__thread_inst_executed_per_inst_executed.ratio']
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
              "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, "--csv"] + list(args), capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("key")
    ap.add_argument("paths", type=float, help="paths (underlying QMC points) per launch")
    ap.add_argument("--build", default="")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = ncu_csv(a.report, "--page", "raw")
    hdr, units, vals = rows[0], rows[1], rows[2]
    raw = dict(zip(hdr, vals))
    unit = dict(zip(hdr, units))
    lines = [f"kernel: {raw.get('Kernel Name', '?')[:120]}"]
    for k in COUNTERS:
        lines.append(f"{k:70s} {raw.get(k)} {unit.get(k, '')}")

    def num(k):
        v = raw.get(k, "")
        try:
            return float(str(v).replace(",", "")) * UNIT_SCALE.get(unit.get(k, ""), 1.0)
        except ValueError:
            return None
    st = [(k, float(raw[k] or 0)) for k in raw if 'pcsamp_warps_issue_stalled' in k and not k.endswith('not_issued')]
    tot = sum(v for _, v in st) or 1.0
    lines.append("stalls: " + ", ".join(f"{k.split('stalled_')[1]}={v / tot * 100:.1f}%"
                                        for k, v in sorted(st, key=lambda x: -x[1])[:10]))
    # SASS opcode mix per path
    srows = ncu_csv(a.report, "--page", "source", "--print-source", "sass")
    hi = next(i for i, r in enumerate(srows) if "Instructions Executed" in r)
    h = srows[hi]
    ie, src = h.index("Instructions Executed"), h.index("Source")
    op = collections.Counter()
    n_all = 0
    for r in srows[hi + 1:]:
        try:
            n = int(r[ie])
        except (ValueError, IndexError):
            continue
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[src])
        op[m.group(2) if m else '?'] += n
        n_all += n
    # lane-instructions per path: every warp instruction serves 32 lanes (paths, or a quad's share)
    per_path = 32.0 / a.paths
    lines.append("instr per path %.0f" % (n_all * per_path))
    lines.append(", ".join(f"{o}:{n * per_path:.0f}" for o, n in op.most_common(28)))
    fp64 = sum(op[o] for o in ("DFMA", "DMUL", "DADD", "DSETP")) * per_path
    dmma = op["DMMA"] * per_path
    lines.append(f"FP64 vector instr per path {fp64:.0f} ({100 * fp64 / max(n_all * per_path, 1):.1f} % of issued), "
                 f"DMMA {dmma:.1f}")
    # top stalled CUDA source lines
    crows = ncu_csv(a.report, "--page", "source", "--print-source", "cuda,sass")
    per, stall, text = collections.Counter(), collections.Counter(), {}
    fname, hdrc = None, None
    for r in crows:
        if r and r[0] == 'File Path':
            fname = r[1].split('/')[-1]
            continue
        if r and r[0] == 'Line No':
            hdrc = r
            continue
        # per-line aggregate rows carry "-" in the SASS address column
        if not r or hdrc is None or fname is None or len(r) < 8 or r[2] != '-':
            continue
        try:
            key = (fname, r[0])
            text[key] = r[1][:80]
            per[key] += int(r[7] or 0)
            stall[key] += int(float(r[4] or 0))
        except ValueError:
            continue
    ts = sum(stall.values()) or 1
    for k, n in stall.most_common(20):
        lines.append(f"stall {n / ts * 100:5.1f}% instr {per[k] * per_path:7.1f}/path {k[0]}:{k[1]} {text.get(k, '')}")
    if a.build:
        lines.append(f"({a.build})")
    txt = "\n".join(lines)
    print(txt)
    if a.out:
        open(a.out, "w").write(txt + "\n")
    path = os.path.join(ROOT, "profiles", "ncu_metrics.json")
    db = json.load(open(path)) if os.path.exists(path) else {}
    rd, wr = num('dram__bytes_read.sum'), num('dram__bytes_write.sum')
    db[a.key] = {
        "fp64_pipe_pct": num('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'),
        # DMMA (FP64 tensor core): same per-SM FMA rate as the vector pipe (qmccpw_fp64_roof), so the
        # FP64 datapath's utilisation is the sum of the two
        "dmma_pipe_pct": num('sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active') or 0.0,
        "issue_active_pct": num('smsp__issue_active.avg.pct_of_peak_sustained_active'),
        "xu_pipe_pct": num('sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active'),
        "warps_active": num('sm__warps_active.avg.per_cycle_active'),
        "registers": num('launch__registers_per_thread'),
        "kernel_ms": num('gpu__time_duration.sum'),
        "dram_bytes_per_launch": (rd or 0) + (wr or 0) if rd is not None else None,
        "instr_per_path": n_all * per_path, "fp64_instr_per_path": fp64, "dmma_instr_per_path": dmma,
        "build": a.build, "source": os.path.relpath(a.out, ROOT) if a.out else os.path.basename(a.report),
    }
    db[a.key]["fp64_plus_dmma_pct"] = (db[a.key]["fp64_pipe_pct"] or 0.0) + db[a.key]["dmma_pipe_pct"]
    json.dump(db, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
