import csv, re, sys, collections
raw, cs, sass = sys.argv[1:4]
rows = list(csv.reader(open(raw))); a = dict(zip(rows[0], rows[2])); u = dict(zip(rows[0], rows[1]))
for k in ['gpu__time_duration.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
          'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.per_cycle_active',
          'launch__registers_per_thread', 'smsp__inst_executed.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
          'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
          'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active']:
    print(f"{k:70s} {a.get(k)} {u.get(k)}")
st = [(k, float(a[k] or 0)) for k in a if 'pcsamp_warps_issue_stalled' in k and not k.endswith('not_issued')]
tot = sum(v for _, v in st)
print("stalls:", ", ".join(f"{k.split('stalled_')[1]}={v/tot*100:.1f}%" for k, v in sorted(st, key=lambda x: -x[1])[:8]))
rows = list(csv.reader(open(sass))); hdr = rows[1]; ie = hdr.index("Instructions Executed"); src = hdr.index("Source")
op = collections.Counter(); n_all = 0
paths = int(sys.argv[4]) if len(sys.argv) > 4 else 2 ** 26  # points per launch
for r in rows[2:]:
    try: n = int(r[ie])
    except: continue
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[src]); op[m.group(2) if m else '?'] += n; n_all += n
print("warp-instr per path %.0f" % (n_all * 32 / paths))
print(", ".join(f"{o}:{n*32/paths:.0f}" for o, n in op.most_common(24)))
rows = list(csv.reader(open(cs))); hdr = rows[2]; ie = hdr.index("Instructions Executed"); sti = hdr.index("Warp Stall Sampling (All Samples)")
per = collections.Counter(); stall = collections.Counter(); text = {}; fname = None; cur = None
for r in rows:
    if r and r[0] == 'File Path': fname = r[1].split('/')[-1]; continue
    if not r or r[0] in ('Function Name', 'Line No'): continue
    if r[0] != '': cur = (fname, r[0]); text[cur] = r[1][:70]; continue
    try: per[cur] += int(r[ie]); stall[cur] += int(r[sti] or 0)
    except: pass
ts = sum(stall.values())
for k, n in stall.most_common(16):
    print(f"stall {n/ts*100:5.1f}% instr {per[k]*32/paths:7.0f}/path {k[0]}:{k[1]} {text.get(k,'')}")
