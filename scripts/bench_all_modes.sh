#!/bin/bash
# every mode's bench line (C4 unless noted) -> gpurun_out/bench_all_modes.jsonl
out=gpurun_out/bench_all_modes.jsonl; rm -f $out
run() { timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline "$@" 2>/dev/null | grep '^{' >> $out; }
for c in "1 0 0" "0 0 0" "2 0 0" "3 0 0" "2 1 0" "3 1 0" "0 1 0" "1 1 0" "1 0 4" "2 1 4"; do set -- $c
  run --construction $1 --conditioning $2 --randomization $3
done
for c in "2 1" "1 1" "0 1"; do set -- $c; run --construction $1 --conditioning $2 --options 0,1,2; done   # f1
for c in "1 0" "2 0" "2 1" "3 0" "3 1"; do set -- $c; run --method $1 --construction $2; done                 # f2
timeout 600 python bench.py --workload C5 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | grep '^{' >> $out
timeout 600 python bench.py --points 8388608 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | grep '^{' >> $out   # x8 variant of C4
timeout 600 python bench.py --scaling weak --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | grep '^{' >> $out
