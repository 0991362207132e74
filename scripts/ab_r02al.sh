#!/bin/bash
# pr: X1 lookback walk scans only each lane's own upper-envelope lines (pruned by a bit-mask
# stack pass before the walk).  Parity + A/B.
V=$PWD/paper_2209_11337_b200/build/var
L=gpurun_out/r02al.log; rm -f $L
QMCCPW_LIB=$V/pr.so timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -m gpu -k "lookback or x1 or bench_launch or c3 or d256 or owen" >> $L 2>&1; echo rc=$? >> $L
for rep in 1 2; do for lib in cur pr; do export QMCCPW_LIB=$V/$lib.so; echo "== $lib rep $rep" >> $L
  for a in "--construction 2 --conditioning 1 --options 0,1,2" "--construction 3 --conditioning 1 --options 0,1,2" "--construction 2 --conditioning 1"; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$a', json.loads(l)['ms_per_step']) for l in sys.stdin if l.startswith('{')]" >> $L
  done; done; done
