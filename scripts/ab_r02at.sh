#!/bin/bash
# lg: log1p(r) + ln c_i as fma(r, fma(r, L, 1), ln c_i) (two FP64 ops instead of three, one
# rounding fewer).  Parity + A/B.
V=$PWD/paper_2209_11337_b200/build/var
L=gpurun_out/r02at.log; rm -f $L
QMCCPW_LIB=$V/lg2.so timeout 1200 python -m pytest -q -x tests/ -m gpu >> $L 2>&1; echo rc=$? >> $L
for rep in 1 2; do for lib in cur lg2; do export QMCCPW_LIB=$V/$lib.so; echo "== $lib rep $rep" >> $L
  for a in "--construction 1 --conditioning 0" "--construction 0 --conditioning 0" "--construction 2 --conditioning 0" "--construction 2 --conditioning 1" "--workload C5"; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$a', json.loads(l)['ms_per_step']) for l in sys.stdin if l.startswith('{')]" >> $L
  done; done; done
