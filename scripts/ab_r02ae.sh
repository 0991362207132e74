#!/bin/bash
# X1 lookback: per-date loop unroll 1 vs 2 on the LB quad kernel, and the r02y build
V=$PWD/paper_2209_11337_b200/build/var
L=gpurun_out/r02ae.log; rm -f $L
QMCCPW_LIB=$V/lbu1.so timeout 300 python -m pytest -q -x tests/test_gpu_parity.py -k "lookback" >> $L 2>&1; echo rc=$? >> $L
for rep in 1 2; do for lib in old lbu1 r02y; do export QMCCPW_LIB=$V/$lib.so; echo "== $lib rep $rep" >> $L
  for a in "--construction 2 --conditioning 1 --options 0,1,2" "--construction 2 --conditioning 1"; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$a', json.loads(l)['ms_per_step']) for l in sys.stdin if l.startswith('{')]" >> $L
  done; done; done
