#!/bin/bash
# xe: X1 units' exp from the 256-entry table (through L1) with the degree-4 polynomial.
V=$PWD/paper_2209_11337_b200/build/var
L=gpurun_out/r02bd.log; rm -f $L
QMCCPW_LIB=$V/xe.so timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -m gpu -k "x1 or lookback or bench_launch or d256 or owen" >> $L 2>&1; echo rc=$? >> $L
for rep in 1 2; do for lib in cur xe; do export QMCCPW_LIB=$V/$lib.so; echo "== $lib rep $rep" >> $L
  for a in "--construction 2 --conditioning 1" "--construction 1 --conditioning 1" "--construction 0 --conditioning 1" "--construction 2 --conditioning 1 --options 0,1,2" "--construction 1 --conditioning 1 --options 0,1,2"; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$a', json.loads(l)['ms_per_step']) for l in sys.stdin if l.startswith('{')]" >> $L
  done; done; done
