#!/bin/bash
# xt: X1 date table (c_j offsets, R_j - sigma t) in the PCA quad kernel; ic3: + central Phi^-1
# coefficients from shared memory (interleaved chains) in the W1 units.  Parity + A/B.
V=$PWD/paper_2209_11337_b200/build/var
L=gpurun_out/r02ai.log; rm -f $L
QMCCPW_LIB=$V/ic3.so timeout 900 python -m pytest -q -x tests/ -m gpu >> $L 2>&1; echo rc=$? >> $L
for rep in 1 2; do for lib in cur xt ic3; do export QMCCPW_LIB=$V/$lib.so; echo "== $lib rep $rep" >> $L
  for a in "--construction 1 --conditioning 0" "--construction 0 --conditioning 0" "--construction 2 --conditioning 0" "--construction 2 --conditioning 1" "--construction 1 --conditioning 1" "--construction 2 --conditioning 1 --options 0,1,2"; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$a', json.loads(l)['ms_per_step']) for l in sys.stdin if l.startswith('{')]" >> $L
  done; done; done
