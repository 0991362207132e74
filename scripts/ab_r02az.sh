#!/bin/bash
# e256: W1 units' exp from a 256-entry table with a degree-4 polynomial (one DFMA fewer, same fit
# error).  Parity + A/B.
V=$PWD/paper_2209_11337_b200/build/var
L=gpurun_out/r02az.log; rm -f $L
QMCCPW_LIB=$V/e256.so timeout 1200 python -m pytest -q -x tests/ -m gpu >> $L 2>&1; echo rc=$? >> $L
for rep in 1 2; do for lib in cur e256; do export QMCCPW_LIB=$V/$lib.so; echo "== $lib rep $rep" >> $L
  for a in "--construction 1 --conditioning 0" "--construction 0 --conditioning 0" "--construction 2 --conditioning 0" "--method 3 --construction 1" "--workload C5"; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$a', json.loads(l)['ms_per_step']) for l in sys.stdin if l.startswith('{')]" >> $L
  done; done; done
