#!/bin/bash
# pe: the portfolio unit's exp from the 256-entry table (through L1), degree 4.
V=$PWD/paper_2209_11337_b200/build/var
L=gpurun_out/r02be.log; rm -f $L
QMCCPW_LIB=$V/pe.so timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -m gpu -k "portfolio or c5" >> $L 2>&1; echo rc=$? >> $L
for rep in 1 2; do for lib in cur pe; do export QMCCPW_LIB=$V/$lib.so; echo "== $lib rep $rep" >> $L
  for a in "--workload C5"; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$a', json.loads(l)['ms_per_step']) for l in sys.stdin if l.startswith('{')]" >> $L
  done; done; done
