#!/bin/bash
# ms: the upper-half mirror of Phi^-1 as a sign-bit XOR instead of a negation and two selects.
V=$PWD/paper_2209_11337_b200/build/var
L=gpurun_out/r02an.log; rm -f $L
QMCCPW_LIB=$V/ms.so timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -m gpu -k "normal or sobol or bench_launch or path_values" >> $L 2>&1; echo rc=$? >> $L
for rep in 1 2; do for lib in cur ms; do export QMCCPW_LIB=$V/$lib.so; echo "== $lib rep $rep" >> $L
  for a in "--construction 1 --conditioning 0" "--construction 0 --conditioning 0" "--construction 2 --conditioning 0" "--construction 2 --conditioning 1" "--workload C5"; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$a', json.loads(l)['ms_per_step']) for l in sys.stdin if l.startswith('{')]" >> $L
  done; done; done
