#!/bin/bash
# pf: portfolio kernel reads the direction numbers from global memory (16 KB less shared memory
# per block at d = 128).  Parity + A/B.
V=$PWD/paper_2209_11337_b200/build/var
L=gpurun_out/r02am.log; rm -f $L
QMCCPW_LIB=$V/pf.so timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_memory_safety.py -m gpu -k "portfolio or c5 or poison or concurrent" >> $L 2>&1; echo rc=$? >> $L
for rep in 1 2; do for lib in cur pf; do export QMCCPW_LIB=$V/$lib.so; echo "== $lib rep $rep" >> $L
  for a in "--workload C5"; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$a', json.loads(l)['ms_per_step']) for l in sys.stdin if l.startswith('{')]" >> $L
  done; done; done
