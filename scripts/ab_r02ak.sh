#!/bin/bash
# vg: PCA kernels read the direction numbers from global memory (8 KB less shared memory per
# block: smaller carveout, more L1).  Parity + A/B.
V=$PWD/paper_2209_11337_b200/build/var
L=gpurun_out/r02ak.log; rm -f $L
QMCCPW_LIB=$V/vg.so timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_memory_safety.py -m gpu -k "pca or x1 or lookback or bench_launch or sobol or owen or portfolio or poison or concurrent" >> $L 2>&1; echo rc=$? >> $L
for rep in 1 2; do for lib in cur vg; do export QMCCPW_LIB=$V/$lib.so; echo "== $lib rep $rep" >> $L
  for a in "--construction 2 --conditioning 0" "--construction 2 --conditioning 1" "--construction 1 --conditioning 1" "--construction 2 --conditioning 1 --options 0,1,2" "--construction 2 --conditioning 1 --randomization 4"; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$a', json.loads(l)['ms_per_step']) for l in sys.stdin if l.startswith('{')]" >> $L
  done; done; done
