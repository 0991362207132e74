#!/bin/bash
# fx: no date table in the X1 PCA kernels (back under the 196 KiB carveout); pt: + PCA-W1 exp/log
# tables through L1 (its date table then fits the 196 KiB carveout too).  Parity + A/B.
V=$PWD/paper_2209_11337_b200/build/var
L=gpurun_out/r02aj.log; rm -f $L
QMCCPW_LIB=$V/pt.so timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -m gpu -k "pca or x1 or lookback or bench_launch" >> $L 2>&1; echo rc=$? >> $L
for rep in 1 2; do for lib in cur fx pt; do export QMCCPW_LIB=$V/$lib.so; echo "== $lib rep $rep" >> $L
  for a in "--construction 2 --conditioning 0" "--construction 2 --conditioning 1" "--construction 1 --conditioning 1" "--construction 2 --conditioning 1 --options 0,1,2"; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$a', json.loads(l)['ms_per_step']) for l in sys.stdin if l.startswith('{')]" >> $L
  done; done; done
