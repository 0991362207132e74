#!/bin/bash
# slope table in shared memory for the X1 quad kernels: parity quick + A/B PCA-X1, BB-X1, PCA-X1 LB
V=$PWD/paper_2209_11337_b200/build/var
L=gpurun_out/r02ad.log; rm -f $L
QMCCPW_LIB=$V/aq.so timeout 300 python -m pytest -q -x tests/test_gpu_parity.py -k "x1 or lookback or bench_launch" >> $L 2>&1; echo rc=$? >> $L
for rep in 1 2; do for lib in old aq; do export QMCCPW_LIB=$V/$lib.so; echo "== $lib rep $rep" >> $L
  for a in "--construction 2 --conditioning 1" "--construction 1 --conditioning 1" "--construction 2 --conditioning 1 --options 0,1,2" "--construction 1 --conditioning 1 --options 0,1,2"; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print(json.loads(l)['config'].get('mode', ''), '$a', json.loads(l)['ms_per_step']) for l in sys.stdin if l.startswith('{')]" >> $L
  done; done; done
