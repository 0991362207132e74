#!/bin/bash
# m1: PCA-W1 contracts with M - row 0 (W~ straight out of the DMMA, no per-date subtraction).
V=$PWD/paper_2209_11337_b200/build/var
L=gpurun_out/r02aq.log; rm -f $L
QMCCPW_LIB=$V/m1.so timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_memory_safety.py tests/test_distributed_gpu.py -m gpu -k "pca or gpca or bench_launch or c3 or poison or concurrent or distributed or owen" >> $L 2>&1; echo rc=$? >> $L
for rep in 1 2; do for lib in cur m1; do export QMCCPW_LIB=$V/$lib.so; echo "== $lib rep $rep" >> $L
  for a in "--construction 2 --conditioning 0" "--construction 3 --conditioning 0" "--construction 2 --conditioning 1"; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$a', json.loads(l)['ms_per_step']) for l in sys.stdin if l.startswith('{')]" >> $L
  done; done; done
