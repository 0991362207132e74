#!/bin/bash
# x2s: the path-kernel unit's paired normals also through the shifted-log four-chain form (now that
# STD-W1 runs four dates per step, the pairs are the MC methods' and the remainders).
V=$PWD/paper_2209_11337_b200/build/var
L=gpurun_out/r02ba.log; rm -f $L
QMCCPW_LIB=$V/x2s.so timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -m gpu -k "std or mc or bench_launch or c1 or normal" >> $L 2>&1; echo rc=$? >> $L
for rep in 1 2; do for lib in cur x2s; do export QMCCPW_LIB=$V/$lib.so; echo "== $lib rep $rep" >> $L
  for a in "--construction 1 --conditioning 0" "--construction 0 --conditioning 0" "--method 2 --construction 0" "--method 3 --construction 1" "--method 1 --construction 0"; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$a', json.loads(l)['ms_per_step']) for l in sys.stdin if l.startswith('{')]" >> $L
  done; done; done
