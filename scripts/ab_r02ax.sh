#!/bin/bash
# s4: STD-W1 four dates per step (four-chain normals).
V=$PWD/paper_2209_11337_b200/build/var
L=gpurun_out/r02ax.log; rm -f $L
QMCCPW_LIB=$V/s4.so timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -m gpu -k "std or bench_launch or c1 or owen or path_values" >> $L 2>&1; echo rc=$? >> $L
for rep in 1 2; do for lib in cur s4; do export QMCCPW_LIB=$V/$lib.so; echo "== $lib rep $rep" >> $L
  for a in "--construction 0 --conditioning 0" "--construction 1 --conditioning 0"; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$a', json.loads(l)['ms_per_step']) for l in sys.stdin if l.startswith('{')]" >> $L
  done; done; done
