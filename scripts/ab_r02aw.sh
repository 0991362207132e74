#!/bin/bash
# h4: BB-W1's terminal and group 0's first three descent normals as one four-way batch.
V=$PWD/paper_2209_11337_b200/build/var
L=gpurun_out/r02aw.log; rm -f $L
QMCCPW_LIB=$V/h4.so timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_memory_safety.py -m gpu -k "bb or bench_launch or c3 or c1 or poison or concurrent or owen or path_values" >> $L 2>&1; echo rc=$? >> $L
for rep in 1 2; do for lib in cur h4; do export QMCCPW_LIB=$V/$lib.so; echo "== $lib rep $rep" >> $L
  for a in "--construction 1 --conditioning 0" "--construction 1 --conditioning 0 --randomization 4"; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$a', json.loads(l)['ms_per_step']) for l in sys.stdin if l.startswith('{')]" >> $L
  done; done; done
