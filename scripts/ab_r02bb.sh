#!/bin/bash
# x4b: PCA-X1 and the X1 lookback at 4 blocks/SM (128 registers) instead of 5 (96).
V=$PWD/paper_2209_11337_b200/build/var
L=gpurun_out/r02bb.log; rm -f $L
for rep in 1 2; do for lib in cur x4b; do export QMCCPW_LIB=$V/$lib.so; echo "== $lib rep $rep" >> $L
  for a in "--construction 2 --conditioning 1" "--construction 1 --conditioning 1" "--construction 2 --conditioning 1 --options 0,1,2"; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$a', json.loads(l)['ms_per_step']) for l in sys.stdin if l.startswith('{')]" >> $L
  done; done; done
