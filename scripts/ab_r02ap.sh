#!/bin/bash
# PCA-W1 register cap re-checked after the round-2 changes: 8 (cur), 7, 6 blocks/SM.
V=$PWD/paper_2209_11337_b200/build/var
L=gpurun_out/r02ap.log; rm -f $L
for rep in 1 2 3; do for lib in cur pw7 pw6; do export QMCCPW_LIB=$V/$lib.so; echo "== $lib rep $rep" >> $L
  for a in "--construction 2 --conditioning 0" "--construction 3 --conditioning 0"; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$a', json.loads(l)['ms_per_step']) for l in sys.stdin if l.startswith('{')]" >> $L
  done; done; done
