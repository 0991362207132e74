#!/bin/bash
# register caps re-checked after the round-2 changes: BB-W1 at 7 blocks/SM, STD-W1 at 8.
V=$PWD/paper_2209_11337_b200/build/var
L=gpurun_out/r02ay.log; rm -f $L
for rep in 1 2; do for lib in cur bb7 st8; do export QMCCPW_LIB=$V/$lib.so; echo "== $lib rep $rep" >> $L
  for a in "--construction 1 --conditioning 0" "--construction 0 --conditioning 0"; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$a', json.loads(l)['ms_per_step']) for l in sys.stdin if l.startswith('{')]" >> $L
  done; done; done
