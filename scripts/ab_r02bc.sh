#!/bin/bash
# BB-W1 normal grouping re-checked on the final code: nx3 = the group's last three normals as 2 + 1
# instead of three chains; n1i = the rare single normals inlined instead of out of line.
V=$PWD/paper_2209_11337_b200/build/var
L=gpurun_out/r02bc.log; rm -f $L
for rep in 1 2; do for lib in cur nx3 n1i; do export QMCCPW_LIB=$V/$lib.so; echo "== $lib rep $rep" >> $L
  for a in "--construction 1 --conditioning 0"; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$a', json.loads(l)['ms_per_step']) for l in sys.stdin if l.startswith('{')]" >> $L
  done; done; done
