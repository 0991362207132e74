#!/bin/bash
# A/B timing of library variants (QMCCPW_LIB) on one GPU: smoke parity + bench per mode.
# usage: bash scripts/ab.sh lib1.so lib2.so ...   -> gpurun_out/ab.log
rm -f gpurun_out/ab.log
for rep in 1 2; do
for lib in "$@"; do
  export QMCCPW_LIB=$lib
  echo "== $lib rep $rep" >> gpurun_out/ab.log
  if [ $rep = 1 ]; then timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> gpurun_out/ab.log 2>&1; fi
  for c in ${AB_MODES:-"1,0" "0,0" "2,0"}; do IFS=, read c1 c2 <<< "$c"
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --construction $c1 --conditioning $c2 >> gpurun_out/ab.log 2>&1
  done
done
done
