#!/bin/bash
# one ncu --set full capture of the first paths/pca kernel of a bench mode: bash scripts/ncu_one.sh NAME CONSTR COND
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"paths_kernel|pca_kernel" -c 1 \
  -o gpurun_out/$1 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --construction $2 --conditioning $3 > gpurun_out/ncu_$1.log 2>&1
echo ncu_$1=$? >> gpurun_out/rc.txt
