#!/bin/bash
# parity + bench (as gpu_check.sh), then one ncu --set full capture of the headline paths kernel
bash scripts/gpu_check.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:paths_kernel -c 1 \
  -o gpurun_out/paths_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo ncu=$? >> gpurun_out/rc.txt
