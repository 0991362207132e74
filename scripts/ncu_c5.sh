#!/bin/bash
# C5 portfolio: bench line, then one ncu --set full capture of portfolio_kernel
timeout 600 python bench.py --workload C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:portfolio_kernel -c 1 \
  -o gpurun_out/c5_full -f python bench.py --workload C5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c5.log 2>&1
echo ncu_c5=$? >> gpurun_out/rc.txt
