#!/bin/bash
V=$PWD/paper_2209_11337_b200/build/var
QMCCPW_LIB=$V/new.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_distributed_gpu.py -q -k "portfolio or c5 or path_values or c4_fused or c3_full or deep or configs or gpca" > gpurun_out/r02l_parity_new.log 2>&1; echo rc=$? >> gpurun_out/r02l_parity_new.log
rm -f gpurun_out/ab.log
for rep in 1 2; do for lib in $V/old.so $V/new.so $V/bpipe.so; do
  for m in "--workload C5" "--construction 2 --conditioning 1" "--construction 1 --conditioning 1" "--construction 2 --conditioning 0"; do
    echo "== $lib $m" >> gpurun_out/ab.log
    QMCCPW_LIB=$lib timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline $m >> gpurun_out/ab.log 2>&1
  done; done; done
cp gpurun_out/ab.log gpurun_out/r02l_ab.log
