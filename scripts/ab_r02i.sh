#!/bin/bash
V=$PWD/paper_2209_11337_b200/build/var
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mix paper_2209_11337_b200/tools/fp64_mix_bench.cu && /tmp/mix > gpurun_out/r02i_mix.log 2>&1
QMCCPW_LIB=$V/gPN.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "path_values or c4_fused or bench_launch or edge" -x > gpurun_out/r02i_parity_gPN.log 2>&1; echo rc=$? >> gpurun_out/r02i_parity_gPN.log
QMCCPW_LIB=$V/lbNew.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "path_values or c4_fused or c3_full or deep" -x > gpurun_out/r02i_parity_lb.log 2>&1; echo rc=$? >> gpurun_out/r02i_parity_lb.log
AB_MODES="1,0" bash scripts/ab.sh $V/g0.so $V/gP.so $V/gN.so $V/gPN.so $V/gPN7.so; cp gpurun_out/ab.log gpurun_out/r02i_ab_bb.log
rm -f gpurun_out/ab_lb.log
for rep in 1 2; do for lib in $V/lbOld.so $V/lbNew.so; do echo "== $lib" >> gpurun_out/ab_lb.log
 QMCCPW_LIB=$lib timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --construction 2 --conditioning 1 --options 0,1,2 >> gpurun_out/ab_lb.log 2>&1; done; done
cp gpurun_out/ab_lb.log gpurun_out/r02i_ab_lb.log
