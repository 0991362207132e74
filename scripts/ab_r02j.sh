#!/bin/bash
V=$PWD/paper_2209_11337_b200/build/var
QMCCPW_LIB=$V/lbS.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "path_values or c4_fused or c3_full or deep" -x > gpurun_out/r02j_parity_lbS.log 2>&1; echo rc=$? >> gpurun_out/r02j_parity_lbS.log
rm -f gpurun_out/ab_lb.log
for rep in 1 2; do for lib in $V/lb0.so $V/lbS.so $V/lbSH.so; do for c in 2 1; do echo "== $lib $c" >> gpurun_out/ab_lb.log
 QMCCPW_LIB=$lib timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --construction $c --conditioning 1 --options 0,1,2 >> gpurun_out/ab_lb.log 2>&1; done; done; done
cp gpurun_out/ab_lb.log gpurun_out/r02j_ab_lb.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02j_bench_default.jsonl 2>&1
