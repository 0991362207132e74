#!/bin/bash
V=$PWD/paper_2209_11337_b200/build/var
QMCCPW_LIB=$V/lqb.so timeout 120 python -m pytest -q -x "tests/test_gpu_parity.py::test_path_values[64-2-2-1]" "tests/test_gpu_parity.py::test_path_values[16-2-2-1]" > gpurun_out/r02v_quick.log 2>&1; echo rc=$? >> gpurun_out/r02v_quick.log
grep -q "rc=0" gpurun_out/r02v_quick.log || exit 3
QMCCPW_LIB=$V/lqb.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "path_values or c4_fused or deep or gpca or owen or pca or c3_full" > gpurun_out/r02v_parity.log 2>&1; echo rc=$? >> gpurun_out/r02v_parity.log
rm -f gpurun_out/ab_lb.log
for rep in 1 2; do for lib in $V/lq5base.so $V/lqb.so; do echo "== $lib" >> gpurun_out/ab_lb.log
 QMCCPW_LIB=$lib timeout 120 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --construction 2 --conditioning 1 --options 0,1,2 >> gpurun_out/ab_lb.log 2>&1; done; done
cp gpurun_out/ab_lb.log gpurun_out/r02v_ab_lb.log
