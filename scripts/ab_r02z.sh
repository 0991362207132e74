#!/bin/bash
V=$PWD/paper_2209_11337_b200/build/var
QMCCPW_LIB=$V/ss6.so timeout 120 python -m pytest -q -x "tests/test_gpu_parity.py::test_path_values[64-0-0-1]" "tests/test_gpu_parity.py::test_path_values[4-1-0-1]" "tests/test_gpu_parity.py::test_path_values[1-2-0-1]" "tests/test_gpu_parity.py::test_path_values[64-2-0-1]" > gpurun_out/r02z_quick.log 2>&1; echo rc=$? >> gpurun_out/r02z_quick.log
grep -q "rc=0" gpurun_out/r02z_quick.log || exit 3
QMCCPW_LIB=$V/ss6.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "path_values or c4_fused or configs or owen or deep or edge or std" > gpurun_out/r02z_parity.log 2>&1; echo rc=$? >> gpurun_out/r02z_parity.log
rm -f gpurun_out/ab.log
for rep in 1 2; do for lib in $V/sso.so $V/ss4.so $V/ss6.so $V/ss8.so; do for o in "" "--options 0,1,2"; do
 echo "== $lib $o" >> gpurun_out/ab.log
 QMCCPW_LIB=$lib timeout 120 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --construction 0 --conditioning 1 $o >> gpurun_out/ab.log 2>&1; done; done; done
cp gpurun_out/ab.log gpurun_out/r02z_ab.log
