#!/bin/bash
V=$PWD/paper_2209_11337_b200/build/var
QMCCPW_LIB=$V/sm.so timeout 120 python -m pytest -q -x "tests/test_gpu_parity.py::test_path_values[64-0-0-1]" "tests/test_gpu_parity.py::test_path_values[4-1-0-1]" "tests/test_gpu_parity.py::test_path_values[1-0-0-1]" > gpurun_out/r02w_quick.log 2>&1; echo rc=$? >> gpurun_out/r02w_quick.log
grep -q "rc=0" gpurun_out/r02w_quick.log || exit 3
QMCCPW_LIB=$V/sm.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_distributed_gpu.py -q -k "path_values or c4_fused or configs or owen or deep or edge or d256 or std or x1" > gpurun_out/r02w_parity_sm.log 2>&1; echo rc=$? >> gpurun_out/r02w_parity_sm.log
AB_MODES="0,1 1,1 2,1" bash scripts/ab.sh $V/so.so $V/sm.so; cp gpurun_out/ab.log gpurun_out/r02w_ab.log
