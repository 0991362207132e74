#!/bin/bash
V=$PWD/paper_2209_11337_b200/build/var
QMCCPW_LIB=$V/bm.so timeout 120 python -m pytest -q -x "tests/test_gpu_parity.py::test_path_values[64-0-1-1]" "tests/test_gpu_parity.py::test_path_values[4-1-1-1]" > gpurun_out/r02u_quick.log 2>&1; echo rc=$? >> gpurun_out/r02u_quick.log
grep -q "rc=0" gpurun_out/r02u_quick.log || exit 3
QMCCPW_LIB=$V/bm.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_memory_safety.py -q -k "path_values or c4_fused or configs or owen or deep or edge or d256 or memory or partials or repeated" > gpurun_out/r02u_parity_bm.log 2>&1; echo rc=$? >> gpurun_out/r02u_parity_bm.log
AB_MODES="1,1" bash scripts/ab.sh $V/bo.so $V/bm.so; cp gpurun_out/ab.log gpurun_out/r02u_ab.log
