#!/bin/bash
V=$PWD/paper_2209_11337_b200/build/var
timeout 120 python -m pytest -q -x "tests/test_gpu_parity.py::test_path_values[64-0-0-1]" "tests/test_gpu_parity.py::test_path_values[4-1-0-1]" "tests/test_gpu_parity.py::test_path_values[1-0-0-1]" > gpurun_out/r02x_quick.log 2>&1; echo rc=$? >> gpurun_out/r02x_quick.log
grep -q "rc=0" gpurun_out/r02x_quick.log || exit 3
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/r02x_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r02x_pytest_gpu.log
AB_MODES="0,1 1,1 2,1 1,0" bash scripts/ab.sh $V/cur.so; cp gpurun_out/ab.log gpurun_out/r02x_ab.log
