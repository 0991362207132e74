#!/bin/bash
V=$PWD/paper_2209_11337_b200/build/var
QMCCPW_LIB=$V/p4.so timeout 300 python -m pytest -q -x tests/test_gpu_parity.py -k "test_path_values and -1-0]" > gpurun_out/r02ac_quick.log 2>&1; echo rc=$? >> gpurun_out/r02ac_quick.log
QMCCPW_LIB=$V/p4.so timeout 300 python -m pytest -q -x tests/test_gpu_parity.py -k "bench_launch or c4_fused" >> gpurun_out/r02ac_quick.log 2>&1; echo rc=$? >> gpurun_out/r02ac_quick.log
AB_MODES="1,0" bash scripts/ab.sh $V/p0.so $V/p4.so; cp gpurun_out/ab.log gpurun_out/r02ac_ab.log
