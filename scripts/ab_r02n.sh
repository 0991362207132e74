#!/bin/bash
V=$PWD/paper_2209_11337_b200/build/var
QMCCPW_LIB=$V/x3f.so timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "path_values or c4_fused or c3 or bench_launch or edge or mc_ or owen or configs" > gpurun_out/r02n_parity_x3f.log 2>&1; echo rc=$? >> gpurun_out/r02n_parity_x3f.log
AB_MODES="1,0" bash scripts/ab.sh $V/base.so $V/x3.so $V/f.so $V/x3f.so; cp gpurun_out/ab.log gpurun_out/r02n_ab.log
