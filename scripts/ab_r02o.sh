#!/bin/bash
V=$PWD/paper_2209_11337_b200/build/var
QMCCPW_LIB=$V/sc5.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_distributed_gpu.py -q -k "path_values or c4_fused or deep or configs or gpca or pca or owen or x1" > gpurun_out/r02o_parity_sc5.log 2>&1; echo rc=$? >> gpurun_out/r02o_parity_sc5.log
AB_MODES="2,1" bash scripts/ab.sh $V/sc0.so $V/sc5.so $V/sc6.so $V/sc7.so $V/sc8.so; cp gpurun_out/ab.log gpurun_out/r02o_ab.log
