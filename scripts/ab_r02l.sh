#!/bin/bash
V=$PWD/paper_2209_11337_b200/build/var
QMCCPW_LIB=$V/x1phi.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "path_values or c4_fused or c3_full or deep or configs or gpca" -x > gpurun_out/r02l_parity_x1phi.log 2>&1; echo rc=$? >> gpurun_out/r02l_parity_x1phi.log
AB_MODES="2,1 1,1 3,1" bash scripts/ab.sh $V/x1old.so $V/x1phi.so; cp gpurun_out/ab.log gpurun_out/r02l_ab_x1.log
