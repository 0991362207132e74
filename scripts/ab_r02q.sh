#!/bin/bash
V=$PWD/paper_2209_11337_b200/build/var
QMCCPW_LIB=$V/p4.so timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "path_values or c4_fused or configs or gpca or pca" > gpurun_out/r02q_parity_p4.log 2>&1; echo rc=$? >> gpurun_out/r02q_parity_p4.log
AB_MODES="2,0 2,1" bash scripts/ab.sh $V/p2.so $V/p4.so $V/p4m6.so; cp gpurun_out/ab.log gpurun_out/r02q_ab.log
bash scripts/gpu_ncu_r02.sh r02q "pcax1lb:--construction=2,--conditioning=1,--options=0+1+2"
