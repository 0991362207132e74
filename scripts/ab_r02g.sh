#!/bin/bash
V=$PWD/paper_2209_11337_b200/build/var
QMCCPW_LIB=$V/bbG8.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "path_values or c4_fused or bench_launch or edge or owen" -x > gpurun_out/r02g_parity_bbG8.log 2>&1; echo rc=$? >> gpurun_out/r02g_parity_bbG8.log
AB_MODES="1,0" bash scripts/ab.sh $V/bbOld.so $V/bbG8.so $V/bbG7.so $V/bbG6.so; cp gpurun_out/ab.log gpurun_out/r02g_ab_bb.log
AB_MODES="2,0" bash scripts/ab.sh $V/pcaC.so $V/pcaE.so $V/pcaF.so; cp gpurun_out/ab.log gpurun_out/r02g_ab_pca.log
