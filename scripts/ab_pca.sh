#!/bin/bash
# safety rerun of the checked build + PCA-W1 variant A/B + the FP64 DMMA/DFMA sharing microbench
QMCCPW_LIB=$PWD/paper_2209_11337_b200/libqmccpw_checked.so timeout 900 python tests/tools/diag_checked.py > gpurun_out/r02f_checked.log 2>&1
timeout 600 python -m pytest tests/test_memory_safety.py -q -rf > gpurun_out/r02f_safety.log 2>&1; echo rc=$? >> gpurun_out/r02f_safety.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mix paper_2209_11337_b200/tools/fp64_mix_bench.cu && /tmp/mix > gpurun_out/r02f_mix.log 2>&1
AB_MODES="2,0" bash scripts/ab.sh $PWD/paper_2209_11337_b200/libqmccpw.so $PWD/paper_2209_11337_b200/build/var/pcaB.so $PWD/paper_2209_11337_b200/build/var/pcaC.so $PWD/paper_2209_11337_b200/build/var/pcaD.so
cp gpurun_out/ab.log gpurun_out/r02f_ab.log
