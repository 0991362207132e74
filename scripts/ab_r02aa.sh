#!/bin/bash
V=$PWD/paper_2209_11337_b200/build/var
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "d256 or deep" > gpurun_out/r02aa_parity_new_tests.log 2>&1; echo rc=$? >> gpurun_out/r02aa_parity_new_tests.log
AB_MODES="2,1 1,1" bash scripts/ab.sh $V/u1.so $V/u2.so $V/u4.so; cp gpurun_out/ab.log gpurun_out/r02aa_ab.log
