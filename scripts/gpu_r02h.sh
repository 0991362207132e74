#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/r02h_pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/r02h_rc.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02h_bench.jsonl 2>&1; echo bench=$? >> gpurun_out/r02h_rc.txt
bash scripts/gpu_ncu_r02.sh r02h "bbw1: pcaw1:--construction=2"
