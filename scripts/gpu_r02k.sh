#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/r02k_pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/r02k_rc.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02k_bench.jsonl 2>&1; echo bench=$? >> gpurun_out/r02k_rc.txt
bash scripts/bench_all_modes.sh; cp gpurun_out/bench_all_modes.jsonl gpurun_out/r02k_bench_all_modes.jsonl
bash scripts/gpu_ncu_r02.sh r02k "bbw1: pcaw1:--construction=2"
