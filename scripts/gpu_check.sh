#!/bin/bash
# one GPU round: parity tests, headline bench, other modes (used with gpurun)
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/rc.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_head.log 2>&1
rm -f gpurun_out/bench_modes.log
for c in "0 0" "2 0" "2 1"; do set -- $c; timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --construction $1 --conditioning $2 >> gpurun_out/bench_modes.log 2>&1; done
