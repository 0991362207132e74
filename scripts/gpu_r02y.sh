#!/bin/bash
# end-of-round evidence on the current default build
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/r02y_pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/r02y_rc.txt
QMCCPW_LIB=$PWD/paper_2209_11337_b200/libqmccpw_checked.so timeout 900 python tests/tools/diag_checked.py > gpurun_out/r02y_checked.log 2>&1; echo checked=$? >> gpurun_out/r02y_rc.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02y_bench.jsonl 2>&1; echo bench=$? >> gpurun_out/r02y_rc.txt
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 >> gpurun_out/r02y_bench.jsonl 2>&1
timeout 1800 bash scripts/bench_all_modes.sh; cp gpurun_out/bench_all_modes.jsonl gpurun_out/r02y_bench_all_modes.jsonl
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02y_smoke.log 2>&1; echo smoke=$? >> gpurun_out/r02y_rc.txt
bash scripts/gpu_ncu_r02.sh r02y "bbw1: stdx1:--construction=0,--conditioning=1 bbx1:--construction=1,--conditioning=1 pcax1:--construction=2,--conditioning=1"
