#!/bin/bash
# full check of the current default build: GPU tests (bounded), the checked build over every
# kernel, the default bench line, every mode's line, and the lookback A/B at 6 blocks/SM
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/r02s_pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/r02s_rc.txt
QMCCPW_LIB=$PWD/paper_2209_11337_b200/libqmccpw_checked.so timeout 900 python tests/tools/diag_checked.py > gpurun_out/r02s_checked.log 2>&1; echo checked=$? >> gpurun_out/r02s_rc.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02s_bench.jsonl 2>&1; echo bench=$? >> gpurun_out/r02s_rc.txt
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 >> gpurun_out/r02s_bench.jsonl 2>&1
timeout 1800 bash scripts/bench_all_modes.sh; cp gpurun_out/bench_all_modes.jsonl gpurun_out/r02s_bench_all_modes.jsonl
for lib in $PWD/paper_2209_11337_b200/build/var/lq6.so ""; do echo "== $lib" >> gpurun_out/r02s_ab_lb.log
  QMCCPW_LIB=${lib:-$PWD/paper_2209_11337_b200/libqmccpw.so} timeout 120 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --construction 2 --conditioning 1 --options 0,1,2 >> gpurun_out/r02s_ab_lb.log 2>&1; done
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02s_smoke.log 2>&1; echo smoke=$? >> gpurun_out/r02s_rc.txt
