#!/bin/bash
# end-of-round evidence on the current default build
rm -f gpurun_out/parity_per_path_deviations.txt; QMCCPW_PARITY_LOG=$PWD/gpurun_out/parity_per_path_deviations.txt timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/r02f_pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/r02f_rc.txt
QMCCPW_LIB=$PWD/paper_2209_11337_b200/libqmccpw_checked.so timeout 900 python tests/tools/diag_checked.py > gpurun_out/r02f_checked.log 2>&1; echo checked=$? >> gpurun_out/r02f_rc.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02f_bench.jsonl 2>&1; echo bench=$? >> gpurun_out/r02f_rc.txt
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 >> gpurun_out/r02f_bench.jsonl 2>&1
timeout 1800 bash scripts/bench_all_modes.sh; cp gpurun_out/bench_all_modes.jsonl gpurun_out/r02f_bench_all_modes.jsonl
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; echo smoke=$? >> gpurun_out/r02f_rc.txt
timeout 900 python tests/tools/parity_report.py > gpurun_out/r02f_parity_report.log 2>&1; echo parity_report=$? >> gpurun_out/r02f_rc.txt
bash scripts/gpu_ncu_r02.sh r02f "bbw1: pcaw1:--construction=2 stdw1:--construction=0 pcax1:--construction=2,--conditioning=1 bbx1:--construction=1,--conditioning=1 stdx1:--construction=0,--conditioning=1 lb:--construction=2,--conditioning=1,--options=0+1+2 c5:--workload=C5"
