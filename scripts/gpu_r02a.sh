#!/bin/bash
# round 2, session A: full GPU parity (tightened tolerances, 2-rank DistributedPricer), the
# measured deviations, default bench (strong, N=1), weak and C5 lines, the --gpus 2 refusal
mkdir -p gpurun_out; rm -f gpurun_out/r02a_*
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/r02a_pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/r02a_rc.txt
timeout 900 python tests/tools/parity_report.py > gpurun_out/r02a_parity_report.log 2>&1; echo report=$? >> gpurun_out/r02a_rc.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02a_bench.jsonl 2> gpurun_out/r02a_bench.err; echo bench=$? >> gpurun_out/r02a_rc.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --points 8388608 >> gpurun_out/r02a_bench.jsonl 2>> gpurun_out/r02a_bench.err
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --workload C5 >> gpurun_out/r02a_bench.jsonl 2>> gpurun_out/r02a_bench.err
timeout 300 python bench.py --gpus 2 --steps 2 --warmup 1 > gpurun_out/r02a_gpus2.log 2>&1; echo gpus2=$? >> gpurun_out/r02a_rc.txt
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 >> gpurun_out/r02a_bench.jsonl 2>> gpurun_out/r02a_bench.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a_smoke.log 2>&1; echo smoke=$? >> gpurun_out/r02a_rc.txt
