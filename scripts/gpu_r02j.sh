#!/bin/bash
# final evidence pass on the current default build (the W1 units are unchanged since r02i: ncu of the X1 modes and C5) (ncu reports summarised on the box; only the
# BB-W1 and PCA-W1 .ncu-rep files are kept, to stay under gpurun's 64 MiB return limit)
mkdir -p gpurun_out
rm -f gpurun_out/parity_per_path_deviations.txt; QMCCPW_PARITY_LOG=$PWD/gpurun_out/parity_per_path_deviations.txt timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/r02j_pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/r02j_rc.txt
QMCCPW_LIB=$PWD/paper_2209_11337_b200/libqmccpw_checked.so timeout 900 python tests/tools/diag_checked.py > gpurun_out/r02j_checked.log 2>&1; echo checked=$? >> gpurun_out/r02j_rc.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02j_bench.jsonl 2>&1; echo bench=$? >> gpurun_out/r02j_rc.txt
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 >> gpurun_out/r02j_bench.jsonl 2>&1
timeout 1800 bash scripts/bench_all_modes.sh; cp gpurun_out/bench_all_modes.jsonl gpurun_out/r02j_bench_all_modes.jsonl
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02j_smoke.log 2>&1; echo smoke=$? >> gpurun_out/r02j_rc.txt
timeout 900 python tests/tools/parity_report.py > gpurun_out/r02j_parity_report.log 2>&1; echo parity_report=$? >> gpurun_out/r02j_rc.txt
for m in "pcax1|PCA-X1|67108864|--construction 2 --conditioning 1" "bbx1|BB-X1|67108864|--construction 1 --conditioning 1" "stdx1|STD-X1|67108864|--construction 0 --conditioning 1" "lb|PCA-X1/o0,1,2/m0/r0|67108864|--construction 2 --conditioning 1 --options 0,1,2" "c5|C5|4194304|--workload C5"; do
  IFS='|' read name key paths args <<< "$m"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"paths_kernel|pca_kernel|portfolio_kernel" -c 1 \
    -o gpurun_out/r02j_$name -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline $args > gpurun_out/r02j_${name}_ncu.log 2>&1
  echo "${name}_ncu=$?" >> gpurun_out/r02j_rc.txt
  python scripts/ncu_to_json.py gpurun_out/r02j_$name.ncu-rep "$key" $paths --build "r02j (v30): end of round 2" --out gpurun_out/r02j_${name}_ncu.txt > /dev/null 2>&1
  echo "${name}_summary=$?" >> gpurun_out/r02j_rc.txt
  case $name in pcax1|c5) ;; *) rm -f gpurun_out/r02j_$name.ncu-rep ;; esac
done
cp profiles/ncu_metrics.json gpurun_out/r02j_ncu_metrics.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02j_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02j_launches.log 2>&1
echo "launches=$?" >> gpurun_out/r02j_rc.txt
rm -f gpurun_out/bench_all_modes.jsonl
du -sh gpurun_out >> gpurun_out/r02j_rc.txt
