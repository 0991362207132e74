#!/bin/bash
# ncu captures of the dominant kernel of each bench mode (one GPU; each after its own command
# ran clean without ncu), plus the launch list of the default bench.  Usage: bash scripts/gpu_ncu_r02.sh TAG [MODES]
# MODES: space-separated NAME:args, args comma-separated with = for spaces; a + inside a value
# stands for a comma (e.g. "lb:--options=0+1+2").  Default: the four headline modes.
TAG=${1:-r02}
MODES=${2:-"bbw1: pcaw1:--construction=2 pcax1:--construction=2,--conditioning=1 c5:--workload=C5"}
mkdir -p gpurun_out
for m in $MODES; do
  name=${m%%:*}; a=${m#*:}; a=${a//,/ }; a=${a//=/ }; a=${a//+/,}
  timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline $a > gpurun_out/${TAG}_${name}_bench.jsonl 2>&1
  echo "${name}_bench=$?" >> gpurun_out/${TAG}_ncu_rc.txt
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"paths_kernel|pca_kernel|portfolio_kernel" -c 1 \
    -o gpurun_out/${TAG}_${name} -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline $a > gpurun_out/${TAG}_${name}_ncu.log 2>&1
  echo "${name}_ncu=$?" >> gpurun_out/${TAG}_ncu_rc.txt
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_launches.log 2>&1
echo "launches=$?" >> gpurun_out/${TAG}_ncu_rc.txt
