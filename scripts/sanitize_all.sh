#!/bin/bash
# One compute-sanitizer pass per tool over scripts/sanitize_run.py.
# Logs go to gpurun_out/sanitize_<tool>.log; the summary line of each is the verdict.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout 1200 $CS --tool $tool $extra --print-limit 100 --error-exitcode 9 \
      python scripts/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_rc.txt
  tail -3 gpurun_out/sanitize_$tool.log
done
