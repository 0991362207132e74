#!/bin/bash
# ti: the lookback argmax tracking's two compares on the bits of e - e_max (integer pipe) instead
# of two DSETPs (same decisions).  Bit check + parity + A/B.
V=$PWD/paper_2209_11337_b200/build/var
L=gpurun_out/r02av.log; rm -f $L gpurun_out/r02av_bits.log
for lib in cur ti; do
  for a in "--construction 1 --conditioning 0" "--construction 0 --conditioning 0" "--method 3 --construction 1"; do
    QMCCPW_LIB=$V/$lib.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$lib', '$a', json.dumps(json.loads(l)['results_sample'])) for l in sys.stdin if l.startswith('{')]" >> gpurun_out/r02av_bits.log
  done
done
QMCCPW_LIB=$V/ti.so timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -m gpu -k "bb or std or lookback or bench_launch or c3 or c1 or mc" >> $L 2>&1; echo rc=$? >> $L
for rep in 1 2; do for lib in cur ti; do export QMCCPW_LIB=$V/$lib.so; echo "== $lib rep $rep" >> $L
  for a in "--construction 1 --conditioning 0" "--construction 0 --conditioning 0" "--method 3 --construction 1"; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$a', json.loads(l)['ms_per_step']) for l in sys.stdin if l.startswith('{')]" >> $L
  done; done; done
