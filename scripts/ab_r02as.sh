#!/bin/bash
# sa: X1 passes read (sigma a_j, a_j^2) from a per-launch table instead of two DMULs per date and
# pass (bit-identical).  Bit check + parity + A/B.
V=$PWD/paper_2209_11337_b200/build/var
L=gpurun_out/r02as.log; rm -f $L gpurun_out/r02as_bits.log
for lib in cur sa; do
  for a in "--construction 2 --conditioning 1" "--construction 1 --conditioning 1" "--construction 2 --conditioning 1 --options 0,1,2"; do
    QMCCPW_LIB=$V/$lib.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$lib', '$a', json.dumps(json.loads(l)['results_sample'])) for l in sys.stdin if l.startswith('{')]" >> gpurun_out/r02as_bits.log
  done
done
QMCCPW_LIB=$V/sa.so timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -m gpu -k "x1 or lookback or bench_launch or d256 or owen" >> $L 2>&1; echo rc=$? >> $L
for rep in 1 2; do for lib in cur sa; do export QMCCPW_LIB=$V/$lib.so; echo "== $lib rep $rep" >> $L
  for a in "--construction 2 --conditioning 1" "--construction 1 --conditioning 1" "--construction 2 --conditioning 1 --options 0,1,2"; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$a', json.loads(l)['ms_per_step']) for l in sys.stdin if l.startswith('{')]" >> $L
  done; done; done
