#!/bin/bash
# zt: z = 2u - 1 in one fma from the lattice word and t = fma(-z, z, 1) (bit-identical normals,
# three FP64 operations fewer per normal).  Bit-identity of the bench results + parity + A/B.
V=$PWD/paper_2209_11337_b200/build/var
L=gpurun_out/r02ao.log; rm -f $L
for lib in cur zt zt3; do
  for a in "--construction 1 --conditioning 0" "--construction 2 --conditioning 1" "--method 2 --construction 1" "--workload C5"; do
    QMCCPW_LIB=$V/$lib.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$lib', '$a', json.dumps(json.loads(l)['results_sample'])) for l in sys.stdin if l.startswith('{')]" >> gpurun_out/r02ao_bits.log
  done
done
QMCCPW_LIB=$V/zt.so timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -m gpu -k "normal or sobol or bench_launch or path_values or owen" >> $L 2>&1; echo rc=$? >> $L
for rep in 1 2; do for lib in cur zt zt3; do export QMCCPW_LIB=$V/$lib.so; echo "== $lib rep $rep" >> $L
  for a in "--construction 1 --conditioning 0" "--construction 0 --conditioning 0" "--construction 2 --conditioning 0" "--construction 2 --conditioning 1" "--workload C5"; do
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>/dev/null | python -c "import sys,json; [print('$a', json.loads(l)['ms_per_step']) for l in sys.stdin if l.startswith('{')]" >> $L
  done; done; done
