#!/bin/bash
# One GPU iteration: tensor-core parity tests, then a same-box A/B of the bench step
# (A = product library, B = $B_LIB), then a bench line with the occupancy counters.
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_tc.py tests/test_gpu_parity.py tests/test_gpu_next.py tests/test_gpu_variants.py} -x -q > $O/pytest_iter.log 2>&1; tail -3 $O/pytest_iter.log
if [ -n "$B_LIB" ]; then B_LIB=$B_LIB bash tools/ab_bench.sh 2>&1 | tee $O/ab.log; fi
timeout 300 python bench.py --no-cpu-baseline --steps 50 > $O/bench_iter.json 2> $O/bench_iter.err; cat $O/bench_iter.json; tail -3 $O/bench_iter.err
