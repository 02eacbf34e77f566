# same-box A/B over library builds (LIBS) + TC parity tests on the product library
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q > $O/pytest_tc.log 2>&1; tail -2 $O/pytest_tc.log
ROUNDS=${ROUNDS:-3} bash tools/ab_multi.sh 2>&1 | tee $O/ab.log
