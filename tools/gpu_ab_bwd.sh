# backward: TC backward parity tests on the product library, then a same-box A/B over LIBS
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_backward_tc.py -x -q > $O/pytest_bwd.log 2>&1; tail -2 $O/pytest_bwd.log
ROUNDS=${ROUNDS:-2} bash tools/ab_bwd.sh 2>&1 | tee $O/ab_bwd.log
