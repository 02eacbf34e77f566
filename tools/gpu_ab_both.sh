# forward (cfg3 bench step) and backward (f1 TC rows) same-box A/B over LIBS; TC parity
# tests (forward + backward) on TEST_LIB (default: the product library)
O=gpurun_out; mkdir -p $O
DMV3D_LIB=${TEST_LIB:-} timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_backward_tc.py -x -q > $O/pytest_ab.log 2>&1; tail -2 $O/pytest_ab.log
ROUNDS=${ROUNDS:-3} bash tools/ab_multi.sh 2>&1 | tee $O/ab.log
ROUNDS=${BROUNDS:-2} bash tools/ab_bwd.sh 2>&1 | tee $O/ab_bwd.log
