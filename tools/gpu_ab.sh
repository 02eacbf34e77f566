#!/bin/bash
# One GPU iteration: parity subset on the product library, same-box A/B of the bench step
# over $LIBS, and a targeted ncu metric pass of render_tc on the product library.
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_tc.py tests/test_gpu_parity.py} -x -q > $O/pytest_ab.log 2>&1; tail -3 $O/pytest_ab.log
LIBS="${LIBS:-$PWD/paper_2605_18052_b200/libdmv3d_r1.so $PWD/paper_2605_18052_b200/libdmv3d.so}" ROUNDS=${ROUNDS:-3} bash tools/ab_multi.sh 2>&1 | tee $O/ab.log
if [ -n "$NCU_METRICS" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed --clock-control none -k regex:render_tc -s 3 -c 1 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_metrics.csv 2>&1
  grep -E "gpu__time|pipe_tensor|issue_active|bank_conf|inst_exec|wavefronts" $O/ncu_metrics.csv | awk -F'","' '{print $(NF-2), $NF}'
fi
