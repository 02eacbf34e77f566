#!/bin/bash
# quick GPU iteration: TC parity tests, bench, launch list (+ optional full ncu of the render kernel)
set -x
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -5
python bench.py --steps 50 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
if [ -n "$NCU_FULL" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:render_tc -s 2 -c 1 -o gpurun_out/prof_tc python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
  tail -2 gpurun_out/ncu_full.log
fi
