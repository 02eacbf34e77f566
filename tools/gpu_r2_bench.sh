O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_bench_dist.py tests/test_gpu_dist.py -x -q > $O/pytest_dist.log 2>&1; tail -15 $O/pytest_dist.log
timeout 600 python bench.py > $O/bench_r2.json 2> $O/bench_r2.err; tail -c 3000 $O/bench_r2.json; tail -5 $O/bench_r2.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:render_tc -s 3 -c 1 -o $O/prof_tc python bench.py --steps 1 --warmup 3 --no-cpu-baseline --sustained-s 0 > $O/ncu_tc.log 2>&1; tail -1 $O/ncu_tc.log
