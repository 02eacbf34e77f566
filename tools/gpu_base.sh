O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 300 python bench.py --no-cpu-baseline --steps 50 > $O/bench_base.json 2> $O/bench_base.err; tail -c 400 $O/bench_base.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:render_tc -s 3 -c 1 -o $O/prof_base python bench.py --steps 2 --warmup 3 --no-cpu-baseline --sustained-s 0 > $O/ncu_base.log 2>&1; tail -2 $O/ncu_base.log
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
