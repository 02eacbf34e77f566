#!/bin/bash
# One GPU call that refreshes every judged number: GPU parity suite, the default bench
# line (with the CPU oracle leg and the sustained run), the launch list of the bench
# command, one full ncu capture of the render kernel, the SURVEY §8(f) rows, the §8(d)
# variants, the cfg2 bench and the ray-count sweep.  Outputs land in gpurun_out/.
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_final.json 2> $O/bench_final.err; tail -c 300 $O/bench_final.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --sustained-s 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_tc -s 3 -c 1 -o $O/prof_tc python bench.py --steps 2 --warmup 3 --no-cpu-baseline --sustained-s 0 > $O/ncu_tc.log 2>&1
timeout 900 python tools/bench_rows.py > $O/rows.jsonl 2> $O/rows.err
timeout 600 python bench.py --config cfg2 --no-cpu-baseline --sustained-s 0 > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 900 python tools/sweep.py > $O/sweep.jsonl 2> $O/sweep.err
bash tools/gpu_variants.sh > /dev/null 2>&1
echo done-main
# phase split of the render kernel (DMV3D_PHASES build, prebuilt in-tree)
[ -f paper_2605_18052_b200/libdmv3d_phases.so ] && DMV3D_LIB=$PWD/paper_2605_18052_b200/libdmv3d_phases.so timeout 300 python tools/phases.py > $O/phases.txt 2>&1
