#!/bin/bash
# One GPU call that refreshes every judged number: GPU parity suite, the default bench
# line (with the CPU oracle leg), the SIMT-engine bench, the launch list of the bench
# command, one full ncu capture of each render kernel, and the SURVEY §8(f) rows.
# Outputs land in gpurun_out/ (copied to profiles/ by hand).
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_final.json 2> $O/bench_final.err; tail -c 400 $O/bench_final.json
timeout 600 python bench.py --engine simt --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_simt.json 2> $O/bench_simt.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_tc -s 3 -c 1 -o $O/prof_tc python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_tc.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_simt -s 3 -c 1 -o $O/prof_simt python bench.py --engine simt --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_simt.log 2>&1
timeout 600 python tools/bench_rows.py > $O/rows.jsonl 2> $O/rows.err
timeout 600 python bench.py --config cfg2 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 900 python tools/sweep.py > $O/sweep.jsonl 2> $O/sweep.err
echo done-main
timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_bwd_tc -s 1 -c 1 -o $O/prof_bwtc python tools/bw_prof.py tcgen05 > $O/ncu_bwtc.log 2>&1
echo done-bwtc
