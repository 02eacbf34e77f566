# microbenchmark: MMA chain issue style + Plucker rows with both flush modes
O=gpurun_out; mkdir -p $O
./tools/mma_uniform > $O/mma_uniform.txt 2>&1; cat $O/mma_uniform.txt
timeout 300 python tools/bench_rows.py --rows f2 > $O/rows_f2.jsonl 2> $O/rows_f2.err; cut -c1-200 $O/rows_f2.jsonl
