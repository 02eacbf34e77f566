#!/bin/bash
# SURVEY §8(d) variants: throughput lines + per-variant ncu DRAM bytes of K0 / K1.
O=gpurun_out
timeout 900 python tools/variants.py > $O/variants.jsonl 2> $O/variants.err; cat $O/variants.jsonl | cut -c1-400; tail -3 $O/variants.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
for v in cfg3_eta1_keep cfg3_c32 cfg3_l2 cfg2x8 cfg4 cachebust; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:"render_tc|preproject" -s 6 -c 2 --csv python tools/variants.py --only $v --steps 1 > $O/ncu_var_$v.csv 2>/dev/null
done
echo done
