#!/bin/bash
# Same-box A/B of the bench step over environment settings (ENVS="A=1 B=2;A=3" ...,
# ';'-separated), alternated ROUNDS times; prints ms/step, render-kernel ms, occupancy.
IFS=';' read -ra CFGS <<< "$ENVS"
for r in $(seq ${ROUNDS:-3}); do
  for C in "${CFGS[@]}"; do
    env $C timeout 120 python bench.py --no-cpu-baseline --steps 50 ${BENCH_ARGS} 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$C', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), d.get('mma_row_occupancy'))"
  done
done
