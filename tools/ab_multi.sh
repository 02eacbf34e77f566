#!/bin/bash
# Same-box A/B/C... of the bench step over several library builds (LIBS="a.so b.so ..."),
# alternated ROUNDS times; prints ms/step and the render kernel's CUDA-event ms.
for r in $(seq ${ROUNDS:-3}); do
  for L in $LIBS; do
    DMV3D_LIB=$L timeout 90 python bench.py --no-cpu-baseline --steps 50 ${BENCH_ARGS} 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$(basename $L)', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), d.get('mma_row_occupancy'))"
  done
done
