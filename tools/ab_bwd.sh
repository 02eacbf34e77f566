#!/bin/bash
# Same-box A/B of the tensor-core backward (row f1, 8 x 128^2, N = 128) over $LIBS.
for r in $(seq ${ROUNDS:-2}); do
  for L in $LIBS; do
    DMV3D_LIB=$L timeout 300 python tools/bench_rows.py --rows f1tc 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$(basename $L)', d['row'][:60], round(d['kernel_ms'],4), round(d['roofline']['frac'],4))"
  done
done
