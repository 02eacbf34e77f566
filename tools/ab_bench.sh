#!/bin/bash
# Same-box A/B of the bench step: A = the product library, B = $B_LIB (default: an
# experimental build in paper_2605_18052_b200/libdmv3d_exp.so), alternated 3 times.
B_LIB=${B_LIB:-$PWD/paper_2605_18052_b200/libdmv3d_exp.so}
for r in 1 2 3; do
  python bench.py --no-cpu-baseline --steps 50 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('A', d['ms_per_step'], d['roofline']['kernel_ms'])"
  DMV3D_LIB=$B_LIB python bench.py --no-cpu-baseline --steps 50 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('B', d['ms_per_step'], d['roofline']['kernel_ms'])"
done
