B_LIB=$PWD/paper_2605_18052_b200/libdmv3d_exp.so
for r in 1 2; do
  python bench.py --config cfg2 --no-cpu-baseline --steps 50 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('A', d['ms_per_step'], d['roofline']['kernel_ms'])"
  DMV3D_LIB=$B_LIB python bench.py --config cfg2 --no-cpu-baseline --steps 50 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('B', d['ms_per_step'], d['roofline']['kernel_ms'])"
done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:preproject -c 4 --csv python bench.py --config cfg2 --no-cpu-baseline --steps 2 --warmup 3 2>/dev/null | grep preproject | head -2 | cut -c1-200
DMV3D_LIB=$B_LIB ncu --metrics gpu__time_duration.sum --clock-control none -k regex:preproject -c 4 --csv python bench.py --config cfg2 --no-cpu-baseline --steps 2 --warmup 3 2>/dev/null | grep preproject | head -2 | cut -c1-200
