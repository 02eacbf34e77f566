O=gpurun_out
{ echo "# compute-sanitizer on tools/sanitize.py (B200, round 2): every CUDA entry point on small inputs"
  echo "# (round 1's set + SiLU/softplus tensor-core renders, range flags, batched step, Plucker 1/2/4 rays per thread)"
  for t in memcheck racecheck synccheck initcheck; do echo "== $t"; timeout 900 compute-sanitizer --tool $t python tools/sanitize.py 2>&1 | grep -E "SUMMARY|sanitize workload done" ; done; } > $O/sanitizer_r02.txt
cat $O/sanitizer_r02.txt
