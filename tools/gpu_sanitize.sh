# compute-sanitizer evidence: racecheck (shared-memory hazards), synccheck
# (barrier misuse), memcheck (out-of-bounds) on one small run of each kernel family
mkdir -p gpurun_out/sanitizer
for tool in racecheck synccheck memcheck; do
  for c in c2 c1 i8 tile gemm lowrank select; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py $c \
      > gpurun_out/sanitizer/${tool}_$c.log 2>&1
    echo "rc=$?" >> gpurun_out/sanitizer/${tool}_$c.log
  done
done
echo done
