#!/bin/bash
# Round-2 re-entry evidence: GPU tests + smoke + default bench on HEAD, then sanitizer logs.
mkdir -p gpurun_out/sanitizer
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for tool in racecheck synccheck memcheck; do
  for c in c2 c1 i8 tile gemm lowrank select; do
    timeout 300 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py $c \
      > gpurun_out/sanitizer/${tool}_$c.log 2>&1
    echo "rc=$?" >> gpurun_out/sanitizer/${tool}_$c.log
  done
done
echo done
