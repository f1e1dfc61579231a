#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "ragged or C3 or C4 or C5 or golden" > gpurun_out/pytest_large.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_large.log
for c in C3 C4 C2 C1; do
timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
echo done
