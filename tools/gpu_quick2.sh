#!/bin/bash
mkdir -p gpurun_out
./tools/peaks > gpurun_out/peaks.json 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
for c in C1 C3; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 600 python bench.py --config C5 --steps 2 --warmup 3 --batch 32 --no-cpu-baseline > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
echo done
