#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --scheme baseline > gpurun_out/bench_C2_alg1.json 2> gpurun_out/bench_C2_alg1.err
python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_C1.json 2> gpurun_out/bench_C1.err
python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline --scheme baseline > gpurun_out/bench_C1_alg1.json 2> gpurun_out/bench_C1_alg1.err
echo done
