#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "C3 or ragged" > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err
EXPMB_NO_TC=1 timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C3_simt.json 2> gpurun_out/bench_C3_simt.err
echo done
