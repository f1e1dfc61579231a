#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
for v in 0 1; do
EXPMB_VARIANT=$v python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C1 variant $v', d['ms_per_step'])"
done > gpurun_out/ab5.txt 2>&1
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
