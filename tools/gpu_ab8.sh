#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
for v in 0 1; do
EXPMB_NO_DMMA=$v timeout 300 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C4 no_dmma=$v', d['ms_per_step'], d['useful_tflops'], d['value'])"
done > gpurun_out/ab8.txt 2>&1
