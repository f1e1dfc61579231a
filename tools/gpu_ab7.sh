#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
for rep in 1 2; do for v in 0 1; do
EXPMB_NO_DMMA=$v python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('no_dmma=$v', d['ms_per_step'], d['useful_tflops'])"
done; done > gpurun_out/ab7.txt 2>&1
