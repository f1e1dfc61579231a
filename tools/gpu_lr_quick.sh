#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_lowrank.py -q -x -p no:cacheprovider > gpurun_out/lr.log 2>&1; tail -2 gpurun_out/lr.log
python bench.py --config LR --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('LR', d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'])"
