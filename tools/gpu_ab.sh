#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('static', d['ms_per_step'], d['clocks'])"
EXPMB_CLAIM=1 python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('claim', d['ms_per_step'], d['clocks'])"
done > gpurun_out/ab.txt 2>&1
