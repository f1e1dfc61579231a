#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do for mb in 2 3 4; do
EXPMB_C2_MINB=$mb python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('minb $mb', d['ms_per_step'])"
done; done > gpurun_out/ab2.txt 2>&1
