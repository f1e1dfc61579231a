#!/bin/bash
mkdir -p gpurun_out
EXPMB_C2_MINB=3 timeout 300 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "C2 or golden_fp32 or ragged" > gpurun_out/pytest_v3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_v3.log
for rep in 1 2; do for mb in 2 3 4; do
EXPMB_C2_MINB=$mb python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('minb $mb', d['ms_per_step'])"
done; done > gpurun_out/ab6.txt 2>&1
