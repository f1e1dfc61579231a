#!/bin/bash
mkdir -p gpurun_out
EXPMB_VARIANT=2 timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -k "C2 or golden_fp32 or ragged or host or named or determinism" > gpurun_out/pytest_v2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_v2.log
for rep in 1 2; do for v in 1 2; do
EXPMB_VARIANT=$v python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('variant $v', d['ms_per_step'])"
done; done > gpurun_out/ab10.txt 2>&1
