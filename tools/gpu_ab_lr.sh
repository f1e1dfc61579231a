#!/bin/bash
# A/B of two builds of the library on the same box: LR bench, alternating.
mkdir -p gpurun_out
for i in 1 2; do
for v in libexpmb.so libexpmb_a.so; do
EXPMB_LIB=$v python bench.py --config LR --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3))"
done; done > gpurun_out/ab_lr.txt 2>&1
cat gpurun_out/ab_lr.txt
