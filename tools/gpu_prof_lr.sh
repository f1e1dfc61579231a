#!/bin/bash
mkdir -p gpurun_out
python bench.py --config LR --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain_lr.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lowrank -s 3 -c 1 -o gpurun_out/prof_LR -f \
    python bench.py --config LR --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_lr.log 2>&1
tail -1 gpurun_out/ncu_lr.log
