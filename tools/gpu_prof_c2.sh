#!/bin/bash
# C2 kernel profile: plain run, then one full ncu capture with source counters.
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:expm_fused -s 3 -c 1 \
    -o gpurun_out/prof_C2 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/ncu_c2.log 2>&1
echo done
