#!/bin/bash
mkdir -p gpurun_out
python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --batch 32 > gpurun_out/plain_i8.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_i8.csv \
    python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --batch 32 > gpurun_out/ncu_i8.log 2>&1
tail -2 gpurun_out/ncu_i8.log
ncu --set full --clock-control none --import-source on -k regex:k_i8_stage -s 8 -c 1 -o gpurun_out/prof_i8 -f \
    python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --batch 32 > gpurun_out/ncu_i8b.log 2>&1
tail -1 gpurun_out/ncu_i8b.log
