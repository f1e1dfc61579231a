#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/i8_crossover.py > gpurun_out/i8_crossover.txt 2>&1
timeout 300 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu-baseline --no-per-config > gpurun_out/c3_ffma.json 2>gpurun_out/c3_ffma.err
EXPMB_I8=1 timeout 300 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu-baseline --no-per-config > gpurun_out/c3_i8.json 2>gpurun_out/c3_i8.err
echo done
