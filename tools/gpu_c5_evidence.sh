#!/bin/bash
# C5 (int8-slice path) evidence: bench line, launch list, ncu of one int8 stage.
mkdir -p gpurun_out
python bench.py --config C5 --steps 2 --warmup 3 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
./tools/gpu_i8_prof.sh
