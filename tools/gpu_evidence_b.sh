#!/bin/bash
# Evidence part B (separate call: each ncu --set full report is 25-35 MB and
# gpurun returns at most 64 MB): the C1 (DMMA) capture and one squaring-stage
# launch of the C5 int8 stage (launch 5 of a 64-matrix run).
mkdir -p gpurun_out
python bench.py --config C1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dmma -s 3 -c 1 \
    -o gpurun_out/prof_C1 -f python bench.py --config C1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu3.log 2>&1
python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --batch 64 > gpurun_out/plain5.log 2>&1 && \
ncu --set full --clock-control none -k regex:k_i8_stage -s 5 -c 1 \
    -o gpurun_out/prof_C5 -f python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --batch 64 > gpurun_out/ncu5.log 2>&1
echo done
