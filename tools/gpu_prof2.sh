#!/bin/bash
mkdir -p gpurun_out
python bench.py --config C1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:expm_fused -s 3 -c 1 \
    -o gpurun_out/prof_C1 -f python bench.py --config C1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu3.log 2>&1
python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_stage -s 20 -c 1 \
    -o gpurun_out/prof_C4 -f python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_p4.log 2>&1
echo done
