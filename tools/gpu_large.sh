#!/bin/bash
mkdir -p gpurun_out
for c in C3 C4; do
timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C3.csv \
    python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_stage -s 20 -c 1 \
    -o gpurun_out/prof_C3 -f python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_p3.log 2>&1
python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_stage -s 20 -c 1 \
    -o gpurun_out/prof_C4 -f python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_p4.log 2>&1
echo done
