#!/bin/bash
# Low-rank path: bench line (ours + reference arm) and ncu evidence.
mkdir -p gpurun_out
python bench.py --config LR > gpurun_out/bench_LR.json 2> gpurun_out/bench_LR.err
python bench.py --config LR --impl reference --steps 3 --warmup 1 > gpurun_out/bench_LR_reference.json 2> gpurun_out/bench_LR_reference.err
python bench.py --config LR --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain_lr.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lowrank -s 3 -c 1 \
    -o gpurun_out/prof_LR -f python bench.py --config LR --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_lr.log 2>&1
echo done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_LR.csv \
    python bench.py --config LR --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_lr1.log 2>&1
python -m pytest tests/test_gpu_lowrank.py -q -p no:cacheprovider > gpurun_out/pytest_lr.log 2>&1
