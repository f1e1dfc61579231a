#!/bin/bash
mkdir -p gpurun_out
python bench.py --config C3 --timegrid --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain_tg.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C3tg.csv \
    python bench.py --config C3 --timegrid --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_tg.log 2>&1
python -m pytest tests/test_gpu_timegrid.py -q -p no:cacheprovider > gpurun_out/pytest_tg.log 2>&1
tail -1 gpurun_out/pytest_tg.log
