#!/bin/bash
# i8 tests on the new default, then ncu --set full of the C5 stage kernel and the C2 kernel, C3 launch list
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_i8.py tests/test_gpu_configs.py tests/test_gpu_shards.py -m gpu -q -rf -p no:cacheprovider > gpurun_out/pytest_i8.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_i8.log
python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --no-per-config --batch 8 > gpurun_out/plain5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_i8_stage -s 30 -c 1 \
    -o gpurun_out/prof_C5 -f python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --no-per-config --batch 8 > gpurun_out/ncu5.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:w16 -s 3 -c 1 \
    -o gpurun_out/prof_C2 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/ncu2.log 2>&1
python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/plain3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C3.csv \
    python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/ncu_l3.log 2>&1
echo done
