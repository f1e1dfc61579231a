#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_i8.py tests/test_gpu_configs.py -m gpu -q -x -rf -p no:cacheprovider --timeout 600 > gpurun_out/ab_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab_pytest.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum --clock-control none -k regex:k_i8_prep -s 0 -c 12 --csv --log-file gpurun_out/prep_metrics.csv python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --no-per-config --batch 64 > gpurun_out/ncu5m.log 2>&1
for rep in 1 2; do
timeout 300 python bench.py --config C5 --steps 2 --warmup 2 --no-cpu-baseline --no-per-config > gpurun_out/ab_c5_new_$rep.json 2>gpurun_out/ab_c5_new_$rep.err
done
echo done
