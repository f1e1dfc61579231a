#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_i8.py -m gpu -q -x -rf -p no:cacheprovider --timeout 600 > gpurun_out/ab_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab_pytest.log
for rep in 1 2; do
timeout 300 python bench.py --config C5 --steps 2 --warmup 2 --no-cpu-baseline --no-per-config > gpurun_out/ab_c5_prep1_$rep.json 2>gpurun_out/ab_c5_prep1_$rep.err
EXPMB_I8_PREP=0 timeout 300 python bench.py --config C5 --steps 2 --warmup 2 --no-cpu-baseline --no-per-config > gpurun_out/ab_c5_prep0_$rep.json 2>gpurun_out/ab_c5_prep0_$rep.err
done
echo done
