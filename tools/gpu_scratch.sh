#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_i8.py -m gpu -q -x -rf -p no:cacheprovider > gpurun_out/s8_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s8_pytest.log
if grep -q "rc=0" gpurun_out/s8_pytest.log; then
for rep in 1 2; do
timeout 300 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/s8_mc_$rep.json 2>gpurun_out/s8_mc_$rep.err
EXPMB_I8_MC=0 timeout 300 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/s8_nomc_$rep.json 2>gpurun_out/s8_nomc_$rep.err
done
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_shards.py tests/test_gpu_parity.py -m gpu -q -rf -p no:cacheprovider > gpurun_out/s8_pytest2.log 2>&1; echo "rc=$?" >> gpurun_out/s8_pytest2.log
fi
echo done
