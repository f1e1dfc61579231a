#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_w16.py -m gpu -q -rf -p no:cacheprovider > gpurun_out/s3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s3_pytest.log
for rep in 1 2; do
for lib in libexpmb.so libexpmb_w10.so libexpmb_w12.so; do
EXPMB_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-per-config > gpurun_out/s3_${lib}_$rep.json 2>gpurun_out/s3_${lib}_$rep.err
done
EXPMB_W16_MINB=3 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-per-config > gpurun_out/s3_m3_$rep.json 2>gpurun_out/s3_m3_$rep.err
done
echo done
