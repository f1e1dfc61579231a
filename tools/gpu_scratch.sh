#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_i8.py -m gpu -q -x -rf -p no:cacheprovider > gpurun_out/s15_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s15_pytest.log
if grep -q "rc=0" gpurun_out/s15_pytest.log; then
for rep in 1 2; do
timeout 300 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/s15_m3_$rep.json 2>gpurun_out/s15_m3_$rep.err
EXPMB_LIB=libexpmb_p4.so timeout 300 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/s15_m4_$rep.json 2>gpurun_out/s15_m4_$rep.err
done
fi
echo done
