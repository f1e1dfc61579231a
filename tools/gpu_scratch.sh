#!/bin/bash
# scratch A/B runner (overwritten per experiment; results land in gpurun_out/)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_w16.py tests/test_gpu_select.py tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -rf -p no:cacheprovider > gpurun_out/s_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s_pytest.log
for rep in 1 2; do
for lib in libexpmb.so libexpmb_p1.so; do
EXPMB_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-per-config > gpurun_out/s_${lib}_$rep.json 2>gpurun_out/s_${lib}_$rep.err
done
done
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/plain_s.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:w16 -s 3 -c 1 \
    -o gpurun_out/prof_s -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/ncu_s.log 2>&1
echo done
