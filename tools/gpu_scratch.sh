#!/bin/bash
# scratch A/B: w16 variants (a = round-2 baseline, b = opaque+redux static, c = redux+dyn, default = all)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_w16.py tests/test_gpu_select.py -m gpu -q -x -rf -p no:cacheprovider > gpurun_out/ab_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab_pytest.log
for rep in 1 2 3; do
for lib in libexpmb_a.so libexpmb_b.so libexpmb_c.so libexpmb.so; do
EXPMB_LIB=$lib timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-per-config > gpurun_out/ab_${lib}_$rep.json 2>gpurun_out/ab_${lib}_$rep.err
done
done
echo done
