#!/bin/bash
# Template for a same-box A/B on the GPU box: build the committed tree as
# paper_2512_20777_b200/libexpmb_a.so (git archive HEAD + nvcc, or make variant
# VNAME=a VFLAGS=...), then compare it with the working tree's default build.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_i8.py tests/test_gpu_w16.py -m gpu -q -x -rf -p no:cacheprovider --timeout 600 > gpurun_out/ab_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab_pytest.log
for rep in 1 2; do
for cfg in C2 C5; do
timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-per-config > gpurun_out/ab_${cfg}_new_$rep.json 2>gpurun_out/ab_${cfg}_new_$rep.err
EXPMB_LIB=libexpmb_a.so timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-per-config > gpurun_out/ab_${cfg}_head_$rep.json 2>gpurun_out/ab_${cfg}_head_$rep.err
done
done
echo done
