#!/bin/bash
# quick loop: parity subset + C2/C1 bench + C2 ncu capture
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "C2 or C1 or golden or ragged or named" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
python bench.py --config C1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C1.json 2> gpurun_out/bench_C1.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:expm_fused -s 3 -c 1 \
    -o gpurun_out/prof_C2 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1
echo done
python bench.py --config C1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:expm_fused -s 3 -c 1 \
    -o gpurun_out/prof_C1 -f python bench.py --config C1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu3.log 2>&1
