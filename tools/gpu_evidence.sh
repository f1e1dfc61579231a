#!/bin/bash
# Full evidence run: GPU tests, default bench (C2, with CPU baseline), reference arm,
# per-config bench lines, launch list + full ncu capture of the C2 kernel.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
for c in C1 C3 C4; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 1200 python bench.py --config C5 --steps 2 --warmup 3 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:expm_fused -s 3 -c 1 \
    -o gpurun_out/prof_C2 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1
echo done
python bench.py --scheme baseline > gpurun_out/bench_C2_alg1.json 2> gpurun_out/bench_C2_alg1.err
python bench.py --config C1 --scheme baseline --no-cpu-baseline > gpurun_out/bench_C1_alg1.json 2> gpurun_out/bench_C1_alg1.err
python bench.py --config C1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dmma -s 3 -c 1 \
    -o gpurun_out/prof_C1 -f python bench.py --config C1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu3.log 2>&1
python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_stage -s 20 -c 1 \
    -o gpurun_out/prof_C4 -f python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_p4.log 2>&1
python bench.py --config C3 --timegrid --steps 5 --warmup 3 > gpurun_out/bench_C3_timegrid.json 2> gpurun_out/bench_C3_timegrid.err
python bench.py --config LR > gpurun_out/bench_LR.json 2> gpurun_out/bench_LR.err
python bench.py --config LR --impl reference --steps 3 --warmup 1 > gpurun_out/bench_LR_reference.json 2> gpurun_out/bench_LR_reference.err
echo done2
