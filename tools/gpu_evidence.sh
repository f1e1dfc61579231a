#!/bin/bash
# Full evidence run (round 2): GPU tests, smoke, default bench (C2 headline +
# per_config C1/C3/C4/C5, CPU baseline), reference arm, Alg. 1 / time-grid /
# low-rank lines, then the C2 launch list and one ncu --set full capture each
# of the C2 (w16) kernel; tools/gpu_evidence_b.sh has the C1 / C5 captures.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 300 python bench.py --scheme baseline --no-per-config > gpurun_out/bench_C2_alg1.json 2> gpurun_out/bench_C2_alg1.err
timeout 300 python bench.py --config C1 --scheme baseline --no-cpu-baseline > gpurun_out/bench_C1_alg1.json 2> gpurun_out/bench_C1_alg1.err
timeout 600 python bench.py --config C3 --timegrid --steps 5 --warmup 3 > gpurun_out/bench_C3_timegrid.json 2> gpurun_out/bench_C3_timegrid.err
timeout 600 python bench.py --config LR > gpurun_out/bench_LR.json 2> gpurun_out/bench_LR.err
timeout 600 python bench.py --config LR --impl reference --steps 3 --warmup 1 > gpurun_out/bench_LR_reference.json 2> gpurun_out/bench_LR_reference.err
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:w16 -s 3 -c 1 \
    -o gpurun_out/prof_C2 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/ncu2.log 2>&1
echo done
