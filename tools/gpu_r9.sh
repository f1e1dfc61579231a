mkdir -p gpurun_out
timeout 300 python bench.py --config C5 --steps 4 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/r9_C5.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r9_launch_C5.csv python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --no-per-config --batch 32 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_lowrank.py tests/test_gpu_i8.py tests/test_gpu_timegrid.py -q -x > gpurun_out/r9_pytest.log 2>&1
echo done
