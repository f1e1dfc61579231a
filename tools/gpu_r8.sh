mkdir -p gpurun_out
for lib in libexpmb.so libexpmb_ten.so libexpmb_old.so; do
EXPMB_LIB=$lib timeout 300 python bench.py --config C5 --steps 4 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/r8_$lib.json 2>/dev/null
done
for lib in libexpmb.so libexpmb_old.so; do
EXPMB_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r8_launch_$lib.csv python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --no-per-config --batch 32 > /dev/null 2>&1
done
timeout 600 python -m pytest tests/test_gpu_timegrid.py -q -x > gpurun_out/r8_pytest.log 2>&1
echo done
