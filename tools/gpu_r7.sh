mkdir -p gpurun_out
for rep in 1 2; do
timeout 300 python bench.py --config C5 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/r7_np_$rep.json 2>/dev/null
EXPMB_I8_PERSIST=1 timeout 300 python bench.py --config C5 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/r7_p_$rep.json 2>/dev/null
done
timeout 900 python -m pytest tests/test_gpu_select.py tests/test_gpu_i8.py tests/test_gpu_parity.py -q -x -k "baseline or select or i8 or graph" > gpurun_out/r7_pytest.log 2>&1
echo done
