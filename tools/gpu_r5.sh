mkdir -p gpurun_out
EXPMB_DEBUG_OCC=1 timeout 300 python bench.py --config C5 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/r5_C5.json 2>gpurun_out/r5_C5.err
EXPMB_DEBUG_OCC=1 timeout 300 python bench.py --config C3 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/r5_C3.json 2>gpurun_out/r5_C3.err
EXPMB_DEBUG_OCC=1 timeout 300 python bench.py --config C4 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/r5_C4.json 2>gpurun_out/r5_C4.err
timeout 900 python -m pytest tests/test_gpu_select.py tests/test_gpu_i8.py tests/test_gpu_shards.py -q -x > gpurun_out/r5_pytest.log 2>&1
echo done
