mkdir -p gpurun_out
for c in C5 C3 C4; do
EXPMB_DEBUG_OCC=1 timeout 300 python bench.py --config $c --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/r6_$c.json 2>gpurun_out/r6_$c.err
EXPMB_LIB=libexpmb_old.so timeout 300 python bench.py --config $c --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/r6_old_$c.json 2>/dev/null
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-per-config > gpurun_out/r6_C2.json 2>/dev/null
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r6_pytest.log 2>&1
echo done
