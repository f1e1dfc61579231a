mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r1_smi.txt
./tools/peaks > gpurun_out/r1_peaks.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf -p no:cacheprovider -x > gpurun_out/r1_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r1_pytest.log
timeout 900 python bench.py > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r1_ref.json 2> gpurun_out/r1_ref.err
echo done
