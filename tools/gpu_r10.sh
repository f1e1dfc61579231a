mkdir -p gpurun_out
timeout 600 python tools/fused_tile_bench.py gpurun_out/r10_fused_tile.json > gpurun_out/r10_fused_tile.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x -rf > gpurun_out/r10_pytest.log 2>&1
for c in C3 C4; do timeout 300 python bench.py --config $c --steps 4 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/r10_$c.json 2>/dev/null; done
EXPMB_FUSED_TILE_MAX=256 timeout 300 python bench.py --config C3 --steps 4 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/r10_C3_fused.json 2>/dev/null
echo done
