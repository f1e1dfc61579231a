# device scheduler + persistent stage kernels: quick i8 smoke under a short timeout first
mkdir -p gpurun_out
timeout 120 python -c "
import torch, paper_2512_20777_b200 as X
W = torch.randn(4, 2048, 2048, device='cuda') / 45
r = X.expm(W, 2.0**-24); torch.cuda.synchronize(); print('i8 ok', r.plan.s.tolist())
W = torch.randn(6, 256, 256, device='cuda') / 5
r = X.expm(W, 2.0**-24); torch.cuda.synchronize(); print('ffma ok', r.plan.s.tolist())
" > gpurun_out/r2_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2_smoke.log
grep -q "ffma ok" gpurun_out/r2_smoke.log || exit 3
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider -x --timeout 600 > gpurun_out/r2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pytest.log
for c in C3 C4 C5; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_$c.json 2> gpurun_out/r2_bench_$c.err
done
echo done
