#!/bin/bash
mkdir -p gpurun_out
for w in 0 1; do EXPMB_W16=$w timeout 300 python tools/w16_check.py > gpurun_out/w16d_check_$w.log 2>&1; done
for rep in 1 2; do
for lib in libexpmb.so libexpmb_acc1.so libexpmb_acc2.so; do
EXPMB_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-per-config > gpurun_out/w16d_${lib}_$rep.json 2>gpurun_out/w16d_${lib}_$rep.err
done
EXPMB_W16_MINB=3 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-per-config > gpurun_out/w16d_m3_$rep.json 2>gpurun_out/w16d_m3_$rep.err
EXPMB_W16_Q=2 EXPMB_W16_MINB=3 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-per-config > gpurun_out/w16d_q2m3_$rep.json 2>gpurun_out/w16d_q2m3_$rep.err
EXPMB_LIB=libexpmb_acc2.so EXPMB_W16_MINB=3 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-per-config > gpurun_out/w16d_acc2m3_$rep.json 2>gpurun_out/w16d_acc2m3_$rep.err
done
echo done
