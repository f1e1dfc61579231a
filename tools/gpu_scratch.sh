#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-per-config > gpurun_out/s4_base_$rep.json 2>gpurun_out/s4_base_$rep.err
EXPMB_LIB=libexpmb_w6.so EXPMB_W16_Q=8 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-per-config > gpurun_out/s4_q8w6_$rep.json 2>gpurun_out/s4_q8w6_$rep.err
EXPMB_LIB=libexpmb_w4.so EXPMB_W16_Q=8 EXPMB_W16_MINB=3 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-per-config > gpurun_out/s4_q8w4m3_$rep.json 2>gpurun_out/s4_q8w4m3_$rep.err
EXPMB_LIB=libexpmb_w6.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-per-config > gpurun_out/s4_q4w6_$rep.json 2>gpurun_out/s4_q4w6_$rep.err
done
echo done
