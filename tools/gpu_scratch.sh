#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
for lib in libexpmb_old.so libexpmb_c686.so libexpmb.so; do
for c in C3 C4; do
EXPMB_LIB=$lib timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/s7_${c}_${lib}_$rep.json 2>gpurun_out/s7_${c}_${lib}_$rep.err
done
done
done
echo done
