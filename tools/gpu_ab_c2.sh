# A/B of C2 kernel variants (same box), then the int8 path after the persistent-loop fixes
mkdir -p gpurun_out
for rep in 1 2; do
for lib in libexpmb.so libexpmb_c2a.so libexpmb_c2i.so libexpmb_c2n.so libexpmb_c2ain.so; do
  EXPMB_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-per-config > gpurun_out/c2ab_${rep}_${lib}.json 2>/dev/null
done
done
for c in C5 C3; do
  timeout 300 python bench.py --config $c --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/r4_$c.json 2>gpurun_out/r4_$c.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_i8_stage -s 30 -c 1 -o gpurun_out/r4_i8stage -f python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --batch 8 > gpurun_out/r4_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_i8_stats -s 30 -c 1 -o gpurun_out/r4_i8stats -f python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --batch 8 > gpurun_out/r4_ncu2.log 2>&1
echo done
