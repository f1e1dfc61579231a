# A/B: old (host-sync scheduler, non-persistent stages) vs new builds on C3/C4/C5 + launch lists
mkdir -p gpurun_out
for lib in libexpmb_old.so libexpmb.so libexpmb_ten.so; do
  for c in C5 C3 C4; do
    EXPMB_LIB=$lib timeout 300 python bench.py --config $c --steps 4 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/ab_${lib}_$c.json 2>gpurun_out/ab_${lib}_$c.err
  done
done
for lib in libexpmb_old.so libexpmb.so; do
EXPMB_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_launch_${lib}_C5.csv python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --batch 32 > /dev/null 2>&1
EXPMB_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_launch_${lib}_C3.csv python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --batch 512 > /dev/null 2>&1
done
echo done
