#!/bin/bash
# int8-slice stage A/B: libraries (make variant) x env, bit identity vs the default build and C5 step time
mkdir -p gpurun_out
LIBS="libexpmb_bn128c.so libexpmb_bn128c8.so libexpmb_bn128e8.so"
EXPMB_LIB=libexpmb.so timeout 300 python tools/i8_lib_ab.py /tmp/ab_base.npz > gpurun_out/ab_base.log 2>&1
for lib in $LIBS; do
  EXPMB_LIB=$lib timeout 300 python tools/i8_lib_ab.py /tmp/ab_$lib.npz > gpurun_out/ab_$lib.log 2>&1
  EXPMB_I8_PERSIST=1 EXPMB_LIB=$lib timeout 300 python tools/i8_lib_ab.py /tmp/ab_${lib}_p.npz > gpurun_out/ab_${lib}_p.log 2>&1
done
python - > gpurun_out/ab_cmp.log 2>&1 <<'PY'
import glob, numpy as np
a = np.load('/tmp/ab_base.npz')
for f in sorted(glob.glob('/tmp/ab_lib*.npz')):
    try:
        b = np.load(f)
        print(f, all(np.array_equal(a[k], b[k]) for k in a.files), max(float(np.abs(a[k]-b[k]).max()) for k in a.files))
    except Exception as e:
        print(f, 'ERR', e)
PY
for rep in 1 2; do
for lib in $LIBS; do
  EXPMB_LIB=$lib timeout 300 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/c5_${lib}_$rep.json 2>gpurun_out/c5_${lib}_$rep.err
done
EXPMB_I8_PERSIST=1 EXPMB_LIB=libexpmb_bn128c.so timeout 300 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/c5_persist_$rep.json 2>gpurun_out/c5_persist_$rep.err
done
EXPMB_LIB=libexpmb_bn128c8.so ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C5.csv \
    python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --no-per-config --batch 32 > gpurun_out/ncu_l5.log 2>&1
echo done
