#!/bin/bash
for i in 1 2; do for f in write writeread; do for c in C2 C1; do
BENCH_FLUSH=$f python bench.py --config $c --no-cpu-baseline --steps 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f $c', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3))"
done; done; done
