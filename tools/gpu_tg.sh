#!/bin/bash
mkdir -p gpurun_out
python bench.py --config C3 --timegrid --steps 5 --warmup 3 > gpurun_out/bench_C3_timegrid.json 2> gpurun_out/bench_C3_timegrid.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_C3_timegrid.json').read().strip().splitlines()[-1])
print('C3tg', d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'], d['gpu_launches'])"
tail -3 gpurun_out/bench_C3_timegrid.err
