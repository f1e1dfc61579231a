#!/bin/bash
for i in 1 2 3; do
python bench.py --config C1 --no-cpu-baseline --steps 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C1 steps20', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
python bench.py --config C1 --no-cpu-baseline --steps 5 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C1 steps5', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done
python -m pytest tests/test_gpu_i8.py -q -p no:cacheprovider 2>&1 | tail -1
for i in 1 2; do python bench.py --config C5 --no-cpu-baseline --steps 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5', round(d['ms_per_step'],1), round(d['value'],1))"; done
