#!/bin/bash
python -m pytest tests/test_gpu_i8.py -q -p no:cacheprovider 2>&1 | tail -1
for i in 1 2; do for v in libexpmb.so libexpmb_a.so; do
EXPMB_LIB=$v python bench.py --config C5 --no-cpu-baseline --steps 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],1), 'ms', round(d['value'],1))"
done; done
