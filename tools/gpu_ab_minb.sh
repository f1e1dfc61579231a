#!/bin/bash
for i in 1 2; do for mb in 2 3 4; do
EXPMB_C2_MINB=$mb python bench.py --no-cpu-baseline --steps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('minb $mb', round(d['ms_per_step']*1e3,1), 'us')"
done; done
