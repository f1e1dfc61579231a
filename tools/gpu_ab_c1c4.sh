#!/bin/bash
python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "C1 or C4 or golden_fp64 or ragged or odd" 2>&1 | tail -1
for i in 1 2; do for v in libexpmb.so libexpmb_a.so; do
EXPMB_LIB=$v python bench.py --config C1 --no-cpu-baseline --steps 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v C1', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3))"
EXPMB_LIB=$v python bench.py --config C4 --no-cpu-baseline --steps 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v C4', round(d['ms_per_step'],2), 'ms', round(d['roofline']['frac'],3))"
done; done
