#!/bin/bash
# tcgen05 3xTF32 path (EXPMB_TC=1) with 4 accumulators: C3/C5 parity + speed
mkdir -p gpurun_out
EXPMB_TC=1 python -m pytest tests/test_gpu_parity.py -q -s -p no:cacheprovider -k "C3 or C5 or odd or large_path" > gpurun_out/pytest_tc.log 2>&1; tail -3 gpurun_out/pytest_tc.log
grep -E "C3|C5|worst" gpurun_out/pytest_tc.log | head
for c in C3 C5; do
EXPMB_TC=1 python bench.py --config $c --no-cpu-baseline --steps 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TC $c', round(d['ms_per_step'],2), 'ms', d['value'])"
python bench.py --config $c --no-cpu-baseline --steps 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('SIMT $c', round(d['ms_per_step'],2), 'ms', d['value'])"
done
