#!/bin/bash
# int8-slice (Ozaki) tensor-core path, opt-in EXPMB_I8=1: parity + speed
mkdir -p gpurun_out
EXPMB_I8=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -x -p no:cacheprovider -k "C5 or C3 or odd or large_path" > gpurun_out/pytest_i8.log 2>&1; tail -3 gpurun_out/pytest_i8.log
grep -E "subset|worst" gpurun_out/pytest_i8.log | head
for c in C5 C3 C4; do
EXPMB_I8=1 timeout 600 python bench.py --config $c --no-cpu-baseline --steps 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('I8 $c', round(d['ms_per_step'],2), 'ms', d['value'])"
done
