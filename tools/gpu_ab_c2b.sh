#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "golden_fp32 or ragged or C2" > gpurun_out/pytest_ab.log 2>&1; tail -1 gpurun_out/pytest_ab.log
for i in 1 2 3; do
for v in libexpmb.so libexpmb_a.so; do
EXPMB_LIB=$v python bench.py --no-cpu-baseline --steps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step']*1e3,1), 'us')"
done; done
