mkdir -p gpurun_out
for c in C2 C1; do python bench.py --config $c --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'])"; done > gpurun_out/q.txt 2>&1
