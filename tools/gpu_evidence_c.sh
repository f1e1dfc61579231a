#!/bin/bash
# Evidence part C: C5 launch list (full batch), per-launch metrics of the
# twelve int8 stage launches of a 64-matrix chunk (W^2, E1-E3, squarings) and
# one k_i8_prep capture.
mkdir -p gpurun_out
python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --no-per-config > gpurun_out/plain5f.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C5.csv \
    python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --no-per-config > gpurun_out/ll_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:k_i8_stage -s 0 -c 12 --csv --log-file gpurun_out/stage_metrics.csv \
    python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --no-per-config --batch 64 > gpurun_out/ncu5m.log 2>&1
ncu --set full --clock-control none -k regex:k_i8_prep -s 6 -c 1 \
    -o gpurun_out/prof_prep -f python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --no-per-config --batch 64 > gpurun_out/ncuprep.log 2>&1
timeout 600 python tools/i8_crossover.py > gpurun_out/i8_crossover.txt 2>&1
echo done
