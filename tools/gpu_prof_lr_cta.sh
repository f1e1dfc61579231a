#!/bin/bash
# ncu capture of the low-rank CTA kernel at n = 64, t = 32
set -e
python tools/lr_one.py 64 32 16384
ncu --set full --clock-control none --import-source on -k regex:expm_lowrank_kernel -s 1 -c 1 \
  -o gpurun_out/lr_cta_t32 -f python tools/lr_one.py 64 32 16384 > gpurun_out/lr_cta_ncu.log 2>&1
