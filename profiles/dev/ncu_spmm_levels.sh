#!/bin/bash
# ncu of the 2-bit APB layer (config 4 shape, profiles/dev/time_apb2.py): the launch list of one
# layer call (per-kernel durations) and a full capture of the residual pass (spmm_levels_kernel).
# Usage (on the GPU box): bash profiles/dev/ncu_spmm_levels.sh TAG
set -e
tag=${1:-r02}
mkdir -p gpurun_out
BITMM_APB2_FUSED=0 python profiles/dev/time_apb2.py > gpurun_out/time_apb2_$tag.log 2>&1
export BITMM_APB2_FUSED=0 BITMM_SPMM_LEVELS_V1=0
ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 8 --csv \
  python profiles/dev/time_apb2.py --only "two-pass bf16 levels" > gpurun_out/launches_apb2_$tag.csv 2>&1
ncu --set full --import-source on --clock-control none -k regex:spmm_levels -s 3 -c 1 \
  -o gpurun_out/spmm_levels_$tag -f \
  python profiles/dev/time_apb2.py --only "two-pass bf16 levels" > gpurun_out/ncu_spmm_levels_$tag.log 2>&1
