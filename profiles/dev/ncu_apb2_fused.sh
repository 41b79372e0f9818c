#!/bin/bash
# ncu of the fused 2-bit APB layer (config 4 shape, profiles/dev/time_apb2.py): the launch list of
# one layer call and a full capture of apb2_fused_kernel. Usage (GPU box): bash profiles/dev/ncu_apb2_fused.sh TAG
set -e
tag=${1:-r02}
mkdir -p gpurun_out
python profiles/dev/time_apb2.py > gpurun_out/time_apb2_$tag.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 6 --csv \
  python profiles/dev/time_apb2.py --only fused > gpurun_out/launches_apb2f_$tag.csv 2>&1
ncu --set full --import-source on --clock-control none -k regex:apb2_fused -s 3 -c 1 \
  -o gpurun_out/apb2_fused_$tag -f python profiles/dev/time_apb2.py --only fused > gpurun_out/ncu_apb2_fused_$tag.log 2>&1
