#!/bin/bash
# Bench step (device-resident value) A/B of library builds on one box:
#   bash profiles/dev/ab_step_libs.sh build/ab/a.so build/ab/b.so ...
cd $GRAFT_REPO_ROOT
cp paper_2306_08960_b200/libbitmm_b200.so /tmp/lib_keep.so
for r in 1 2; do for lib in "$@"; do
  cp $lib paper_2306_08960_b200/libbitmm_b200.so
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-c5-plan 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$(basename $lib)', round(d['value'],1), 'c5', round(d['c5_sweep']['kernel_ms'],3), '1x1', round(d['routines']['1x1']['ms']*1e3,1))"
done; done
cp /tmp/lib_keep.so paper_2306_08960_b200/libbitmm_b200.so
