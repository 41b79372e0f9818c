#!/bin/bash
# One gpurun session: smoke, GPU tests, bench, then ncu (launch list + full capture of the
# top kernel), each ncu pass only after the identical command exited 0 without ncu.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${1:-r01}
BENCH_SMALL="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; cat gpurun_out/bench_$TAG.json
if [ "${NCU:-1}" = "1" ]; then
  timeout 300 $BENCH_SMALL > gpurun_out/plain_$TAG.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches_$TAG.csv $BENCH_SMALL > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
  timeout 300 $BENCH_SMALL > gpurun_out/plain2_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 2 \
      -o gpurun_out/prof_tc_$TAG $BENCH_SMALL > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
fi
