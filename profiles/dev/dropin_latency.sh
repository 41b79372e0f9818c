#!/bin/bash
# Drop-in per-call latency: the late-output / staged-copy tests, then latency_b200 (the
# reference bench_routine through the drop-in) with and without the late overlap.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_late_output_gpu.py tests/test_host_pipeline_gpu.py tests/test_dropin_gpu.py tests/test_reentrancy_gpu.py -q -x > gpurun_out/lat_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/lat_tests.log
nproc; lscpu | grep -i "model name\|numa\|socket"
for v in "" "BITMM_STAGED_POOL=0" "BITMM_LATE_EAGER=1" "BITMM_LATE_EAGER=1 BITMM_HOST_STAGED=0"; do
  echo "== $v"; env $v ./oracle/_ref/latency_b200; env $v ./oracle/_ref/latency_b200 256 256 256 21
done
BITMM_STAGED_TRACE=1 ./oracle/_ref/latency_b200 1024 1024 1024 5 2>&1 | tail -8
BITMM_STAGED_TRACE=1 BITMM_STAGED_POOL=0 ./oracle/_ref/latency_b200 1024 1024 1024 5 2>&1 | tail -8
./oracle/_ref/acceptance_b200 2>&1 | tail -3
