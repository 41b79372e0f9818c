#!/bin/bash
# compute-sanitizer, ONE tool per gpurun call (B200_PROFILING.md), after a clean plain run of the
# same smoke-size driver: bash profiles/dev/sanitize.sh memcheck|racecheck|synccheck|initcheck
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TOOL=${1:-memcheck}
timeout 300 python profiles/dev/sanitize_smoke.py > gpurun_out/san_plain.log 2>&1; rc=$?; echo "plain rc=$rc"; tail -2 gpurun_out/san_plain.log
[ $rc -eq 0 ] || exit 1
timeout 1500 compute-sanitizer --tool $TOOL --print-limit 50 python profiles/dev/sanitize_smoke.py > gpurun_out/san_$TOOL.log 2>&1
echo "sanitizer rc=$?"; tail -15 gpurun_out/san_$TOOL.log
