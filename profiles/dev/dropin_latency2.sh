#!/bin/bash
# A/B of the staged copy's host side (see run_staged): plain memcpy vs streaming stores.
cd $GRAFT_REPO_ROOT
for v in "BITMM_STAGED_NT=0" "BITMM_STAGED_NT=1" "BITMM_STAGED_NT=0" "BITMM_STAGED_NT=1"; do
  echo "== $v"; env $v BITMM_STAGED_TRACE=1 ./oracle/_ref/latency_b200 1024 1024 1024 9 2>&1 | tail -5
done
