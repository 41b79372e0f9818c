#!/bin/bash
# A/B of the staged copy's host side (see run_staged): calling thread vs the host pool (with
# CUDA waits on the pool or not, 4-16 threads), and glibc keeping freed DenseMatrix memory.
cd $GRAFT_REPO_ROOT
for v in "BITMM_STAGED_POOL=0" "BITMM_STAGED_POOL=1" "BITMM_STAGED_POOL=2 BITMM_HOST_THREADS=4" "BITMM_STAGED_POOL=1 MALLOC_MMAP_THRESHOLD_=67108864" "BITMM_STAGED_POOL=0 MALLOC_MMAP_THRESHOLD_=67108864"; do
  echo "== $v"; env $v BITMM_STAGED_TRACE=1 ./oracle/_ref/latency_b200 1024 1024 1024 7 2>&1 | tail -5
done
