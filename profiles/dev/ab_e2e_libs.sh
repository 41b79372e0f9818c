#!/bin/bash
# e2e A/B of two library builds on one box: bash profiles/dev/ab_e2e_libs.sh build/ab/a.so build/ab/b.so
cd $GRAFT_REPO_ROOT
cp paper_2306_08960_b200/libbitmm_b200.so /tmp/lib_keep.so
for r in 1 2 3; do for lib in "$@"; do cp $lib paper_2306_08960_b200/libbitmm_b200.so; python profiles/dev/e2e_ab.py $(basename $lib); done; done
cp /tmp/lib_keep.so paper_2306_08960_b200/libbitmm_b200.so
