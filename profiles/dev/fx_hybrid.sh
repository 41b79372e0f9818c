#!/bin/bash
# In-GEMM expansion, hybrid (BITMM_FX=2: A expanded by unpack_operands, B inside the GEMM):
# bit-exactness, then per-call timings against the default path and the full fx path.
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_fx_gpu.py -q -x 2>&1 | tail -3
for fx in 0 2 1 2 0; do echo "== BITMM_FX=$fx"; BITMM_FX=$fx timeout 300 python profiles/ab_fx.py paper_2306_08960_b200/libbitmm_b200.so; done
