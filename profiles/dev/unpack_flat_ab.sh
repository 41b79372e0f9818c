#!/bin/bash
# Flat bulk-copy expansion (unpack_flat_kernel) vs the per-slice kernel: parity, then timings.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_unpack_flat_gpu.py tests/test_gemm_gpu.py tests/test_batch_gpu.py tests/test_full_parity_gpu.py tests/test_bounds_gpu.py -q -x > gpurun_out/flat_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/flat_tests.log
for f in 0 1 0 1; do echo "== BITMM_UNPACK_FLAT=$f"; BITMM_UNPACK_FLAT=$f python profiles/ab_fx.py paper_2306_08960_b200/libbitmm_b200.so; BITMM_UNPACK_FLAT=$f python profiles/dev/time_1x1.py 2>&1 | tail -3; done
for f in 0 1; do BITMM_UNPACK_FLAT=$f python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('flat=$f', round(d['value'],1), 'frac', round(d['roofline']['frac'],4), 'kernels', d['kernels'], 'seq', round(d['sequential_calls']['value'],1), 'c5', round(d['c5_sweep']['kernel_ms'],3))"; done
