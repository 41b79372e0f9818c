"""Standalone exact spmm_csr at the config-4 shape (3072 x 768 CSR, top-2% residual, times a
768 x 8192 fp32 X): the 64-token persistent kernel (default) against the 32-token chunk kernel
(BITMM_SPMM_V1=1). python profiles/dev/time_spmm.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2306_08960_b200 import _lib, api, data  # noqa: E402

lib = _lib.load()
rng = np.random.default_rng(7)
rows, cols, tokens = 3072, 768, 8192
a, alpha, _ = data.apb_weights(rng, rows, cols)
r = api.decompose_apb(a, alpha).residual
x = rng.standard_normal((cols, tokens)).astype(np.float32)
T = lambda v: torch.from_numpy(np.ascontiguousarray(v)).cuda()  # noqa: E731
d = [T(r.row_ptr.view(np.int64)), T(r.col_idx.view(np.int64)), T(r.vals), T(x)]
s = torch.cuda.current_stream().cuda_stream
outs = {}
for mode in ("0", "1"):
    os.environ["BITMM_SPMM_V1"] = mode
    out = torch.empty((rows, tokens), dtype=torch.float32, device="cuda")

    def call():
        assert lib.bitmm_spmm_csr_dev(rows, cols, d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr(),
                                      d[3].data_ptr(), tokens, tokens, out.data_ptr(), tokens, s) == 0
    for _ in range(5):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        call()
    e1.record()
    torch.cuda.synchronize()
    outs[mode] = out
    print(f"BITMM_SPMM_V1={mode}: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us/call")
print("bit-identical:", torch.equal(outs["0"], outs["1"]))
