"""A/B of the fp32 APB layer (BASELINE config 4: 3072 x 768 x 8192 tokens, per-row alpha, top-2%
residual): median of 20 L2-flushed launches and the error against the oracle on every row.
BITMM_APB_WIDE=1 python profiles/dev/ab_apb.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2306_08960_b200 import api, data, device  # noqa: E402

rng = np.random.default_rng(2306_08960 + 4)
rows, cols, tokens = 3072, 768, 8192
a, alpha, keep = data.apb_weights(rng, rows, cols)
layer = api.decompose_apb(a, alpha)
x = rng.standard_normal((cols, tokens)).astype(np.float32)
r = layer.residual
T = lambda v: torch.from_numpy(np.ascontiguousarray(v)).cuda()  # noqa: E731
args = (T(layer.bin.words.view(np.int64)), cols, T(alpha), T(r.row_ptr.view(np.int64)),
        T(r.col_idx.view(np.int64)), T(r.vals), T(x))
out = torch.empty((rows, tokens), dtype=torch.float32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    device.layer_forward(*args, out)
device.status()
ts = []
for _ in range(20):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    device.layer_forward(*args, out)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
want = oracle.Oracle().layer_forward(rows, cols, 1.0, layer.bin.words, layer.bin.words_per_row(), r.row_ptr,
                                     r.col_idx, r.vals, x, row_alpha=alpha).astype(np.float64)
got = out.cpu().numpy().astype(np.float64)
rel = np.linalg.norm(got - want) / np.linalg.norm(want)
print(f"WIDE={os.environ.get('BITMM_APB_WIDE', '0')}: {np.median(ts) * 1e3:.1f} us  rel_frob {rel:.2e}  "
      f"max_abs {np.max(np.abs(got - want)):.2e} (max|C| {np.max(np.abs(want)):.2f})", flush=True)
