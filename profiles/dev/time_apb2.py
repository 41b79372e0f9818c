"""Chained time of the 2-bit APB layer (BASELINE config 4 shape, 3072 x 768 weights, 8192
tokens): fused residual, two-pass with the bf16-level SpMM, two-pass with the fp32-level SpMM.
python profiles/dev/time_apb2.py"""
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
layer = api.decompose_apb(a, alpha)
r = layer.residual
t, h, m, wpr = data.random_planes(rng, tokens, cols)
T = lambda v: torch.from_numpy(np.ascontiguousarray(v)).cuda()  # noqa: E731
d = [T(layer.bin.words.view(np.int64)), T(alpha), T(r.row_ptr.view(np.int64)), T(r.col_idx.view(np.int64)),
     T(r.vals), T(t.view(np.int64)), T(h.view(np.int64)), T(m.view(np.int64))]
s = torch.cuda.current_stream().cuda_stream
P = lambda x: x.data_ptr()  # noqa: E731
outs = {}
MODES = {"fused": {"BITMM_APB2_FUSED": "1", "BITMM_APB2_L8": "1"},
         "fused bf16 chunks": {"BITMM_APB2_FUSED": "1", "BITMM_APB2_L8": "0"},
         "two-pass bf16 levels": {"BITMM_APB2_FUSED": "0", "BITMM_SPMM_LEVELS_V1": "0"},
         "two-pass fp32 levels (v1)": {"BITMM_APB2_FUSED": "0", "BITMM_SPMM_LEVELS_V1": "1"}}
only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
for mode, env in MODES.items():
    if only and mode != only:
        continue
    os.environ.update(env)
    out = torch.empty((rows, tokens), dtype=torch.float32, device="cuda")

    def call():
        assert lib.bitmm_layer_forward_2bit_dev(rows, cols, 1.0, P(d[1]), P(d[0]), wpr, P(d[2]), P(d[3]),
                                                P(d[4]), P(d[5]), P(d[6]), P(d[7]), tokens, 0.5, 0, 1.0, P(out),
                                                tokens, s) == 0
    for _ in range(5):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    outs[mode] = out
    print(f"{mode}: {e0.elapsed_time(e1) / reps * 1e3:.1f} us/call")
if not only:
    ref = outs["two-pass fp32 levels (v1)"]
    print("bit-identical to v1:", {k: torch.equal(v, ref) for k, v in outs.items()})
