"""A/B of spmm_levels_kernel build variants (-DSL_THREADS_CFG, -DSL_MINB_CFG, -DSL_CPREF) on the
2-bit APB layer, config 4 shape. Each argument is a library built with
`python -m paper_2306_08960_b200.build --out build/ab/NAME.so -- -D...`.
python profiles/dev/ab_spmm_levels.py build/ab/a.so build/ab/b.so ..."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2306_08960_b200 import _lib, api, data  # noqa: E402

os.environ["BITMM_APB2_FUSED"] = os.environ.get("AB_FUSED", "0")  # AB_FUSED=1: time the fused form
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
ref = None
for path in sys.argv[1:]:
    lib = C.CDLL(os.path.abspath(path))
    for name, (res, args) in _lib.SIGNATURES.items():
        if hasattr(lib, name):
            getattr(lib, name).restype = res
            getattr(lib, name).argtypes = args
    out = torch.empty((rows, tokens), dtype=torch.float32, device="cuda")

    def call():
        assert lib.bitmm_layer_forward_2bit_dev(rows, cols, 1.0, P(d[1]), P(d[0]), wpr, P(d[2]), P(d[3]),
                                                P(d[4]), P(d[5]), P(d[6]), P(d[7]), tokens, 0.5, 0, 1.0, P(out),
                                                tokens, s) == 0
    for _ in range(5):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        call()
    e1.record()
    torch.cuda.synchronize()
    if ref is None:
        ref = out.clone()
    print(f"{os.path.basename(path)}: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us/call, same as first: {torch.equal(out, ref)}")
