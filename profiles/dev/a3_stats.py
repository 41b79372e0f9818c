"""Per-role cycle counters of the fused 2-bit APB layer (a -DA3_STATS build of the library).
python -m paper_2306_08960_b200.build --out build/ab/a3.so -- -DA3_STATS
python profiles/dev/a3_stats.py build/ab/a3.so"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2306_08960_b200 import _lib, api, data  # noqa: E402

lib = C.CDLL(os.path.abspath(sys.argv[1]))
for name, (res, args) in _lib.SIGNATURES.items():
    if hasattr(lib, name):
        getattr(lib, name).restype = res
        getattr(lib, name).argtypes = args
rng = np.random.default_rng(7)
rows, cols, tokens = 3072, 768, 8192
a, alpha, _ = data.apb_weights(rng, rows, cols)
layer = api.decompose_apb(a, alpha)
r = layer.residual
t, h, m, wpr = data.random_planes(rng, tokens, cols)
T = lambda v: torch.from_numpy(np.ascontiguousarray(v)).cuda()  # noqa: E731
d = [T(layer.bin.words.view(np.int64)), T(alpha), T(r.row_ptr.view(np.int64)), T(r.col_idx.view(np.int64)),
     T(r.vals), T(t.view(np.int64)), T(h.view(np.int64)), T(m.view(np.int64))]
out = torch.empty((rows, tokens), dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
P = lambda x: x.data_ptr()  # noqa: E731
for _ in range(3):
    assert lib.bitmm_layer_forward_2bit_dev(rows, cols, 1.0, P(d[1]), P(d[0]), wpr, P(d[2]), P(d[3]), P(d[4]),
                                            P(d[5]), P(d[6]), P(d[7]), tokens, 0.5, 0, 1.0, P(out), tokens, s) == 0
torch.cuda.synchronize()
buf = (C.c_ulonglong * (8 * 160))()
lib.bitmm_debug_a3_stats(buf)
st = np.frombuffer(buf, dtype=np.uint64).reshape(8, 160).astype(np.float64)
nz = st[3] > 0
names = ["res_staging", "res_compute", "res_wait_free", "res_total", "epi_wait_acc", "epi_wait_S", "epi_work",
         "epi_store_wait"]
print({n: int(st[i][nz].mean()) for i, n in enumerate(names)})
print("res_total min/max", int(st[3][nz].min()), int(st[3][nz].max()))
