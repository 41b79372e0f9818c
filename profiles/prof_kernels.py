"""Profiling driver (one pass of each hot-path routine at its BASELINE size, after one
warm pass) for `ncu --set full` captures. Not a benchmark: run bench.py for numbers."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2306_08960_b200 import api, data, device  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
rng = np.random.default_rng(1)
T = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()  # noqa: E731
k = 4096
a, _ = data.random_words(rng, 4096, k)
b, _ = data.random_words(rng, 4096, k)
t, h, m, _ = data.random_planes(rng, 8192, k)
da, db, dt, dh, dm = T(a), T(b), T(t), T(h), T(m)
u = torch.empty((4096, 8192), dtype=torch.int32, device="cuda")
f = torch.empty((4096, 8192), dtype=torch.float32, device="cuda")
gam = torch.rand(4096, device="cuda") + 0.5
bet = torch.rand(8192, device="cuda") + 0.5
rows, cols, tokens = 3072, 768, 8192
w, alpha, _ = data.apb_weights(rng, rows, cols)
layer = api.decompose_apb(w, alpha)
x = torch.randn(cols, tokens, device="cuda")
r = layer.residual
Tf = lambda v: torch.from_numpy(np.ascontiguousarray(v)).cuda()  # noqa: E731
apb_args = (T(layer.bin.words), cols, Tf(alpha), T(r.row_ptr), T(r.col_idx), Tf(r.vals), x,
            torch.empty((rows, tokens), device="cuda"))
for _ in range(2):
    if which in ("all", "1x1"):
        device.gemm_1x1(da, db, k, units=u[:, :4096].contiguous() if False else torch.empty((4096, 4096), dtype=torch.int32, device="cuda"))
    if which in ("all", "1x2"):
        device.gemm_1x2(da, 1.0, dt, dh, dm, k, row_scale=gam, col_scale=bet, out=f)
    if which in ("all", "2x2"):
        device.gemm_2x2(dt[:4096], dh[:4096], dm[:4096], dt[4096:], dh[4096:], dm[4096:], k,
                        units=torch.empty((4096, 4096), dtype=torch.int32, device="cuda"))
    if which in ("all", "apb"):
        device.layer_forward(*apb_args)
    torch.cuda.synchronize()
device.status()
print("ok")
