"""Grouped (bitmm_gemm_batch_dev) vs per-routine timing of the bench GEMMs, by group composition."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2306_08960_b200 import data, device
rng = np.random.default_rng(1)
k = 4096
T = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()  # noqa: E731
a, wpr = data.random_words(rng, 4096, k)
b, _ = data.random_words(rng, 4096, k)
t, h, m, _ = data.random_planes(rng, 8192, k)
wt, wh, wm, _ = data.random_planes(rng, 4096, k)
da, db, dt, dh, dm, dwt, dwh, dwm = map(T, (a, b, t, h, m, wt, wh, wm))
u = torch.empty((4096, 4096), dtype=torch.int32, device="cuda")
u2 = torch.empty((4096, 4096), dtype=torch.int32, device="cuda")
f = torch.empty((4096, 8192), dtype=torch.float32, device="cuda")
gam = torch.rand(4096, device="cuda") + 0.5
bet = torch.rand(8192, device="cuda") + 0.5
I11 = dict(routine="1x1", a=da, b=db, k=k, units=u)
I12 = dict(routine="1x2", w=da, t=dt, h=dh, m=dm, k=k, row_scale=gam, col_scale=bet, out=f)
I22 = dict(routine="2x2", wt=dwt, wh=dwh, wm=dwm, t=dt[:4096], h=dh[:4096], m=dm[:4096], k=k, units=u2)
flush = torch.zeros(64 << 20, device="cuda")
f2 = torch.empty((4096, 8192), dtype=torch.float32, device="cuda")
I12b = dict(I12, out=f2)
cases = {
    "b[12,12]": lambda: device.gemm_batch([I12, I12b]),
    "b[12,11]": lambda: device.gemm_batch([I12, I11]),
    "b[11]": lambda: device.gemm_batch([I11]),
    "b[11,22]": lambda: device.gemm_batch([I11, I22]),
    "b[12]": lambda: device.gemm_batch([I12]),
    "b[11,12]": lambda: device.gemm_batch([I11, I12]),
    "b[11,12,22]": lambda: device.gemm_batch([I11, I12, I22]),
    "seq 11+12+22": lambda: (device.gemm_1x1(da, db, k, units=u),
                             device.gemm_1x2(da, 1.0, dt, dh, dm, k, row_scale=gam, col_scale=bet, out=f),
                             device.gemm_2x2(dwt, dwh, dwm, dt[:4096], dh[:4096], dm[:4096], k, units=u2)),
}
for name, fn in cases.items():
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(name.ljust(14), f"median {np.median(ts):.1f} us")
device.status()
