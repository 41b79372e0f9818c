"""Per-SM throughput of the 1/1 GEMM vs grid size (BITMM_AB_UNITS caps the CTA pairs)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2306_08960_b200 import data, device
rng = np.random.default_rng(1)
k = 4096
T = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()  # noqa: E731
m = n = 8192
a, wpr = data.random_words(rng, m, k)
b, _ = data.random_words(rng, n, k)
da, db = T(a), T(b)
u = torch.empty((m, n), dtype=torch.int32, device="cuda")
for _ in range(3): device.gemm_1x1(da, db, k, units=u)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); device.gemm_1x1(da, db, k, units=u); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
print(f"units={sys.argv[1]} 1x1 8192x8192x4096: {np.median(ts):.1f} us  {m*n*k/np.median(ts)/1e6:.0f} T-upd/s")
