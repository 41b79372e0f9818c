"""1/1 4096^3 through both GEMM paths for one ncu capture: the LOP3+POPC CUDA-core kernel
(bitmm_gemm_1x1_popc_dev) and the tcgen05 path (expansion + tc_gemm). Not a benchmark."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2306_08960_b200 import data, device  # noqa: E402

rng = np.random.default_rng(1)
k = 4096
a, _ = data.random_words(rng, 4096, k)
b, _ = data.random_words(rng, 4096, k)
T = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()  # noqa: E731
da, db = T(a), T(b)
u1 = torch.empty((4096, 4096), dtype=torch.int32, device="cuda")
u2 = torch.empty_like(u1)
for _ in range(2):
    device.gemm_1x1(da, db, k, units=u1, popc=True)
    device.gemm_1x1(da, db, k, units=u2)
torch.cuda.synchronize()
device.status()
assert torch.equal(u1, u2)
print("popc and tensor paths agree")
