"""Per-kernel breakdown of the fp32 APB layer (BASELINE config 4) via the library's event
profiler (events between kernels serialise PDL, so the sum exceeds the chained time)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2306_08960_b200 import _lib, api, data, device  # noqa: E402

rng = np.random.default_rng(7)
rows, cols, tokens = 3072, 768, 8192
a, alpha, _ = data.apb_weights(rng, rows, cols)
layer = api.decompose_apb(a, alpha)
x = rng.standard_normal((cols, tokens)).astype(np.float32)
r = layer.residual
T = lambda v: torch.from_numpy(np.ascontiguousarray(v)).cuda()  # noqa: E731
I = lambda v: T(v.view(np.int64))  # noqa: E731
out = torch.empty((rows, tokens), device="cuda")
args = (I(layer.bin.words), cols, T(alpha), I(r.row_ptr), I(r.col_idx), T(r.vals), T(x), out)
lib = _lib.load()
for _ in range(3):
    device.layer_forward(*args)
torch.cuda.synchronize()
lib.bitmm_profile_reset()
lib.bitmm_profile_enable(1)
for _ in range(20):
    device.layer_forward(*args)
torch.cuda.synchronize()
lib.bitmm_profile_collect()
for i in range(lib.bitmm_profile_kernel_count()):
    n = lib.bitmm_profile_kernel_launches(i)
    print(f"{lib.bitmm_profile_kernel_name(i).decode():24s} {n:4d} launches  {lib.bitmm_profile_kernel_ms(i) / n * 1e3:8.1f} us/launch")
lib.bitmm_profile_enable(0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    device.layer_forward(*args)
e1.record()
torch.cuda.synchronize()
print(f"chained: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us/layer")
