"""1/1 4096^3 through bitmm_gemm_1x1_dev: per-call time back to back (PDL chains each call's
expansion after the previous GEMM) and the library's per-kernel event times.
python profiles/dev/time_1x1.py [M N K]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2306_08960_b200 import _lib, data  # noqa: E402

lib = _lib.load()
m, n, k = (int(v) for v in sys.argv[1:4]) if len(sys.argv) >= 4 else (4096, 4096, 4096)
rng = np.random.default_rng(1)
a, wpr = data.random_words(rng, m, k)
b, _ = data.random_words(rng, n, k)
da = torch.from_numpy(a.view(np.int64)).cuda()
db = torch.from_numpy(b.view(np.int64)).cuda()
u = torch.empty((m, n), dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream


def call():
    assert lib.bitmm_gemm_1x1_dev(da.data_ptr(), m, db.data_ptr(), n, k, wpr, 1.0, 1.0, u.data_ptr(), None, n,
                                  s) == 0


for _ in range(5):
    call()
torch.cuda.synchronize()
reps = 50
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    call()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"1x1 {m}x{n}x{k}: {ms * 1e3:.1f} us/call back to back = {2 * m * n * k / ms / 1e9:.0f} TFLOP/s "
      f"({2 * m * n * k / ms / 1e9 / 9000:.3f} of 9000)")
lib.bitmm_profile_reset()
lib.bitmm_profile_enable(1)
for _ in range(reps):
    call()
lib.bitmm_profile_collect()
lib.bitmm_profile_enable(0)
for i in range(lib.bitmm_profile_kernel_count()):
    nl = lib.bitmm_profile_kernel_launches(i)
    if nl:
        kms = lib.bitmm_profile_kernel_ms(i) / nl
        print(f"  {lib.bitmm_profile_kernel_name(i).decode()}: {kms * 1e3:.1f} us per launch")
lib.bitmm_profile_reset()
