"""A/B timing of two builds of the library on the same box: python profiles/ab_lib.py PATH.so"""
import ctypes as C
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2306_08960_b200 import data, _lib

path = sys.argv[1]
lib = C.CDLL(path)
for name, (res, args) in _lib.SIGNATURES.items():
    if hasattr(lib, name):
        fn = getattr(lib, name); fn.restype = res; fn.argtypes = args
rng = np.random.default_rng(1)
k = 4096
T = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()  # noqa: E731
a, wpr = data.random_words(rng, 4096, k)
b, _ = data.random_words(rng, 4096, k)
t, h, m, _ = data.random_planes(rng, 8192, k)
wt, wh, wm, _ = data.random_planes(rng, 4096, k)
da, db, dt, dh, dm, dwt, dwh, dwm = map(T, (a, b, t, h, m, wt, wh, wm))
u = torch.empty((4096, 4096), dtype=torch.int32, device="cuda")
f = torch.empty((4096, 8192), dtype=torch.float32, device="cuda")
gam = torch.rand(4096, device="cuda") + 0.5
bet = torch.rand(8192, device="cuda") + 0.5
s = torch.cuda.current_stream().cuda_stream
P = lambda x: x.data_ptr()  # noqa: E731
flush = torch.zeros(64 << 20, device="cuda")
def r11(): lib.bitmm_gemm_1x1_dev(P(da), 4096, P(db), 4096, k, wpr, 1.0, 1.0, P(u), None, 4096, s)
def r12(): lib.bitmm_gemm_1x2_dev(P(da), 4096, 1.0, P(dt), P(dh), P(dm), 8192, k, wpr, 1.0, 0, 1.0, P(gam), P(bet), None, P(f), 8192, s)
def r22(): lib.bitmm_gemm_2x2_dev(P(dwt), P(dwh), P(dwm), 4096, 1.0, 0, 1.0, P(dt[:4096]), P(dh[:4096]), P(dm[:4096]), 4096, k, wpr, 1.0, 0, 1.0, None, None, P(u), None, 4096, s)
for name, fn in (("1x1", r11), ("1x2", r12), ("2x2", r22), ("step", lambda: (r11(), r12(), r22()))):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(15):
        flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(path.split('/')[-1], name, f"median {np.median(ts):.1f} us  min {min(ts):.1f}")
