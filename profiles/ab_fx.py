"""A/B timing of library builds of the in-GEMM expansion path (fx_gemm) on one box.

    python profiles/ab_fx.py build/ab/a.so build/ab/b.so ...

Per build: median of 15 L2-flushed launches of 1/1, 1/2 (row/col scales, fp32 out), 2/2 at
4096^3 (1/2: 8192 activation columns), and, for builds compiled with -DFX_STATS, the
fx_gemm wait counters of one 1/1 launch (cycles per CTA, averaged over CTAs).
"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2306_08960_b200 import _lib, data  # noqa: E402

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

for path in sys.argv[1:]:
    lib = C.CDLL(path)
    for name, (res, args) in _lib.SIGNATURES.items():
        if hasattr(lib, name):
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args

    def chk(rc):
        if rc != 0:
            raise RuntimeError(lib.bitmm_last_error().decode())

    def r11():
        chk(lib.bitmm_gemm_1x1_dev(P(da), 4096, P(db), 4096, k, wpr, 1.0, 1.0, P(u), None, 4096, s))

    def r12():
        chk(lib.bitmm_gemm_1x2_dev(P(da), 4096, 1.0, P(dt), P(dh), P(dm), 8192, k, wpr, 1.0, 0, 1.0, P(gam),
                                   P(bet), None, P(f), 8192, s))

    def r22():
        chk(lib.bitmm_gemm_2x2_dev(P(dwt), P(dwh), P(dwm), 4096, 1.0, 0, 1.0, P(dt[:4096]), P(dh[:4096]),
                                   P(dm[:4096]), 4096, k, wpr, 1.0, 0, 1.0, None, None, P(u), None, 4096, s))

    res = []
    for name, fn in (("1x1", r11), ("1x2", r12), ("2x2", r22)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(15):
            flush.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        res.append(f"{name} {np.median(ts):.1f}us")
    print(path.split("/")[-1], " ".join(res), flush=True)
    if hasattr(lib, "bitmm_debug_fx_stats"):
        lib.bitmm_debug_fx_stats.restype = C.c_int
        buf = (C.c_ulonglong * (8 * 160))()
        r11()
        torch.cuda.synchronize()
        lib.bitmm_debug_fx_stats(buf)
        st = np.frombuffer(buf, dtype=np.uint64).reshape(8, 160).astype(np.float64)
        nz = st[1] > 0
        names = ["mma_wait_full", "mma_total", "exp_wait_pfull", "exp_wait_empty", "exp_total", "prod_wait_pempty"]
        print("   1x1 stats (cycles, mean over CTAs):",
              {n: int(st[i][nz].mean() if i in (0, 1) else st[i][st[4] > 0].mean()) for i, n in enumerate(names)},
              flush=True)
