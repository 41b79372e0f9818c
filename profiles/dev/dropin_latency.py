"""Per-call latency of the host flavour at the reference acceptance criterion-8 shape (1024^3),
called the way the drop-in does it: a fresh zero-filled output per call (DenseMatrix), host
operands in pageable memory. python profiles/dev/dropin_latency.py [label]"""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2306_08960_b200 import _lib, data  # noqa: E402

lib = _lib.load()
P = lambda x: x.ctypes.data_as(C.c_void_p)  # noqa: E731
rng = np.random.default_rng(1)
m = n = k = 1024
a, wpr = data.random_words(rng, m, k)
b, _ = data.random_words(rng, n, k)
t, h, mm, _ = data.random_planes(rng, n, k)
wt, wh, wm, _ = data.random_planes(rng, m, k)


def r11(c):
    return lib.bitmm_gemm_1x1_host(P(a), m, P(b), n, k, wpr, 1.0, 1.0, None, P(c), n)


def r12(c):
    return lib.bitmm_gemm_1x2_host(P(a), m, 1.0, P(t), P(h), P(mm), n, k, wpr, 1.0, 0, 1.0, None, None, None,
                                   P(c), n)


def r22(c):
    return lib.bitmm_gemm_2x2_host(P(wt), P(wh), P(wm), m, 1.0, 0, 1.0, P(t), P(h), P(mm), n, k, wpr, 1.0, 0,
                                   1.0, None, None, None, P(c), n)


res = []
for name, fn in (("1x1", r11), ("1x2", r12), ("2x2", r22)):
    ts = []
    for i in range(11):
        t0 = time.perf_counter()
        c = np.empty((m, n), np.float32)  # DenseMatrix(rows, cols): allocated and zero-filled
        c.fill(0.0)                        # (data_.assign(n, 0.0f), tensor.cpp:37-40) in the timed region
        assert fn(c) == 0, _lib.last_error()
        ts.append(time.perf_counter() - t0)
    res.append(f"{name} {np.median(ts[2:]) * 1e3:.3f} ms")
print(sys.argv[1] if len(sys.argv) > 1 else "", " ".join(res), flush=True)

# breakdown: reused output buffer (no first-touch), a tiny call (fixed overhead)
c0 = np.zeros((m, n), np.float32)
for name, fn in (("1x1 reused-out", r11),):
    ts = []
    for i in range(11):
        t0 = time.perf_counter()
        assert fn(c0) == 0
        ts.append(time.perf_counter() - t0)
    print(name, f"{np.median(ts[2:]) * 1e3:.3f} ms")
a64, w64 = data.random_words(rng, 64, 64)
c64 = np.zeros((64, 64), np.float32)
ts = []
for i in range(21):
    t0 = time.perf_counter()
    assert lib.bitmm_gemm_1x1_host(P(a64), 64, P(a64), 64, 64, w64, 1.0, 1.0, None, P(c64), 64) == 0
    ts.append(time.perf_counter() - t0)
print("1x1 64^3", f"{np.median(ts[2:]) * 1e3:.3f} ms")
ts = []
for i in range(11):
    t0 = time.perf_counter()
    c = np.zeros((m, n), np.float32)
    c[:] = 1.0
    ts.append(time.perf_counter() - t0)
print("np.zeros + touch 4 MB", f"{np.median(ts[2:]) * 1e3:.3f} ms")
