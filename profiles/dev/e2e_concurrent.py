"""e2e step (the three host calls of bench.py) issued sequentially vs from three host threads at
once (the C ABI is re-entrant: each host call leases its own context, so the calls' copies,
GEMMs and host widening overlap). python profiles/dev/e2e_concurrent.py"""
import ctypes as C
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2306_08960_b200 import _lib  # noqa: E402

lib = _lib.load()
ops = bench.make_operands(np.random.default_rng(bench.SEED))
pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory()  # noqa: E731
P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
h = {}
for name, m, n, k in bench.ROUTINES:
    h[name] = {kk: pin(v) for kk, v in ops[name].items()}
    h[name]["out"] = torch.empty((m, n), dtype=torch.float32 if name == "1x2" else torch.int32).pin_memory()


def call(name, m, n, k):
    x = h[name]
    wpr = (k + 511) // 512 * 8
    if name == "1x1":
        rc = lib.bitmm_gemm_1x1_host(P(x["a"]), m, P(x["b"]), n, k, wpr, 1.0, 1.0, P(x["out"]), None, n)
    elif name == "1x2":
        rc = lib.bitmm_gemm_1x2_host(P(x["w"]), m, 1.0, P(x["t"]), P(x["h"]), P(x["m"]), n, k, wpr, 1.0, 0, 1.0,
                                     P(x["gamma"]), P(x["beta"]), None, P(x["out"]), n)
    else:
        rc = lib.bitmm_gemm_2x2_host(P(x["wt"]), P(x["wh"]), P(x["wm"]), m, 1.0, 0, 1.0, P(x["at"]), P(x["ah"]),
                                     P(x["am"]), n, k, wpr, 1.0, 0, 1.0, None, None, P(x["out"]), None, n)
    assert rc == 0, _lib.last_error()


def seq():
    for r in bench.ROUTINES:
        call(*r)


def par():
    ts = [threading.Thread(target=call, args=r) for r in bench.ROUTINES]
    for t in ts:
        t.start()
    for t in ts:
        t.join()


upd = sum(m * n * k for _, m, n, k in bench.ROUTINES)
for name, fn in (("sequential", seq), ("3 threads", par), ("sequential", seq), ("3 threads", par)):
    for _ in range(3):
        fn()
    t0 = time.perf_counter()
    reps = 10
    for _ in range(reps):
        fn()
    s = (time.perf_counter() - t0) / reps
    print(f"{name}: {s * 1e3:.3f} ms per step, {upd / s / 1e12:.1f} T-upd/s", flush=True)
