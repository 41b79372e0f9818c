"""Host time to enqueue the bench step (bitmm_gemm_batch_dev through device.gemm_batch, and
through a prebuilt ctypes item array) against the device time of the step: when the host needs
longer than the GPU takes for the L2 flush plus the step, the step's events include host latency.
python profiles/dev/host_enqueue.py"""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2306_08960_b200 import _lib, device  # noqa: E402

lib = _lib.load()
ops = bench.make_operands(np.random.default_rng(bench.SEED))
T = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()  # noqa: E731
d = {}
for name, m, n, k in bench.ROUTINES:
    o = ops[name]
    d[name] = {kk: (T(v) if v.dtype == np.uint64 else torch.from_numpy(v).cuda()) for kk, v in o.items()}
    d[name]["units"] = torch.empty((m, n), dtype=torch.int32, device="cuda")
    d[name]["out"] = torch.empty((m, n), dtype=torch.float32, device="cuda")
items = []
for name, m, n, k in bench.ROUTINES:
    x = d[name]
    if name == "1x1":
        items.append(dict(routine="1x1", a=x["a"], b=x["b"], k=k, units=x["units"]))
    elif name == "1x2":
        items.append(dict(routine="1x2", w=x["w"], t=x["t"], h=x["h"], m=x["m"], k=k, row_scale=x["gamma"],
                          col_scale=x["beta"], out=x["out"]))
    else:
        items.append(dict(routine="2x2", wt=x["wt"], wh=x["wh"], wm=x["wm"], t=x["at"], h=x["ah"], m=x["am"], k=k,
                          units=x["units"]))
flush = torch.zeros(bench.L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
for _ in range(20):
    device.gemm_batch(items)
torch.cuda.synchronize()
for label, fn in (("device.gemm_batch", lambda: device.gemm_batch(items)),):
    n = 200
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{label}: host enqueue {1e6 * (t1 - t0) / n:.1f} us/step, device {1e6 * (t2 - t0) / n:.1f} us/step (wall, back to back)")
    t0 = time.perf_counter()
    for _ in range(n):
        flush.sum()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"flush.sum(): host {1e6 * (t1 - t0) / n:.1f} us, wall {1e6 * (time.perf_counter() - t0) / n:.1f} us")
