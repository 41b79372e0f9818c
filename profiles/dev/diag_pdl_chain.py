"""Dev diagnostic: bisect PDL chains of the integer GEMM routines (not a pytest module)."""
import faulthandler, sys
faulthandler.dump_traceback_later(50, exit=True)
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2306_08960_b200 import data, device
rng = np.random.default_rng(0)
T = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()
k = 4096
a, _ = data.random_words(rng, 4096, k); b, _ = data.random_words(rng, 4096, k)
t, h, m, _ = data.random_planes(rng, 8192, k)
wt, wh, wm, _ = data.random_planes(rng, 4096, k)
da, db, dt, dh, dm, dwt, dwh, dwm = map(T, (a, b, t, h, m, wt, wh, wm))
u = torch.empty((4096, 4096), dtype=torch.int32, device="cuda")
f = torch.empty((4096, 8192), dtype=torch.float32, device="cuda")
g = torch.rand(4096, device="cuda"); be = torch.rand(8192, device="cuda")
flush = torch.zeros(64 << 20, device="cuda")
def r11(): device.gemm_1x1(da, db, k, units=u)
def r12(): device.gemm_1x2(da, 1.0, dt, dh, dm, k, row_scale=g, col_scale=be, out=f)
def r22(): device.gemm_2x2(dwt, dwh, dwm, dt[:4096], dh[:4096], dm[:4096], k, units=u)
for name, seq in [("12x3", [r12]*3), ("22x3", [r22]*3), ("11,12", [r11, r12]), ("12,22", [r12, r22]),
                  ("22,11", [r22, r11]), ("all", [r11, r12, r22]), ("all x3", [r11, r12, r22]*3),
                  ("flush+all x3", [lambda: flush.sum(), r11, r12, r22]*3)]:
    for fn in seq: fn()
    torch.cuda.synchronize(); print(name, "ok", flush=True)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for reps, use_ev, use_flush in [(200, False, False), (200, False, True), (200, True, True), (200, True, False)]:
    for i in range(reps):
        if use_flush: flush.sum()
        if use_ev: ev[0].record()
        r11(); r12(); r22()
        if use_ev: ev[1].record()
    torch.cuda.synchronize(); print("long", reps, "events", use_ev, "flush", use_flush, "ok", flush=True)
