"""The in-GEMM expansion paths (fx_gemm.cuh, BITMM_FX=1 and the hybrid BITMM_FX=2): bit-exact
against the oracle.

It is a selectable alternative to the default expansion pass, so it is exercised in a child
process with the variable set (the library reads it once): random shapes with off-grid K and
lane widths 64/512 (odd words_per_row falls back to the default path), ragged tiles, the
grouped launch, level-plane validation and padding errors.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import numpy as np, torch, oracle
from paper_2306_08960_b200 import api, data, device
orc = oracle.Oracle()
rng = np.random.default_rng(5)
T = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()
shapes = [(int(rng.integers(1, 600)), int(rng.integers(1, 3000)), int(rng.integers(1, 600))) for _ in range(24)]
shapes += [(256, 4096, 192), (300, 513, 257), (513, 1024, 385), (64, 100000, 70)]
for lane in (512, 128):
    for (m, k, n) in shapes:
        a, wpr = data.random_words(rng, m, k, lane)
        b, _ = data.random_words(rng, n, k, lane)
        t, h, mm, _ = data.random_planes(rng, n, k, lane)
        wt, wh, wm, _ = data.random_planes(rng, m, k, lane)
        u = torch.empty((m, n), dtype=torch.int32, device="cuda")
        f = torch.empty((m, n), dtype=torch.float32, device="cuda")
        device.gemm_1x1(T(a), T(b), k, 0.5, 1.5, units=u, out=f)
        wu, wf = orc.gemm_1x1(a, b, k, wpr, 0.5, 1.5)
        assert np.array_equal(u.cpu().numpy(), wu) and np.array_equal(f.cpu().numpy(), wf), ("1x1", m, k, n, lane)
        rs = rng.uniform(0.5, 1.5, m).astype(np.float32); cs = rng.uniform(0.5, 1.5, n).astype(np.float32)
        device.gemm_1x2(T(a), 1.25, T(t), T(h), T(mm), k, 0.5, 0.75, row_scale=torch.from_numpy(rs).cuda(),
                        col_scale=torch.from_numpy(cs).cuda(), units=u, out=f)
        wu, wf = orc.gemm_1x2(a, 1.25, t, h, mm, k, wpr, 0.5, 0.75, rs, cs)
        assert np.array_equal(u.cpu().numpy(), wu) and np.array_equal(f.cpu().numpy(), wf), ("1x2", m, k, n, lane)
        device.gemm_2x2(T(wt), T(wh), T(wm), T(t), T(h), T(mm), k, units=u)
        assert np.array_equal(u.cpu().numpy(), orc.gemm_2x2(wt, wh, wm, t, h, mm, k, wpr)[0]), ("2x2", m, k, n, lane)
        device.status()
# grouped launch
m = n = 640; k = 2000
a, wpr = data.random_words(rng, m, k); b, _ = data.random_words(rng, n, k)
t, h, mm, _ = data.random_planes(rng, n, k); wt, wh, wm, _ = data.random_planes(rng, m, k)
g = [torch.empty((m, n), dtype=torch.int32, device="cuda") for _ in range(3)]
device.gemm_batch([dict(routine="1x1", a=T(a), b=T(b), k=k, units=g[0]),
                   dict(routine="1x2", w=T(a), t=T(t), h=T(h), m=T(mm), k=k, units=g[1]),
                   dict(routine="2x2", wt=T(wt), wh=T(wh), wm=T(wm), t=T(t), h=T(h), m=T(mm), k=k, units=g[2])])
device.status()
assert np.array_equal(g[0].cpu().numpy(), orc.gemm_1x1(a, b, k, wpr)[0])
assert np.array_equal(g[1].cpu().numpy(), orc.gemm_1x2(a, 1.0, t, h, mm, k, wpr)[0])
assert np.array_equal(g[2].cpu().numpy(), orc.gemm_2x2(wt, wh, wm, t, h, mm, k, wpr)[0])
# errors: an illegal plane triple, nonzero padding past K
bad_t = t.copy(); bad_t[3, 0] |= np.uint64(1); bad_h = h.copy(); bad_h[3, 0] |= np.uint64(1)
u = torch.empty((m, n), dtype=torch.int32, device="cuda")
device.gemm_1x2(T(a), 1.0, T(bad_t), T(bad_h), T(mm), k, units=u)
try:
    device.status(); raise SystemExit("illegal planes not reported")
except api.InvalidEncoding:
    pass
a2, wpr2 = data.random_words(rng, 64, 700); a2[5, -1] |= np.uint64(1) << np.uint64(63)
b2, _ = data.random_words(rng, 64, 700)
device.gemm_1x1(T(a2), T(b2), 700, units=u[:64, :64].contiguous())
try:
    device.status(); raise SystemExit("padding not reported")
except ValueError:
    pass
print("fx ok")
'''


@pytest.mark.parametrize("mode", ["1", "2"])
def test_fx_path_bit_exact(mode):
    """mode 1: both operands expanded in the GEMM; 2 (hybrid): A by unpack_operands, B in the GEMM."""
    env = dict(os.environ, BITMM_FX=mode)
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=REPO, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "fx ok" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
