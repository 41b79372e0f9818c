"""Smoke-size calls of every kernel of the library, for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck). Each result is also checked against the oracle, so a clean exit means
the kernels ran and were right under the tool.

    compute-sanitizer --tool memcheck python profiles/dev/sanitize_smoke.py

Covers: unpack_operands + tc_gemm (1/1, 1/2, 2/2; per call and grouped), the in-GEMM
expansion path (BITMM_FX=1 in a child run: prep_operands + fx_gemm), popc_gemm, the host
calls with the 16-bit wire forced on (narrow_units_kernel, the spin-wait kernel), the fp32 APB
layer (apb_fold, split_x_f16_strip, apb_gemm) and gemm_1x32 (unpack_sign_f16), the 2-bit APB
layer (spmm_levels), standalone spmm, the packers (pack_signs, quantize_thm, decompose_thm,
decompose_apb count/fill + CUB scan), row ops and plane validation.
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2306_08960_b200 import _lib, api, data, device  # noqa: E402

os.environ.setdefault("BITMM_WIRE_MIN_BYTES", "0")  # host calls take the wire path
os.environ.setdefault("BITMM_WIRE_WAIT", "kernel")  # ... and the spin-wait kernel
orc = oracle.Oracle()
rng = np.random.default_rng(5)
T = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()  # noqa: E731
P = lambda x: x.ctypes.data_as(C.c_void_p)  # noqa: E731
lib = _lib.load()

m, n, k = 300, 260, 1100
a, wpr = data.random_words(rng, m, k)
b, _ = data.random_words(rng, n, k)
t, h, mm, _ = data.random_planes(rng, n, k)
wt, wh, wm, _ = data.random_planes(rng, m, k)
u = torch.empty((m, n), dtype=torch.int32, device="cuda")
f = torch.empty((m, n), dtype=torch.float32, device="cuda")
device.gemm_1x1(T(a), T(b), k, 0.5, 2.0, units=u, out=f)
device.status()
assert np.array_equal(u.cpu().numpy(), orc.gemm_1x1(a, b, k, wpr)[0])
device.gemm_1x1(T(a), T(b), k, units=u, popc=True)
device.status()
assert np.array_equal(u.cpu().numpy(), orc.gemm_1x1(a, b, k, wpr)[0])
rs = torch.rand(m, device="cuda") + 0.5
cs = torch.rand(n, device="cuda") + 0.5
device.gemm_1x2(T(a), 1.0, T(t), T(h), T(mm), k, row_scale=rs, col_scale=cs, units=u, out=f)
device.status()
assert np.array_equal(u.cpu().numpy(), orc.gemm_1x2(a, 1.0, t, h, mm, k, wpr)[0])
device.gemm_2x2(T(wt), T(wh), T(wm), T(t), T(h), T(mm), k, units=u)
device.status()
assert np.array_equal(u.cpu().numpy(), orc.gemm_2x2(wt, wh, wm, t, h, mm, k, wpr)[0])
g = [torch.empty_like(u) for _ in range(3)]
device.gemm_batch([dict(routine="1x1", a=T(a), b=T(b), k=k, units=g[0]),
                   dict(routine="1x2", w=T(a), t=T(t), h=T(h), m=T(mm), k=k, units=g[1]),
                   dict(routine="2x2", wt=T(wt), wh=T(wh), wm=T(wm), t=T(t), h=T(h), m=T(mm), k=k, units=g[2])])
device.status()
assert np.array_equal(g[2].cpu().numpy(), orc.gemm_2x2(wt, wh, wm, t, h, mm, k, wpr)[0])

# host calls on the 16-bit wire (narrowing kernel, spin-wait kernel, pipelined copies)
uh = np.empty((m, n), np.int32)
assert lib.bitmm_gemm_1x1_host(P(a), m, P(b), n, k, wpr, 1.0, 1.0, P(uh), None, n) == 0, _lib.last_error()
assert np.array_equal(uh, orc.gemm_1x1(a, b, k, wpr)[0])
assert lib.bitmm_gemm_1x2_host(P(a), m, 1.0, P(t), P(h), P(mm), n, k, wpr, 1.0, 0, 1.0, None, None, P(uh),
                               None, n) == 0
assert np.array_equal(uh, orc.gemm_1x2(a, 1.0, t, h, mm, k, wpr)[0])

# late-output host call (the drop-in's path): staged copy through pinned memory
it = _lib.GemmItem()
it.routine, it.a0, it.b0, it.m, it.n, it.k, it.wpr, it.a_scale, it.b_scale = 0, a.ctypes.data, b.ctypes.data, m, n, k, wpr, 1.0, 1.0
late = {}


def _out(user, o):
    late["u"] = np.empty((m, n), np.int32)
    o.contents.c_units = late["u"].ctypes.data
    o.contents.ldc = n
    return 0


cb = _lib.OUT_FN(_out)
assert lib.bitmm_gemm_host_late(C.byref(it), _lib.WANT_UNITS, cb, None) == 0, _lib.last_error()
assert np.array_equal(late["u"], orc.gemm_1x1(a, b, k, wpr)[0])

# APB (fp32 activations): folded residual, and the plain 1x32 GEMM
rows, cols, tokens = 192, 768, 160
w, alpha, _ = data.apb_weights(rng, rows, cols)
layer = api.decompose_apb(w, alpha)
x = rng.standard_normal((cols, tokens)).astype(np.float32)
got = api.layer_forward(layer, x)
r = layer.residual
want = orc.layer_forward(rows, cols, 1.0, layer.bin.words, layer.bin.words_per_row(), r.row_ptr, r.col_idx,
                         r.vals, x, row_alpha=alpha)
assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-5
y = torch.empty((rows, tokens), dtype=torch.float32, device="cuda")
device.gemm_1x32(T(layer.bin.words), cols, 0.5, torch.from_numpy(x).cuda(), y)
device.status()
# APB with 2-bit activations (GEMM + exact residual SpMM)
t2, h2, m2, wpr2 = data.random_planes(rng, tokens, cols)
y2 = torch.empty((rows, tokens), dtype=torch.float32, device="cuda")
Tf = lambda v: torch.from_numpy(np.ascontiguousarray(v)).cuda()  # noqa: E731
device.layer_forward_2bit(T(layer.bin.words), cols, Tf(alpha), T(r.row_ptr), T(r.col_idx), Tf(r.vals), T(t2),
                          T(h2), T(m2), y2, a_scale=0.5)
device.status()
want2 = orc.layer_forward_2bit(rows, cols, 1.0, layer.bin.words, wpr2, r.row_ptr, r.col_idx, r.vals, t2, h2, m2,
                               a_scale=0.5, row_alpha=alpha)
assert np.array_equal(y2.cpu().numpy(), want2)
# standalone SpMM
ys = torch.empty((rows, tokens), dtype=torch.float32, device="cuda")
device.spmm_csr(rows, cols, T(r.row_ptr), T(r.col_idx), Tf(r.vals), torch.from_numpy(x).cuda(), ys)
device.status()

# packers, row ops, plane validation
dense = torch.from_numpy(rng.standard_normal((70, 300)).astype(np.float32)).cuda()
words = device.pack_signs(dense)
device.quantize_thm(dense, 0.5)
lv = torch.from_numpy(rng.integers(0, 4, (70, 300), dtype=np.uint8)).cuda()
tp, hp, mp = device.decompose_thm(lv)
device.decompose_apb(dense, 0.7)
device.dot_binary_rows(words, words, 300)
device.mbm_rows(words, words, words)
assert lib.bitmm_validate_planes_dev(tp.data_ptr(), hp.data_ptr(), mp.data_ptr(), 70, 300, tp.shape[1], 1.0,
                                     None) == 0, _lib.last_error()
torch.cuda.synchronize()
print("sanitize smoke ok")
