"""GPU packers vs the oracle and the reference's golden packing
vectors: pack_signs (tensor.cpp:155-164) and quantize_uniform_2bit + decompose_thm
(transform.cpp:21-36, 47-75), bit-exact including zero padding and the ties of lround."""
import ctypes as C

import numpy as np
import pytest

from paper_2306_08960_b200 import _lib, api, data

pytestmark = pytest.mark.gpu


def _p(x):
    return x.ctypes.data_as(C.c_void_p)


def _gpu_pack(a, lane):
    rows, cols = a.shape
    wpr = data.padded_words(cols, lane)
    out = np.full((rows, wpr), 0xDEADBEEF, np.uint64)  # padding must be overwritten with zeros
    rc = _lib.load().bitmm_pack_signs_host(_p(a), rows, cols, cols, _p(out), wpr)
    assert rc == 0, _lib.last_error()
    return out, wpr


def _gpu_quant(a, s, lane):
    rows, cols = a.shape
    wpr = data.padded_words(cols, lane)
    t, h, m = (np.full((rows, wpr), 0xDEADBEEF, np.uint64) for _ in range(3))
    rc = _lib.load().bitmm_quantize_thm_host(_p(a), rows, cols, cols, s, _p(t), _p(h), _p(m), wpr)
    assert rc == 0, _lib.last_error()
    return t, h, m


def test_packing_golden(packing_golden):
    g = packing_golden
    for i in range(int(g["pack_count"])):
        p = f"p{i:03d}_"
        rows, cols, lane, wpr = (int(x) for x in g[p + "shape"])
        words, w2 = _gpu_pack(np.ascontiguousarray(g[p + "a"]), lane)
        assert w2 == wpr and np.array_equal(words, g[p + "signs"])
        t, h, m = _gpu_quant(np.ascontiguousarray(g[p + "x"]), 0.5, lane)
        assert np.array_equal(t, g[p + "t"]) and np.array_equal(h, g[p + "h"])
        assert np.array_equal(m, g[p + "m"])


@pytest.mark.parametrize("rows,cols,lane", [(1, 1, 512), (3, 63, 64), (5, 65, 512), (64, 4096, 512),
                                            (37, 1000, 128), (8, 513, 512)])
def test_random_vs_oracle(orc, rows, cols, lane):
    rng = np.random.default_rng(rows * cols)
    a = rng.standard_normal((rows, cols)).astype(np.float32)
    a[0, 0] = 0.0
    a[-1, -1] = -0.0
    words, _ = _gpu_pack(a, lane)
    want, _ = orc.pack_signs(a, lane)
    assert np.array_equal(words, want)
    # levels with exact half-step ties (lround away from zero) and out-of-range values
    s = 0.25
    x = (rng.integers(-4, 20, (rows, cols)) * (s / 2)).astype(np.float32)
    t, h, m = _gpu_quant(x, s, lane)
    wt, wh, wm, _ = orc.decompose_thm(orc.quantize_2bit(x, s), lane)
    assert np.array_equal(t, wt) and np.array_equal(h, wh) and np.array_equal(m, wm)


def test_pack_then_gemm_matches_dense(orc):
    # fp32 -> GPU packing -> GPU GEMM == the oracle on the same dense data
    import torch
    from paper_2306_08960_b200 import device
    rng = np.random.default_rng(3)
    a = torch.randn(300, 777, device="cuda")
    b = torch.randn(200, 777, device="cuda")
    wa = device.pack_signs(a)
    wb = device.pack_signs(b)
    u = torch.empty((300, 200), dtype=torch.int32, device="cuda")
    device.gemm_1x1(wa, wb, 777, units=u)
    device.status()
    sa = np.where(a.cpu().numpy() >= 0, 1, -1)
    sb = np.where(b.cpu().numpy() >= 0, 1, -1)
    assert np.array_equal(u.cpu().numpy(), sa @ sb.T)
    t, h, m = device.quantize_thm(torch.rand(200, 777, device="cuda") * 2.0, 0.5)
    u2 = torch.empty_like(u)
    device.gemm_1x2(wa, 1.0, t, h, m, 777, units=u2)
    device.status()


def test_pack_argument_errors():
    lib = _lib.load()
    a = np.zeros((1, 4), np.float32)
    w = np.zeros((1, 1), np.uint64)
    assert lib.bitmm_pack_signs_host(_p(a), 1, 65, 65, _p(w), 1) == _lib.ERR_INVALID_ARGUMENT
    assert lib.bitmm_quantize_thm_host(_p(a), 1, 4, 4, 0.0, _p(w), _p(w), _p(w), 1) == _lib.ERR_INVALID_ARGUMENT
