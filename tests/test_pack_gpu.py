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


@pytest.mark.parametrize("rows,cols,lane", [(1, 1, 512), (37, 100, 64), (300, 777, 512), (64, 4096, 512)])
def test_decompose_thm_vs_oracle(orc, rows, cols, lane):
    """decompose_thm (transform.cpp:47-75) on 2-bit levels: GPU planes equal the oracle's,
    padding zero, for both flavours."""
    import torch
    from paper_2306_08960_b200 import device
    rng = np.random.default_rng(rows * cols + lane)
    lv = rng.integers(0, 4, size=(rows, cols), dtype=np.uint8)
    t, h, m, wpr = orc.decompose_thm(lv, lane)
    gt, gh, gm = device.decompose_thm(torch.from_numpy(lv).cuda(), lane)
    device.status()
    for g, w in ((gt, t), (gh, h), (gm, m)):
        assert np.array_equal(g.cpu().numpy().view(np.uint64), w)
    ht, hh, hm = (np.zeros((rows, wpr), np.uint64) for _ in range(3))
    rc = _lib.load().bitmm_decompose_thm_host(lv.ctypes.data, rows, cols, ht.ctypes.data,
                                              hh.ctypes.data, hm.ctypes.data, wpr)
    assert rc == 0
    assert np.array_equal(ht, t) and np.array_equal(hh, h) and np.array_equal(hm, m)


def test_decompose_thm_level_out_of_range():
    import torch
    from paper_2306_08960_b200 import device
    lv = np.zeros((3, 70), np.uint8)
    lv[2, 69] = 4
    device.decompose_thm(torch.from_numpy(lv).cuda())
    with pytest.raises(ValueError, match="2-bit level out of range"):
        device.status()
    rc = _lib.load().bitmm_decompose_thm_host(lv.ctypes.data, 3, 70, *(np.zeros(24, np.uint64).ctypes.data
                                                                        for _ in range(3)), 8)
    assert rc == _lib.ERR_INVALID_ARGUMENT


def _apb_matrix(rng, rows, cols, alpha):
    """N(0, 0.02) weights with exact +-alpha entries, signed zeros, and differences that sit
    exactly halfway between two floats (ties-away and ties-to-even disagree on them)."""
    a = rng.normal(0.0, 0.02, (rows, cols)).astype(np.float32)
    al = np.broadcast_to(np.asarray(alpha, np.float32).reshape(-1, 1), (rows, 1))
    pick = rng.random((rows, cols))
    a = np.where(pick < 0.4, np.where(a >= 0, al, -al), a).astype(np.float32)
    a[pick > 0.98] = 0.0
    a[(pick > 0.96) & (pick <= 0.98)] = -0.0
    if cols > 3:
        a[:, 1] = np.float32(2.0 ** 24 + 2)   # with alpha = 1: diff 2^24 + 1, a tie
        a[:, 2] = -np.float32(2.0 ** 24 + 2)
        a[:, 3] = np.float32(3 * 2.0 ** 23 + 2)
    return a


@pytest.mark.parametrize("rows,cols,per_row", [(1, 1, False), (17, 300, False), (64, 768, True),
                                               (200, 1000, True), (5, 4096, False)])
def test_decompose_apb_vs_oracle(orc, rows, cols, per_row):
    """decompose_apb (apb.cpp:119-142): GPU sign words, CSR and residual values equal the
    oracle's bit for bit (values compared as bit patterns), scalar or per-row alpha."""
    import torch
    from paper_2306_08960_b200 import device
    rng = np.random.default_rng(rows + cols)
    alpha = (rng.uniform(0.5, 1.5, rows).astype(np.float32) if per_row else np.float32(1.0))
    if per_row:
        alpha[0] = 1.0
    a = _apb_matrix(rng, rows, cols, alpha)
    bw, wpr, rp, ci, v = orc.decompose_apb(a, alpha)
    al_arg = torch.from_numpy(alpha).cuda() if per_row else float(alpha)
    gb, grp, gci, gv = device.decompose_apb(torch.from_numpy(a).cuda(), al_arg)
    assert np.array_equal(gb.cpu().numpy().view(np.uint64), bw)
    assert np.array_equal(grp.cpu().numpy().view(np.uint64), rp)
    assert np.array_equal(gci.cpu().numpy().view(np.uint64), ci)
    assert np.array_equal(gv.cpu().numpy().view(np.uint32), v.view(np.uint32))
    # the host flavour, through the two-call protocol
    lib = _lib.load()
    nnz = C.c_int64(0)
    hb = np.zeros((rows, wpr), np.uint64)
    hrp = np.zeros(rows + 1, np.uint64)
    al_p = alpha.ctypes.data if per_row else None
    sc = 1.0 if per_row else float(alpha)
    assert lib.bitmm_decompose_apb_host(a.ctypes.data, rows, cols, cols, sc, al_p, hb.ctypes.data, wpr,
                                        hrp.ctypes.data, None, None, 0, C.byref(nnz)) == 0
    hci = np.zeros(max(nnz.value, 1), np.uint64)
    hv = np.zeros(max(nnz.value, 1), np.float32)
    assert lib.bitmm_decompose_apb_host(a.ctypes.data, rows, cols, cols, sc, al_p, hb.ctypes.data, wpr,
                                        hrp.ctypes.data, hci.ctypes.data, hv.ctypes.data, hci.size,
                                        C.byref(nnz)) == 0
    assert nnz.value == ci.size
    assert np.array_equal(hb, bw) and np.array_equal(hrp, rp)
    assert np.array_equal(hci[:nnz.value], ci) and np.array_equal(hv[:nnz.value].view(np.uint32),
                                                                  v.view(np.uint32))


def test_decompose_apb_alpha_must_be_positive():
    import torch
    from paper_2306_08960_b200 import device
    a = torch.ones((4, 10), device="cuda")
    with pytest.raises(ValueError, match="alpha must be positive"):
        device.decompose_apb(a, 0.0)
    with pytest.raises(ValueError, match="alpha must be positive"):
        device.decompose_apb(a, torch.tensor([1.0, 1.0, -2.0, 1.0], device="cuda"))
