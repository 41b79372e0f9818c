"""12-bit packing of the host output wire (csrc/wire.cuh, wire12_*; wire_host.cpp unpack12;
BITMM_WIRE_BITS=12, measured and not the default): outputs whose blocks have a multiple of 16 columns cross PCIe as {min, max} headers plus 12-bit
fields per part; a part whose words span more than 4095 values is fetched again as 16-bit
words. Every result must equal the device path bit for bit, whatever the data."""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_2306_08960_b200 import _lib, data, device

pytestmark = pytest.mark.gpu
lib = _lib.load()


def _p(x):
    return C.c_void_p(x.ctypes.data) if x is not None else None


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()


def _full_row(k, wpr):
    full = np.zeros(wpr, np.uint64)
    full[: k // 64] = ~np.uint64(0)
    if k % 64:
        full[k // 64] = np.uint64((1 << (k % 64)) - 1)
    return full


@pytest.fixture(autouse=True, params=["avx", "sse2"])
def simd(request, monkeypatch):
    monkeypatch.setenv("BITMM_WIRE_BITS", "12")
    monkeypatch.delenv("BITMM_HOST_WIRE", raising=False)
    if request.param == "sse2":
        monkeypatch.setenv("BITMM_HOST_SIMD", "sse2")
    else:
        monkeypatch.delenv("BITMM_HOST_SIMD", raising=False)
    return request.param


@pytest.mark.parametrize("k,extreme", [(1000, False), (4096, False), (5000, True)])
def test_1x1_wire12(k, extreme):
    rng = np.random.default_rng(k)
    m, n = 2304, 4096  # 37.7 MB per output: row slices on the 16-bit wire, 12-bit packed
    a, wpr = data.random_words(rng, m, k)
    b, _ = data.random_words(rng, n, k)
    if extreme:  # row 0: popcount 0 at column 0 and K at column 1 -> the part spans K > 4095
        b[0] = a[0]
        b[1] = a[0] ^ _full_row(k, wpr)
    units = np.empty((m, n), np.int32)
    vals = np.empty((m, n), np.float32)
    assert lib.bitmm_gemm_1x1_host(_p(a), m, _p(b), n, k, wpr, 0.75, 1.25, _p(units), _p(vals), n) == 0
    want = torch.empty((m, n), dtype=torch.int32, device="cuda")
    device.gemm_1x1(_dev(a), _dev(b), k, units=want)
    assert np.array_equal(units, want.cpu().numpy())
    assert np.array_equal(vals, np.float32(0.75 * 1.25) * units.astype(np.float32))
    if extreme:
        assert units[0, 0] == k and units[0, 1] == -k
    got = lib.bitmm_last_d2h_bytes()
    assert m * n * 1.5 <= got < m * n * (2.0 if not extreme else 2.5), got


@pytest.mark.parametrize("k,extreme", [(777, False), (10922, True)])
def test_1x2_wire12(k, extreme):
    rng = np.random.default_rng(k)
    m, n = 1024, 8192  # column slices of 1024 activation rows
    w, wpr = data.random_words(rng, m, k)
    t, h, mm, _ = data.random_planes(rng, n, k)
    if extreme:
        full = _full_row(k, wpr)
        w[0] = full
        t[0], h[0], mm[0] = full, 0, full  # units[0, 0] = 6K
    rs = rng.uniform(0.5, 1.5, m).astype(np.float32)
    cs = rng.uniform(0.5, 1.5, n).astype(np.float32)
    units = np.empty((m, n), np.int32)
    vals = np.empty((m, n), np.float32)
    assert lib.bitmm_gemm_1x2_host(_p(w), m, 1.5, _p(t), _p(h), _p(mm), n, k, wpr, 0.5, 1, 2.0, _p(rs), _p(cs),
                                   _p(units), _p(vals), n) == 0
    wu = torch.empty((m, n), dtype=torch.int32, device="cuda")
    wv = torch.empty((m, n), dtype=torch.float32, device="cuda")
    device.gemm_1x2(_dev(w), 1.5, _dev(t), _dev(h), _dev(mm), k, a_scale=0.5, a_gamma=2.0,
                    row_scale=torch.from_numpy(rs).cuda(), col_scale=torch.from_numpy(cs).cuda(), units=wu, out=wv)
    assert np.array_equal(units, wu.cpu().numpy())
    assert np.array_equal(vals, wv.cpu().numpy())
    if extreme:
        assert units[0, 0] == 6 * k


@pytest.mark.parametrize("k,extreme", [(700, False), (7281, True)])
def test_2x2_wire12(k, extreme):
    rng = np.random.default_rng(k)
    m, n = 4160, 2048
    wt, wh, wm, wpr = data.random_planes(rng, m, k)
    at, ah, am, _ = data.random_planes(rng, n, k)
    if extreme:
        full = _full_row(k, wpr)
        for t_, h_, m_ in ((wt, wh, wm), (at, ah, am)):
            t_[0], h_[0], m_[0] = full, 0, full  # units[0, 0] = 36K
    units = np.empty((m, n), np.int32)
    assert lib.bitmm_gemm_2x2_host(_p(wt), _p(wh), _p(wm), m, 0.25, 0, 1.0, _p(at), _p(ah), _p(am), n, k, wpr, 0.5,
                                   1, 3.0, None, None, _p(units), None, n) == 0
    wu = torch.empty((m, n), dtype=torch.int32, device="cuda")
    device.gemm_2x2(*[_dev(x) for x in (wt, wh, wm, at, ah, am)], k, w_scale=0.25, a_scale=0.5, a_gamma=3.0, units=wu)
    assert np.array_equal(units, wu.cpu().numpy())
    if extreme:
        assert units[0, 0] == 36 * k


def test_wire12_off_matches():
    """BITMM_WIRE_BITS=16 (16-bit words, the default) and the 12-bit packing give the same bits."""
    import os
    rng = np.random.default_rng(3)
    m, n, k = 2304, 4096, 1500
    a, wpr = data.random_words(rng, m, k)
    b, _ = data.random_words(rng, n, k)
    outs = []
    for bits in ("12", "16"):
        os.environ["BITMM_WIRE_BITS"] = bits
        u = np.empty((m, n), np.int32)
        assert lib.bitmm_gemm_1x1_host(_p(a), m, _p(b), n, k, wpr, 1.0, 1.0, _p(u), None, n) == 0
        outs.append((u, lib.bitmm_last_d2h_bytes()))
    os.environ["BITMM_WIRE_BITS"] = "12"
    assert np.array_equal(outs[0][0], outs[1][0])
    assert outs[0][1] < outs[1][1] == m * n * 2
