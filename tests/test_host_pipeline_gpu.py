"""The host-flavour entry points (`bitmm_gemm_*_host`) produce outputs of 32 MB and more in
slices: each slice's inputs are copied in and its GEMM runs on the call's stream while the
previous slice's output is copied back on a second stream (bitmm_capi.cu, run_pipelined).
These shapes take that path, with ragged last slices. Results must equal the device-pointer
path bit for bit, and an encoding error in the last slice must still be reported.

Where K allows, the output crosses PCIe as one 16-bit word per cell (csrc/wire.cuh): the
device narrows the int32 units, the host widens them and applies the epilogue's fp32 scale
sequence. Every test here runs with that wire and with BITMM_HOST_WIRE=32 (4-byte copies).
Each slice's GEMM waits for that slice's input copies with cuStreamWaitValue32 on a flag the
copy stream writes (default), a one-warp spin kernel on it (BITMM_WIRE_WAIT=kernel), or an
event (BITMM_WIRE_WAIT=event; also the fallback of a slice whose flag write fails,
BITMM_WIRE_FAULT=flagwrite): all four must give the same bits."""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_2306_08960_b200 import _lib, api, data, device

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["wire16", "wire16-sse2", "wire32", "wire16-kernelwait",
                                      "wire16-eventwait", "wire16-flagfault"])
def wire(request, monkeypatch):
    """wire16: 16-bit words widened with the host's widest streaming stores (AVX-512 where
    present); wire16-sse2: the x86-64 baseline path; wire32: 4-byte copies; *wait / flagfault:
    the other ways a slice waits for its inputs (module docstring)."""
    for v in ("BITMM_HOST_WIRE", "BITMM_HOST_SIMD", "BITMM_WIRE_WAIT", "BITMM_WIRE_FAULT"):
        monkeypatch.delenv(v, raising=False)
    # 16-bit words throughout (the 12-bit packing of eligible parts: tests/test_wire12_gpu.py)
    monkeypatch.setenv("BITMM_WIRE_BITS", "16")
    if request.param == "wire32":
        monkeypatch.setenv("BITMM_HOST_WIRE", "32")
    elif request.param == "wire16-sse2":
        monkeypatch.setenv("BITMM_HOST_SIMD", "sse2")
    elif request.param == "wire16-kernelwait":
        monkeypatch.setenv("BITMM_WIRE_WAIT", "kernel")
    elif request.param == "wire16-eventwait":
        monkeypatch.setenv("BITMM_WIRE_WAIT", "event")
    elif request.param == "wire16-flagfault":
        monkeypatch.setenv("BITMM_WIRE_FAULT", "flagwrite")
    return request.param.split("-")[0]


def _bm(rows, cols, wpr, words):
    return api.BitMatrix.from_words(rows, cols, wpr, words)


def _planes(rng, rows, cols, scale=1.0):
    t, h, m, wpr = data.random_planes(rng, rows, cols)
    return api.ThmPlanes(_bm(rows, cols, wpr, t), _bm(rows, cols, wpr, h), _bm(rows, cols, wpr, m),
                         scale=scale), (t, h, m, wpr)


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()


def test_1x1_row_slices():
    rng = np.random.default_rng(11)
    m, n, k = 4196, 2056, 1000  # 34.5 MB fp32 output: six row slices, the last one ragged
    a, wpr = data.random_words(rng, m, k)
    b, _ = data.random_words(rng, n, k)
    got = api.gemm_1x1(_bm(m, k, wpr, a), _bm(n, k, wpr, b), 0.5, 1.5)
    want = torch.empty((m, n), dtype=torch.float32, device="cuda")
    device.gemm_1x1(_dev(a), _dev(b), k, 0.5, 1.5, out=want)
    assert np.array_equal(got, want.cpu().numpy())


def test_1x2_column_slices():
    rng = np.random.default_rng(12)
    m, n, k = 1100, 8200, 777  # 36 MB output: slices of activation rows = output columns
    w, wpr = data.random_words(rng, m, k)
    a, (t, h, mm, _) = _planes(rng, n, k, scale=0.5)
    rs = rng.uniform(0.5, 1.5, m).astype(np.float32)
    cs = rng.uniform(0.5, 1.5, n).astype(np.float32)
    got = api.gemm_1x2(_bm(m, k, wpr, w), 1.25, a, row_scale=rs, col_scale=cs)
    want = torch.empty((m, n), dtype=torch.float32, device="cuda")
    device.gemm_1x2(_dev(w), 1.25, _dev(t), _dev(h), _dev(mm), k, a_scale=0.5,
                    row_scale=torch.from_numpy(rs).cuda(), col_scale=torch.from_numpy(cs).cuda(),
                    out=want)
    assert np.array_equal(got, want.cpu().numpy())


def test_2x2_row_slices():
    rng = np.random.default_rng(13)
    m, n, k = 4200, 2100, 700
    wp, (wt, wh, wm, _) = _planes(rng, m, k, scale=0.25)
    ap, (at, ah, am, _) = _planes(rng, n, k, scale=0.5)
    got = api.gemm_2x2(wp, ap)
    want = torch.empty((m, n), dtype=torch.float32, device="cuda")
    device.gemm_2x2(*[_dev(x) for x in (wt, wh, wm, at, ah, am)], k, w_scale=0.25, a_scale=0.5,
                    out=want)
    assert np.array_equal(got, want.cpu().numpy())


def test_errors_in_the_last_slice():
    rng = np.random.default_rng(14)
    m, n, k = 4196, 2056, 1000
    a, wpr = data.random_words(rng, m, k)
    b, _ = data.random_words(rng, n, k)
    am = _bm(m, k, wpr, a)
    am.words[m - 1, wpr - 1] |= np.uint64(1) << np.uint64(63)  # padding bit of the last row
    with pytest.raises(ValueError, match="padding"):
        api.gemm_1x1(am, _bm(n, k, wpr, b))
    # an illegal plane state (t = h = 1) in the last activation row of a sliced 1/2 call
    w, _ = data.random_words(rng, 1100, 777)
    ap, (t, h, mm, wpr2) = _planes(rng, 8200, 777)
    t[-1, 0] |= np.uint64(1)
    h[-1, 0] |= np.uint64(1)
    bad = api.ThmPlanes(_bm(8200, 777, wpr2, t), _bm(8200, 777, wpr2, h), _bm(8200, 777, wpr2, mm))
    with pytest.raises(api.InvalidEncoding):
        api.gemm_1x2(_bm(1100, 777, wpr2, w), 1.0, bad)


@pytest.mark.parametrize("k", [4096, 8192])
def test_illegal_planes_in_full_slices(k):
    """K a multiple of 4096: every slice takes the expansion's full-slice fast path, which
    validates the plane states itself. One illegal state (t = h = 1) anywhere must still
    surface as InvalidEncoding, for either operand of 2/2."""
    rng = np.random.default_rng(k)
    m, n = 300, 260
    for side in ("w", "a"):
        wp, (wt, wh, wm, wpr) = _planes(rng, m, k)
        ap, (at, ah, am, _) = _planes(rng, n, k)
        t, h = (wt, wh) if side == "w" else (at, ah)
        row = 7 if side == "w" else n - 1
        t[row, wpr - 1] |= np.uint64(1) << np.uint64(40)
        h[row, wpr - 1] |= np.uint64(1) << np.uint64(40)
        with pytest.raises(api.InvalidEncoding):
            api.gemm_2x2(wp, ap)
    # and a clean call right after still matches the device path
    wp, (wt, wh, wm, _) = _planes(rng, m, k)
    ap, (at, ah, am, _) = _planes(rng, n, k)
    got = api.gemm_2x2(wp, ap)
    want = torch.empty((m, n), dtype=torch.float32, device="cuda")
    device.gemm_2x2(*[_dev(x) for x in (wt, wh, wm, at, ah, am)], k, out=want)
    assert np.array_equal(got, want.cpu().numpy())


def _full_row(k, wpr):
    """One packed row with all K bits set and zero padding."""
    full = np.zeros(wpr, np.uint64)
    full[: k // 64] = ~np.uint64(0)
    if k % 64:
        full[k // 64] = np.uint64((1 << (k % 64)) - 1)
    return full


def _p(x):
    return C.c_void_p(x.ctypes.data) if x is not None else None


@pytest.mark.parametrize("k", [1000, 4096])
def test_1x1_both_outputs_and_wire_bytes(wire, k):
    """int32 units and scaled floats requested together; the units are K - 2*popc exactly and
    the floats are (gamma_a*gamma_b)*float(units). The D2H byte count shows which wire ran."""
    lib = _lib.load()
    rng = np.random.default_rng(k)
    m, n = 2300, 4100  # 37.7 MB per output: row slices, ragged last slice
    a, wpr = data.random_words(rng, m, k)
    b, _ = data.random_words(rng, n, k)
    units = np.empty((m, n), np.int32)
    vals = np.empty((m, n), np.float32)
    rc = lib.bitmm_gemm_1x1_host(_p(a), m, _p(b), n, k, wpr, 0.75, 1.25, _p(units), _p(vals), n)
    assert rc == 0, lib.bitmm_last_error()
    want = torch.empty((m, n), dtype=torch.int32, device="cuda")
    device.gemm_1x1(_dev(a), _dev(b), k, units=want)
    assert np.array_equal(units, want.cpu().numpy())
    assert np.array_equal(vals, np.float32(0.75 * 1.25) * units.astype(np.float32))
    per_cell = 2 if wire == "wire16" else 8
    assert lib.bitmm_last_d2h_bytes() == m * n * per_cell


@pytest.mark.parametrize("k", [777, 10922, 10923])
def test_1x2_wire_bound(wire, k):
    """1/2 units = 2*sum s*p in [-6K, 6K]: K = 10922 is the last K the 16-bit wire carries
    (all-ones weights against all-p3 activations reach the bound); 10923 falls back."""
    lib = _lib.load()
    rng = np.random.default_rng(k)
    m, n = 1030, 8200  # 33.8 MB of output: the wire applies from 32 MB
    w, wpr = data.random_words(rng, m, k)
    t, h, mm, _ = data.random_planes(rng, n, k)
    if k != 777:
        full = _full_row(k, wpr)
        w[0] = full                         # row 0: all +1
        t[0], h[0], mm[0] = full, 0, full   # column 0: all level 3 (t=1, h=0, m=1)
    rs = rng.uniform(0.5, 1.5, m).astype(np.float32)
    cs = rng.uniform(0.5, 1.5, n).astype(np.float32)
    units = np.empty((m, n), np.int32)
    vals = np.empty((m, n), np.float32)
    rc = lib.bitmm_gemm_1x2_host(_p(w), m, 1.5, _p(t), _p(h), _p(mm), n, k, wpr, 0.5, 1, 2.0,
                                 _p(rs), _p(cs), _p(units), _p(vals), n)
    assert rc == 0, lib.bitmm_last_error()
    wu = torch.empty((m, n), dtype=torch.int32, device="cuda")
    wv = torch.empty((m, n), dtype=torch.float32, device="cuda")
    device.gemm_1x2(_dev(w), 1.5, _dev(t), _dev(h), _dev(mm), k, a_scale=0.5, a_gamma=2.0,
                    row_scale=torch.from_numpy(rs).cuda(), col_scale=torch.from_numpy(cs).cuda(),
                    units=wu, out=wv)
    assert np.array_equal(units, wu.cpu().numpy())
    assert np.array_equal(vals, wv.cpu().numpy())
    if k != 777:
        assert units[0, 0] == 6 * k
    narrow = wire == "wire16" and k <= 10922
    assert lib.bitmm_last_d2h_bytes() == m * n * (2 if narrow else 8)


@pytest.mark.parametrize("k", [700, 7281, 7282])
def test_2x2_wire_bound(wire, k):
    """2/2 units = 4*sum p_w*p_a in [0, 36K]; K = 7281 is the last K the 16-bit wire carries."""
    lib = _lib.load()
    rng = np.random.default_rng(k)
    m, n = 4200, 2100  # 35 MB of output: the wire applies from 32 MB
    wt, wh, wm, wpr = data.random_planes(rng, m, k)
    at, ah, am, _ = data.random_planes(rng, n, k)
    full = _full_row(k, wpr)
    for t_, h_, m_ in ((wt, wh, wm), (at, ah, am)):
        t_[0], h_[0], m_[0] = full, 0, full  # row 0 of each side: all level 3
    rs = rng.uniform(0.5, 1.5, m).astype(np.float32)
    units = np.empty((m, n), np.int32)
    vals = np.empty((m, n), np.float32)
    rc = lib.bitmm_gemm_2x2_host(_p(wt), _p(wh), _p(wm), m, 0.25, 0, 1.0, _p(at), _p(ah), _p(am),
                                 n, k, wpr, 0.5, 1, 3.0, _p(rs), None, _p(units), _p(vals), n)
    assert rc == 0, lib.bitmm_last_error()
    wu = torch.empty((m, n), dtype=torch.int32, device="cuda")
    wv = torch.empty((m, n), dtype=torch.float32, device="cuda")
    device.gemm_2x2(*[_dev(x) for x in (wt, wh, wm, at, ah, am)], k, w_scale=0.25, a_scale=0.5,
                    a_gamma=3.0, row_scale=torch.from_numpy(rs).cuda(), units=wu, out=wv)
    assert np.array_equal(units, wu.cpu().numpy())
    assert np.array_equal(vals, wv.cpu().numpy())
    assert units[0, 0] == 36 * k
    narrow = wire == "wire16" and k <= 7281
    assert lib.bitmm_last_d2h_bytes() == m * n * (2 if narrow else 8)


def test_small_outputs_keep_the_4_byte_copy(wire):
    """Below 32 MB of output a host call copies 4-byte cells (one unsliced copy; the wire's
    pool start-up would cost more than it saves)."""
    lib = _lib.load()
    rng = np.random.default_rng(16)
    m, n, k = 1024, 1024, 1024
    a, wpr = data.random_words(rng, m, k)
    b, _ = data.random_words(rng, n, k)
    units = np.empty((m, n), np.int32)
    assert lib.bitmm_gemm_1x1_host(_p(a), m, _p(b), n, k, wpr, 1.0, 1.0, _p(units), None, n) == 0
    assert lib.bitmm_last_d2h_bytes() == m * n * 4
