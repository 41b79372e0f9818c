"""The host-flavour entry points (`bitmm_gemm_*_host`) produce outputs of 32 MB and more in
slices: each slice's inputs are copied in and its GEMM runs on the call's stream while the
previous slice's output is copied back on a second stream (bitmm_capi.cu, run_pipelined).
These shapes take that path, with ragged last slices. Results must equal the device-pointer
path bit for bit, and an encoding error in the last slice must still be reported."""
import numpy as np
import pytest
import torch

from paper_2306_08960_b200 import api, data, device

pytestmark = pytest.mark.gpu


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
