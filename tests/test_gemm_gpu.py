"""GPU parity: the sm_100a 1/1, 1/2, 2/2 GEMMs vs the oracle and the reference's golden
outputs. Integer work is compared bit-exactly (tolerance 0, as acceptance.cpp:245-267 and
verify.cpp:261-287 do: float output == scale * float(units))."""
import numpy as np
import pytest

from conftest import gemm_case
from paper_2306_08960_b200 import api, data

pytestmark = pytest.mark.gpu


def _bm(words, rows, cols, wpr):
    return api.BitMatrix.from_words(rows, cols, wpr, words)


def _tp(t, h, m, rows, cols, wpr, scale=1.0, gamma=None):
    return api.ThmPlanes(_bm(t, rows, cols, wpr), _bm(h, rows, cols, wpr), _bm(m, rows, cols, wpr),
                         scale, gamma)


def _levels_tp(levels, scale=1.0, gamma=None):
    lv = np.asarray(levels, np.uint8).reshape(1, -1)
    return api.decompose_thm(api.TwoBitMatrix(1, lv.shape[1], lv.reshape(-1), scale), gamma)


# ---------------------------------------------------------------- frozen known answers
def test_frozen_cases_gpu():
    # test_kernels.cpp:89-143
    a = api.pack_signs(np.array([[1.0, -1.0, 1.0]], np.float32))
    b = api.pack_signs(np.array([[1.0, 1.0, 1.0]], np.float32))
    assert api.gemm_1x1(a, b)[0, 0] == 1.0
    assert api.gemm_1x1(a, b, 0.5, 2.0)[0, 0] == 1.0
    assert api.gemm_1x1(a, b, 2.0, 3.0)[0, 0] == 6.0
    w = api.pack_signs(np.array([[1.0, -1.0, 1.0, 1.0]], np.float32))
    ap = _levels_tp([0, 1, 2, 3])
    assert api.gemm_1x2(w, 1.0, ap)[0, 0] == 4.0
    assert api.gemm_1x2(w, 2.0, ap)[0, 0] == 8.0
    assert api.gemm_1x2(w, 2.0, _levels_tp([0, 1, 2, 3], gamma=0.5))[0, 0] == 4.0
    assert api.gemm_2x2(_levels_tp([3, 1]), _levels_tp([0, 2]))[0, 0] == 2.0
    assert api.gemm_2x2(_levels_tp([3]), _levels_tp([3]))[0, 0] == 9.0
    assert api.gemm_2x2(_levels_tp([3], 0.5), _levels_tp([3], 0.25))[0, 0] == 1.125


# ---------------------------------------------------------------- golden vectors
def test_golden_reference_outputs(gemm_golden):
    for i in range(int(gemm_golden["gemm_count"])):
        c = gemm_case(gemm_golden, i)
        m, k, n, wpr, lane = c["m"], c["k"], c["n"], c["wpr"], c["lane"]
        a, b = _bm(c["a"], m, k, wpr), _bm(c["b"], n, k, wpr)
        at, ah, am, _ = data.planes_from_levels(c["la"], lane)
        wt, wh, wm, _ = data.planes_from_levels(c["lw"], lane)
        ap = _tp(at, ah, am, n, k, wpr, c["s_a"], c["g_a"])
        wp = _tp(wt, wh, wm, m, k, wpr, c["s_w"])
        assert np.array_equal(api.gemm_1x1(a, b, c["g_a"], c["g_b"]), c["c11"]), i
        assert np.array_equal(api.gemm_1x2(a, c["g_w"], ap), c["c12"]), i
        assert np.array_equal(api.gemm_2x2(wp, ap), c["c22"]), i


# ---------------------------------------------------------------- random sweep vs oracle
def _units_host(fn_name, *args):
    import ctypes as C
    from paper_2306_08960_b200 import _lib
    lib = _lib.load()
    rc = getattr(lib, fn_name)(*args)
    assert rc == 0, _lib.last_error()


def _p(x):
    import ctypes as C
    return None if x is None else x.ctypes.data_as(C.c_void_p)


def test_random_shapes_units_vs_oracle(orc):
    # acceptance.cpp:245-260 style: many shapes incl. K past 256 and off the tile grid
    rng = np.random.default_rng(2024)
    shapes = [(int(rng.integers(1, 300)), int(rng.integers(1, 300)), int(rng.integers(1, 300)))
              for _ in range(60)]
    shapes += [(int(rng.integers(1, 160)), int(rng.integers(257, 4097)), int(rng.integers(1, 300)))
               for _ in range(12)]
    shapes += [(129, 1, 257), (1, 4096, 1), (300, 130, 511), (255, 128, 256), (256, 128, 255)]
    for (m, k, n) in shapes:
        a, wpr = data.random_words(rng, m, k)
        b, _ = data.random_words(rng, n, k)
        at, ah, am, _ = data.random_planes(rng, n, k)
        wt, wh, wm, _ = data.random_planes(rng, m, k)
        u11 = np.empty((m, n), np.int32)
        _units_host("bitmm_gemm_1x1_host", _p(a), m, _p(b), n, k, wpr, 1.0, 1.0, _p(u11), None, n)
        assert np.array_equal(u11, orc.gemm_1x1(a, b, k, wpr)[0]), (m, k, n)
        u12 = np.empty((m, n), np.int32)
        _units_host("bitmm_gemm_1x2_host", _p(a), m, 1.0, _p(at), _p(ah), _p(am), n, k, wpr, 1.0, 0,
                    1.0, None, None, _p(u12), None, n)
        assert np.array_equal(u12, orc.gemm_1x2(a, 1.0, at, ah, am, k, wpr)[0]), (m, k, n)
        u22 = np.empty((m, n), np.int32)
        _units_host("bitmm_gemm_2x2_host", _p(wt), _p(wh), _p(wm), m, 1.0, 0, 1.0, _p(at), _p(ah),
                    _p(am), n, k, wpr, 1.0, 0, 1.0, None, None, _p(u22), None, n)
        assert np.array_equal(u22, orc.gemm_2x2(wt, wh, wm, at, ah, am, k, wpr)[0]), (m, k, n)


def test_row_col_scale_epilogue_vs_oracle(orc):
    # BASELINE config 3 epilogue: per-row gamma (binary weights) x per-column beta
    rng = np.random.default_rng(3)
    for (m, k, n) in [(37, 333, 129), (256, 1024, 512)]:
        a, wpr = data.random_words(rng, m, k)
        at, ah, am, _ = data.random_planes(rng, n, k)
        wt, wh, wm, _ = data.random_planes(rng, m, k)
        rs = rng.uniform(0.5, 1.5, m).astype(np.float32)
        cs = rng.uniform(0.5, 1.5, n).astype(np.float32)
        got = api.gemm_1x2(_bm(a, m, k, wpr), 1.25, _tp(at, ah, am, n, k, wpr, 0.5, 0.75),
                           row_scale=rs, col_scale=cs)
        want = orc.gemm_1x2(a, 1.25, at, ah, am, k, wpr, 0.5, 0.75, rs, cs)[1]
        assert np.array_equal(got, want)
        got = api.gemm_2x2(_tp(wt, wh, wm, m, k, wpr, 0.25), _tp(at, ah, am, n, k, wpr, 0.5),
                           row_scale=rs, col_scale=cs)
        want = orc.gemm_2x2(wt, wh, wm, at, ah, am, k, wpr, 0.25, 0.5, None, None, rs, cs)[1]
        assert np.array_equal(got, want)


@pytest.mark.parametrize("lane", [64, 128, 512])
def test_lane_width_invariance(lane):
    # test_kernels.cpp:185-196: 512-bit vs 64-bit padding gives identical products
    rng = np.random.default_rng(lane)
    for k in (1, 63, 70, 200, 1000):
        bits_a = rng.integers(0, 2, (5, k), dtype=np.uint8)
        bits_b = rng.integers(0, 2, (7, k), dtype=np.uint8)
        wa, wpr = data.pack_bits(bits_a, lane)
        wb, _ = data.pack_bits(bits_b, lane)
        wa5, wpr5 = data.pack_bits(bits_a, 512)
        wb5, _ = data.pack_bits(bits_b, 512)
        got = api.gemm_1x1(_bm(wa, 5, k, wpr), _bm(wb, 7, k, wpr))
        assert np.array_equal(got, api.gemm_1x1(_bm(wa5, 5, k, wpr5), _bm(wb5, 7, k, wpr5)))


def test_shared_dim_cap():
    # test_kernels.cpp:198-204: K = 2^20 accepted, 2^20 + 1 rejected
    k = api.MAX_SHARED_DIM
    rng = np.random.default_rng(1)
    a, wpr = data.random_words(rng, 1, k)
    b, _ = data.random_words(rng, 2, k)
    got = api.gemm_1x1(_bm(a, 1, k, wpr), _bm(b, 2, k, wpr))
    want = (2 * data.unpack_bits(a, k).astype(np.int64) - 1) @ (2 * data.unpack_bits(b, k).astype(np.int64) - 1).T
    assert np.array_equal(got, want.astype(np.float32))
    big = api.BitMatrix(1, k + 1)
    with pytest.raises(ValueError):
        api.gemm_1x1(big, big)


# ---------------------------------------------------------------- errors (reference behaviour)
def test_shape_errors():
    a = api.BitMatrix(1, 3)
    with pytest.raises(ValueError):
        api.gemm_1x1(a, api.BitMatrix(1, 4))
    with pytest.raises(ValueError):
        api.gemm_1x1(a, api.BitMatrix(1, 3, 64))  # padding mismatch (test_kernels.cpp:103-104)
    with pytest.raises(ValueError):
        api.gemm_1x1(api.BitMatrix(0, 3), a)
    with pytest.raises(ValueError):
        api.gemm_1x1(a, a, threads=0)
    w = api.pack_signs(np.ones((1, 4), np.float32))
    bad = _levels_tp([0, 0, 0])
    with pytest.raises(ValueError):  # test_kernels.cpp:121-122
        api.gemm_1x2(w, 1.0, bad)
    with pytest.raises(ValueError):  # test_kernels.cpp:141-142
        api.gemm_2x2(_levels_tp([3, 1]), bad)


def test_invalid_encoding_detected_on_device():
    rng = np.random.default_rng(9)
    k, n = 300, 17
    w, wpr = data.random_words(rng, 4, k)
    for bad in ("t_and_h", "t_without_m", "h_with_m", "padding"):
        t, h, m, _ = data.random_planes(rng, n, k)
        if bad == "t_and_h":
            t[3, 1] |= np.uint64(1 << 5); h[3, 1] |= np.uint64(1 << 5); m[3, 1] |= np.uint64(1 << 5)
        elif bad == "t_without_m":
            t[5, 0] |= np.uint64(1); h[5, 0] &= ~np.uint64(1); m[5, 0] &= ~np.uint64(1)
        elif bad == "h_with_m":
            h[0, 2] |= np.uint64(1 << 7); m[0, 2] |= np.uint64(1 << 7); t[0, 2] &= ~np.uint64(1 << 7)
        else:
            m[n - 1, wpr - 1] |= np.uint64(1 << 63)
        ap = api.ThmPlanes(*(api.BitMatrix.__new__(api.BitMatrix) for _ in range(3)))
        for bm, words in zip((ap.t, ap.h, ap.m), (t, h, m)):
            bm._rows, bm._cols, bm._wpr, bm.words = n, k, wpr, words
        with pytest.raises(api.InvalidEncoding):
            api.gemm_1x2(_bm(w, 4, k, wpr), 1.0, ap)
        # plane errors win over shape errors (kernels.cpp:186 validates first)
        with pytest.raises(api.InvalidEncoding):
            api.gemm_1x2(api.BitMatrix(4, k + 1), 1.0, ap)
    # and a valid call afterwards is unaffected (latched status was cleared)
    t, h, m, _ = data.random_planes(rng, n, k)
    api.gemm_1x2(_bm(w, 4, k, wpr), 1.0, _tp(t, h, m, n, k, wpr))


def test_nonpositive_plane_scale_is_invalid_encoding():
    w = api.pack_signs(np.ones((1, 4), np.float32))
    ap = _levels_tp([0, 1, 2, 3], scale=1.0)
    ap.scale = 0.0
    with pytest.raises(api.InvalidEncoding):
        api.gemm_1x2(w, 1.0, ap)


# ---------------------------------------------------------------- device flavour
def test_device_flavour_matches_host_and_is_deterministic(orc):
    import torch
    rng = np.random.default_rng(11)
    m, n, k = 1000, 777, 2000
    a, wpr = data.random_words(rng, m, k)
    b, _ = data.random_words(rng, n, k)
    from paper_2306_08960_b200 import device
    da = torch.from_numpy(a.view(np.int64)).cuda()
    db = torch.from_numpy(b.view(np.int64)).cuda()
    s = torch.cuda.Stream()
    u1 = torch.empty((m, n), dtype=torch.int32, device="cuda")
    u2 = torch.empty_like(u1)
    u3 = torch.empty_like(u1)
    f1 = torch.empty((m, n), dtype=torch.float32, device="cuda")
    with torch.cuda.stream(s):
        device.gemm_1x1(da, db, k, 0.5, 1.5, units=u1, out=f1, stream=s)
        device.gemm_1x1(da, db, k, units=u2, stream=s)
        device.gemm_1x1(da, db, k, units=u3, stream=s, popc=True)
        device.status(s)
    s.synchronize()
    want = orc.gemm_1x1(a, b, k, wpr, 0.5, 1.5)
    assert np.array_equal(u1.cpu().numpy(), want[0])
    assert np.array_equal(f1.cpu().numpy(), want[1])
    assert torch.equal(u1, u2) and torch.equal(u1, u3)


def test_device_padding_violation_reported():
    import torch
    from paper_2306_08960_b200 import device
    rng = np.random.default_rng(12)
    k = 100
    a, wpr = data.random_words(rng, 3, k)
    a[1, 1] |= np.uint64(1 << 40)  # bit 104 >= K: nonzero padding
    da = torch.from_numpy(a.view(np.int64)).cuda()
    u = torch.empty((3, 3), dtype=torch.int32, device="cuda")
    device.gemm_1x1(da, da, k, units=u)
    with pytest.raises(ValueError):
        device.status()
    device.status()  # cleared


# ---------------------------------------------------------------- full-size properties
def _sample_rows(rng, m, count=8):
    return np.sort(rng.choice(m, size=count, replace=False))


def test_full_size_1x1_4096(orc):
    import torch
    from paper_2306_08960_b200 import device
    rng = np.random.default_rng(4096)
    m = n = k = 4096
    a, wpr = data.random_words(rng, m, k)
    b, _ = data.random_words(rng, n, k)
    da = torch.from_numpy(a.view(np.int64)).cuda()
    db = torch.from_numpy(b.view(np.int64)).cuda()
    u = torch.empty((m, n), dtype=torch.int32, device="cuda")
    up = torch.empty_like(u)
    device.gemm_1x1(da, db, k, units=u)
    device.gemm_1x1(da, db, k, units=up, popc=True)  # independent CUDA-core evaluation
    # complementing every logical bit of B negates every cell (size-independent identity)
    bc = (~b) & data.tail_mask_words(k, wpr)[None, :]
    dbc = torch.from_numpy(bc.view(np.int64)).cuda()
    un = torch.empty_like(u)
    device.gemm_1x1(da, dbc, k, units=un)
    device.status()
    assert torch.equal(u, up)
    assert torch.equal(un, -u)
    assert bool(((u.abs() <= k) & ((u - k) % 2 == 0)).all())
    rows = _sample_rows(rng, m)
    want = orc.gemm_1x1(a[rows], b, k, wpr)[0]
    assert np.array_equal(u.cpu().numpy()[rows], want)


def test_full_size_2x2_and_1x2(orc):
    import torch
    from paper_2306_08960_b200 import device
    rng = np.random.default_rng(22)
    # BASELINE config 2 (2/2 4096^3) and config 3 (1/2, 2-bit activations M=8192 x K=4096 x
    # binary weights N=4096 — reference orientation: binary operand on the rows)
    k = 4096
    wt, wh, wm, wpr = data.random_planes(rng, 4096, k)
    at, ah, am, _ = data.random_planes(rng, 8192, k)
    w, _ = data.random_words(rng, 4096, k)
    T = lambda x: torch.from_numpy(x.view(np.int64)).cuda()  # noqa: E731
    d = [T(x) for x in (wt, wh, wm, at, ah, am, w)]
    u22 = torch.empty((4096, 8192), dtype=torch.int32, device="cuda")
    device.gemm_2x2(d[0], d[1], d[2], d[3], d[4], d[5], k, units=u22)
    u12 = torch.empty((4096, 8192), dtype=torch.int32, device="cuda")
    device.gemm_1x2(d[6], 1.0, d[3], d[4], d[5], k, units=u12)
    rs = torch.empty(4096, device="cuda").uniform_(0.5, 1.5)
    cs = torch.empty(8192, device="cuda").uniform_(0.5, 1.5)
    f12 = torch.empty((4096, 8192), dtype=torch.float32, device="cuda")
    device.gemm_1x2(d[6], 1.0, d[3], d[4], d[5], k, row_scale=rs, col_scale=cs, out=f12)
    device.status()
    rows = _sample_rows(rng, 4096)
    assert np.array_equal(u22.cpu().numpy()[rows],
                          orc.gemm_2x2(wt[rows], wh[rows], wm[rows], at, ah, am, k, wpr)[0])
    want12 = orc.gemm_1x2(w[rows], 1.0, at, ah, am, k, wpr, 1.0, None,
                          rs.cpu().numpy()[rows], cs.cpu().numpy())
    assert np.array_equal(u12.cpu().numpy()[rows], want12[0])
    assert np.array_equal(f12.cpu().numpy()[rows], want12[1])
    # 2/2 units are 4 * sum p_w p_a >= 0, multiples of 4, bounded by 36 K
    assert bool(((u22 >= 0) & (u22 % 4 == 0) & (u22 <= 36 * k)).all())


def test_full_size_1x1_32768_sampled(orc):
    # BASELINE config 5 on one GPU (the N-shard of a multi-GPU run is the same kernel)
    import torch
    from paper_2306_08960_b200 import device
    rng = np.random.default_rng(32768)
    m = n = k = 32768
    a, wpr = data.random_words(rng, m, k)
    b, _ = data.random_words(rng, n, k)
    da = torch.from_numpy(a.view(np.int64)).cuda()
    db = torch.from_numpy(b.view(np.int64)).cuda()
    u = torch.empty((m, n), dtype=torch.int32, device="cuda")
    device.gemm_1x1(da, db, k, units=u)
    device.status()
    rows = _sample_rows(rng, m, 4)
    want = orc.gemm_1x1(a[rows], b, k, wpr)[0]
    assert np.array_equal(u[torch.from_numpy(rows).cuda()].cpu().numpy(), want)
    cols = _sample_rows(rng, n, 4)
    wantc = orc.gemm_1x1(a, b[cols], k, wpr)[0]
    assert np.array_equal(u[:, torch.from_numpy(cols).cuda()].cpu().numpy(), wantc)


@pytest.mark.parametrize("m,n,k", [(256, 256, 1 << 16), (8192, 4352, 2048), (300, 700, 4000)])
def test_long_k_and_ragged_tiles_exact(orc, m, n, k):
    """Long K (one tile, 512 K-blocks), a partial last N-tile (4352 = 17 x 256) and ragged
    M/N: every sampled row equals the integer oracle and all cells match the independent
    CUDA-core kernel; repeated launches are bit-identical."""
    import torch
    from paper_2306_08960_b200 import device
    rng = np.random.default_rng(m + n + k)
    a, wpr = data.random_words(rng, m, k)
    b, _ = data.random_words(rng, n, k)
    u = torch.empty((m, n), dtype=torch.int32, device="cuda")
    f = torch.empty((m, n), dtype=torch.float32, device="cuda")
    T = lambda x: torch.from_numpy(x.view(np.int64)).cuda()  # noqa: E731
    for _ in range(3):
        device.gemm_1x1(T(a), T(b), k, 0.5, 0.75, units=u, out=f)
    device.status()
    rows = np.unique(np.concatenate([np.arange(min(m, 4)), rng.choice(m, 12), [m - 1]]))
    want_u, want_f = orc.gemm_1x1(a[rows], b, k, wpr, 0.5, 0.75)
    assert np.array_equal(u.cpu().numpy()[rows], want_u)
    assert np.array_equal(f.cpu().numpy()[rows], want_f)
    up = torch.empty_like(u)
    device.gemm_1x1(T(a), T(b), k, units=up, popc=True)
    assert torch.equal(u, up)


@pytest.mark.parametrize("k", [1 << 20, (1 << 20) - 77])
def test_extreme_accumulators_at_max_shared_dim(k):
    """Largest partial sums the formats allow: K = 2^20 (BITMM_MAX_SHARED_DIM) with every
    level 3 (2/2: sum p_w p_a = 9K, units 36K), all-equal and all-opposite signs (1/1: +-K)
    and mixed rows, so any accumulator rounding or overflow would show."""
    import torch
    from paper_2306_08960_b200 import device
    m, n = 160, 200
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()  # noqa: E731
    # 2/2, every level 3 on both sides
    lv = np.full((m, k), 3, np.uint8)
    wt, wh, wm, wpr = data.planes_from_levels(lv)
    lva = np.full((n, k), 3, np.uint8)
    at, ah, am, _ = data.planes_from_levels(lva)
    u = torch.empty((m, n), dtype=torch.int32, device="cuda")
    device.gemm_2x2(T(wt), T(wh), T(wm), T(at), T(ah), T(am), k, units=u)
    device.status()
    assert bool((u == 36 * k).all())
    # 1/1: rows of A all +1 or all -1 (alternating), B all +1 -> units = +-K
    sign_rows = (np.arange(m) % 2 == 0)
    bits = np.repeat(sign_rows[:, None], k, axis=1).astype(np.uint8)
    a, _ = data.pack_bits(bits)
    b, _ = data.pack_bits(np.ones((n, k), np.uint8))
    device.gemm_1x1(T(a), T(b), k, units=u)
    device.status()
    want = np.where(sign_rows, k, -k)[:, None].repeat(n, axis=1)
    assert np.array_equal(u.cpu().numpy(), want)
    # 1/2: w all +1, activations all level 3 -> units = 2 * 3K
    device.gemm_1x2(T(b[:m] if m <= n else a), 1.0, T(at), T(ah), T(am), k, units=u)
    device.status()
    assert bool((u == 6 * k).all())


@pytest.mark.parametrize("k", [4095, 4096, 4097, 8192, 8193, 12288, 12352])
def test_expansion_slice_boundaries(orc, k):
    """K around 4096-element slice boundaries: rows mix full slices (the expansion's fast path,
    no per-word checks) with a partial last slice (the checked path), for sign and plane
    operands, with and without level scales (the p/2 level encoding folds into the shift)."""
    rng = np.random.default_rng(k)
    m, n = 67, 45
    a, wpr = data.random_words(rng, m, k)
    b, _ = data.random_words(rng, n, k)
    at, ah, am, _ = data.random_planes(rng, n, k)
    wt, wh, wm, _ = data.random_planes(rng, m, k)
    u11 = np.empty((m, n), np.int32)
    _units_host("bitmm_gemm_1x1_host", _p(a), m, _p(b), n, k, wpr, 1.0, 1.0, _p(u11), None, n)
    assert np.array_equal(u11, orc.gemm_1x1(a, b, k, wpr)[0])
    u12 = np.empty((m, n), np.int32)
    _units_host("bitmm_gemm_1x2_host", _p(a), m, 1.0, _p(at), _p(ah), _p(am), n, k, wpr, 1.0, 0,
                1.0, None, None, _p(u12), None, n)
    assert np.array_equal(u12, orc.gemm_1x2(a, 1.0, at, ah, am, k, wpr)[0])
    u22 = np.empty((m, n), np.int32)
    _units_host("bitmm_gemm_2x2_host", _p(wt), _p(wh), _p(wm), m, 1.0, 0, 1.0, _p(at), _p(ah),
                _p(am), n, k, wpr, 1.0, 0, 1.0, None, None, _p(u22), None, n)
    assert np.array_equal(u22, orc.gemm_2x2(wt, wh, wm, at, ah, am, k, wpr)[0])
    # scaled fp32 outputs (reference scale order) for the level routines
    w_planes = api.ThmPlanes(*(api.BitMatrix.from_words(m, k, wpr, x) for x in (wt, wh, wm)), scale=0.25)
    a_planes = api.ThmPlanes(*(api.BitMatrix.from_words(n, k, wpr, x) for x in (at, ah, am)), scale=0.5,
                             gamma=1.5)
    got = api.gemm_2x2(w_planes, a_planes)
    want = orc.gemm_2x2(wt, wh, wm, at, ah, am, k, wpr, 0.25, 0.5, None, 1.5)[1]
    assert np.array_equal(got, want)
