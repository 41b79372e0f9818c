"""Out-of-bounds writes and run-to-run determinism (compute-sanitizer is closed on this pool, so
these take its place for the output side and for races):

* every routine writes its M x N output into the top-left block of a larger buffer filled with
  a sentinel, with ldc > N (TMA-store pitches and the stride-36 fallback pitch), for ragged
  M / N that leave partial tiles and partial TMA boxes: cells outside the block must keep the
  sentinel, cells inside must equal the oracle. (This found two bugs: TMA stores clip a row at
  16-byte granularity, so an N that is not a multiple of 4 with ldc > N wrote up to 3 cells
  past N; and the fallback's 16-byte stores checked N but not ldc, a misaligned address when
  ldc is not a multiple of 4.)
* the grouped launch, the folded-residual APB layer and the 2-bit APB layer repeated many times
  must give bit-identical results every time (a pipeline race shows up as a changed bit).
"""
import numpy as np
import pytest

from paper_2306_08960_b200 import api, data

pytestmark = pytest.mark.gpu

SENTINEL = -123456789


def _T(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()


@pytest.mark.parametrize("m,n,k,pad", [(257, 193, 1000, 36), (300, 385, 513, 7), (129, 64, 4096, 64),
                                       (1, 1, 1, 3), (513, 191, 256, 4), (200, 64, 700, 1),
                                       (130, 256, 300, 5)])
def test_outputs_stay_inside_their_block(orc, m, n, k, pad):
    import torch
    from paper_2306_08960_b200 import device
    rng = np.random.default_rng(m * n + k)
    a, wpr = data.random_words(rng, m, k)
    b, _ = data.random_words(rng, n, k)
    t, h, mm, _ = data.random_planes(rng, n, k)
    wt, wh, wm, _ = data.random_planes(rng, m, k)
    ldc = n + pad
    buf_u = torch.full((m + 3, ldc), SENTINEL, dtype=torch.int32, device="cuda")
    buf_f = torch.full((m + 3, ldc), float(SENTINEL), dtype=torch.float32, device="cuda")
    lib = __import__("paper_2306_08960_b200._lib", fromlist=["load"]).load()
    s = torch.cuda.current_stream().cuda_stream
    P = lambda x: x.data_ptr()  # noqa: E731

    def check(want_u, want_f=None):
        gu = buf_u.cpu().numpy()
        assert np.array_equal(gu[:m, :n], want_u)
        assert (gu[:m, n:] == SENTINEL).all() and (gu[m:] == SENTINEL).all()
        if want_f is not None:
            gf = buf_f.cpu().numpy()
            assert np.array_equal(gf[:m, :n], want_f)
            assert (gf[:m, n:] == SENTINEL).all() and (gf[m:] == SENTINEL).all()

    da, db = _T(a), _T(b)
    assert lib.bitmm_gemm_1x1_dev(P(da), m, P(db), n, k, wpr, 0.5, 1.5, P(buf_u), P(buf_f), ldc, s) == 0
    device.status()
    check(*orc.gemm_1x1(a, b, k, wpr, 0.5, 1.5))
    dt, dh, dm = _T(t), _T(h), _T(mm)
    assert lib.bitmm_gemm_1x2_dev(P(da), m, 1.0, P(dt), P(dh), P(dm), n, k, wpr, 1.0, 0, 1.0, None, None,
                                  P(buf_u), P(buf_f), ldc, s) == 0
    device.status()
    check(*orc.gemm_1x2(a, 1.0, t, h, mm, k, wpr))
    dwt, dwh, dwm = _T(wt), _T(wh), _T(wm)
    assert lib.bitmm_gemm_2x2_dev(P(dwt), P(dwh), P(dwm), m, 1.0, 0, 1.0, P(dt), P(dh), P(dm), n, k, wpr, 1.0,
                                  0, 1.0, None, None, P(buf_u), None, ldc, s) == 0
    device.status()
    check(orc.gemm_2x2(wt, wh, wm, t, h, mm, k, wpr)[0])


def test_repeated_launches_are_bit_identical(orc):
    import torch
    from paper_2306_08960_b200 import device
    rng = np.random.default_rng(99)
    m, n, k = 1100, 900, 3000
    a, wpr = data.random_words(rng, m, k)
    b, _ = data.random_words(rng, n, k)
    t, h, mm, _ = data.random_planes(rng, n, k)
    wt, wh, wm, _ = data.random_planes(rng, m, k)
    d = {key: _T(v) for key, v in dict(a=a, b=b, t=t, h=h, mm=mm, wt=wt, wh=wh, wm=wm).items()}
    outs = [torch.empty((m, n), dtype=torch.int32, device="cuda") for _ in range(3)]
    f12 = torch.empty((m, n), dtype=torch.float32, device="cuda")
    rs = torch.rand(m, device="cuda") + 0.5
    cs = torch.rand(n, device="cuda") + 0.5

    def group():
        device.gemm_batch([dict(routine="1x1", a=d["a"], b=d["b"], k=k, units=outs[0]),
                           dict(routine="1x2", w=d["a"], t=d["t"], h=d["h"], m=d["mm"], k=k, units=outs[1],
                                out=f12, row_scale=rs, col_scale=cs),
                           dict(routine="2x2", wt=d["wt"], wh=d["wh"], wm=d["wm"], t=d["t"], h=d["h"],
                                m=d["mm"], k=k, units=outs[2])])

    group()
    device.status()
    first = [o.clone() for o in outs] + [f12.clone()]
    assert np.array_equal(first[0].cpu().numpy(), orc.gemm_1x1(a, b, k, wpr)[0])
    for _ in range(100):
        group()
    device.status()
    for o, f in zip(outs + [f12], first):
        assert torch.equal(o, f)

    # APB layers (fp32 folded residual; 2-bit exact), repeated
    rows, cols, tokens = 700, 768, 1000
    w, alpha, _ = data.apb_weights(rng, rows, cols)
    layer = api.decompose_apb(w, alpha)
    r = layer.residual
    x = torch.from_numpy(rng.standard_normal((cols, tokens)).astype(np.float32)).cuda()
    Tf = lambda v: torch.from_numpy(np.ascontiguousarray(v)).cuda()  # noqa: E731
    bw, al, rp, ci, vv = _T(layer.bin.words), Tf(alpha), _T(r.row_ptr), _T(r.col_idx), Tf(r.vals)
    t2, h2, m2, _ = data.random_planes(rng, tokens, cols)
    dt2, dh2, dm2 = _T(t2), _T(h2), _T(m2)
    y = torch.empty((rows, tokens), dtype=torch.float32, device="cuda")
    y2 = torch.empty_like(y)
    device.layer_forward(bw, cols, al, rp, ci, vv, x, y)
    device.layer_forward_2bit(bw, cols, al, rp, ci, vv, dt2, dh2, dm2, y2, a_scale=0.5)
    device.status()
    ref_y, ref_y2 = y.clone(), y2.clone()
    for _ in range(50):
        device.layer_forward(bw, cols, al, rp, ci, vv, x, y)
        device.layer_forward_2bit(bw, cols, al, rp, ci, vv, dt2, dh2, dm2, y2, a_scale=0.5)
    device.status()
    assert torch.equal(y, ref_y) and torch.equal(y2, ref_y2)


@pytest.mark.parametrize("rows,tokens,pad", [(300, 385, 7), (129, 200, 1)])
def test_apb_outputs_stay_inside_their_block(orc, rows, tokens, pad):
    import torch
    from paper_2306_08960_b200 import _lib, device
    lib = _lib.load()
    rng = np.random.default_rng(rows + tokens)
    cols = 768
    w, alpha, _ = data.apb_weights(rng, rows, cols)
    layer = api.decompose_apb(w, alpha)
    r = layer.residual
    x = rng.standard_normal((cols, tokens)).astype(np.float32)
    t2, h2, m2, wpr = data.random_planes(rng, tokens, cols)
    Tf = lambda v: torch.from_numpy(np.ascontiguousarray(v)).cuda()  # noqa: E731
    keep = [_T(layer.bin.words), Tf(alpha), _T(r.row_ptr), _T(r.col_idx), Tf(r.vals), Tf(x), _T(t2), _T(h2),
            _T(m2)]
    bw, al, rp, ci, vv, dx, dt, dh, dm = (v.data_ptr() for v in keep)
    ldc = tokens + pad
    s = torch.cuda.current_stream().cuda_stream
    buf = torch.full((rows + 2, ldc), float(SENTINEL), dtype=torch.float32, device="cuda")
    assert lib.bitmm_layer_forward_dev(rows, cols, 1.0, al, bw, layer.bin.words_per_row(), rp, ci, vv, dx,
                                       tokens, tokens, buf.data_ptr(), ldc, s) == 0
    device.status()
    g = buf.cpu().numpy()
    assert (g[:rows, tokens:] == SENTINEL).all() and (g[rows:] == SENTINEL).all()
    want = orc.layer_forward(rows, cols, 1.0, layer.bin.words, layer.bin.words_per_row(), r.row_ptr, r.col_idx,
                             r.vals, x, row_alpha=alpha)
    assert np.linalg.norm(g[:rows, :tokens] - want) / np.linalg.norm(want) < 1e-5
    buf.fill_(float(SENTINEL))
    assert lib.bitmm_layer_forward_2bit_dev(rows, cols, 1.0, al, bw, wpr, rp, ci, vv, dt, dh, dm, tokens, 0.5,
                                            0, 1.0, buf.data_ptr(), ldc, s) == 0
    device.status()
    g = buf.cpu().numpy()
    assert (g[:rows, tokens:] == SENTINEL).all() and (g[rows:] == SENTINEL).all()
    want2 = orc.layer_forward_2bit(rows, cols, 1.0, layer.bin.words, wpr, r.row_ptr, r.col_idx, r.vals, t2, h2,
                                   m2, a_scale=0.5, row_alpha=alpha)
    assert np.array_equal(g[:rows, :tokens], want2)
