"""GEMM group (bitmm_gemm_batch_dev): several routines in one expansion launch plus one
persistent tensor-core launch must give results bit-identical to the per-routine calls
(gemm_1x1 kernels.cpp:163-183, gemm_1x2 :185-221, gemm_2x2 :223-275) and to the oracle."""
import numpy as np
import pytest

from paper_2306_08960_b200 import api, data

pytestmark = pytest.mark.gpu


def _T(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()


def _case(rng, m, n, n2, k):
    a, wpr = data.random_words(rng, m, k)
    b, _ = data.random_words(rng, n, k)
    t, h, mm, _ = data.random_planes(rng, n2, k)
    wt, wh, wm, _ = data.random_planes(rng, m, k)
    return dict(a=a, b=b, t=t, h=h, mm=mm, wt=wt, wh=wh, wm=wm, wpr=wpr)


@pytest.mark.parametrize("m,n,n2,k", [(4096, 4096, 8192, 4096), (300, 517, 1000, 777), (1, 1, 1, 1)])
@pytest.mark.parametrize("balance", ["0", "1"])
def test_batch_matches_single_calls(orc, monkeypatch, m, n, n2, k, balance):
    """balance "1": the GEMM walks the balanced piece schedule (BITMM_TC_BALANCE=1: contiguous
    column stretches per CTA pair, pieces narrower than the tile with the MMA's N per piece)."""
    monkeypatch.setenv("BITMM_TC_BALANCE", balance)
    import torch
    from paper_2306_08960_b200 import device
    rng = np.random.default_rng(m + n + k)
    c = _case(rng, m, n, n2, k)
    rs = torch.rand(m, device="cuda") + 0.5
    cs = torch.rand(n2, device="cuda") + 0.5
    da, db, dt, dh, dm = _T(c["a"]), _T(c["b"]), _T(c["t"]), _T(c["h"]), _T(c["mm"])
    dwt, dwh, dwm = _T(c["wt"]), _T(c["wh"]), _T(c["wm"])
    u11 = torch.empty((m, n), dtype=torch.int32, device="cuda")
    f12 = torch.empty((m, n2), dtype=torch.float32, device="cuda")
    u22 = torch.empty((m, n2), dtype=torch.int32, device="cuda")
    device.gemm_batch([
        dict(routine="1x1", a=da, b=db, k=k, units=u11),
        dict(routine="1x2", w=da, t=dt, h=dh, m=dm, k=k, gamma=0.75, a_scale=0.5, a_gamma=1.5,
             row_scale=rs, col_scale=cs, out=f12),
        dict(routine="2x2", wt=dwt, wh=dwh, wm=dwm, t=dt, h=dh, m=dm, k=k, units=u22),
    ])
    device.status()
    r11 = torch.empty_like(u11)
    r12 = torch.empty_like(f12)
    r22 = torch.empty_like(u22)
    device.gemm_1x1(da, db, k, units=r11)
    device.gemm_1x2(da, 0.75, dt, dh, dm, k, a_scale=0.5, a_gamma=1.5, row_scale=rs, col_scale=cs,
                    out=r12)
    device.gemm_2x2(dwt, dwh, dwm, dt, dh, dm, k, units=r22)
    device.status()
    assert torch.equal(u11, r11) and torch.equal(f12, r12) and torch.equal(u22, r22)
    rows = np.unique(np.concatenate([[0, m - 1], rng.choice(m, min(m, 6))]))
    want11, _ = orc.gemm_1x1(c["a"][rows], c["b"], k, c["wpr"])
    assert np.array_equal(u11.cpu().numpy()[rows], want11)
    want22, _ = orc.gemm_2x2(c["wt"][rows], c["wh"][rows], c["wm"][rows], c["t"], c["h"], c["mm"],
                             k, c["wpr"])
    assert np.array_equal(u22.cpu().numpy()[rows], want22)


def test_batch_both_outputs_and_mixed_k(orc):
    import torch
    from paper_2306_08960_b200 import device
    rng = np.random.default_rng(9)
    c1 = _case(rng, 260, 300, 10, 2000)
    c2 = _case(rng, 129, 70, 33, 65)
    u1 = torch.empty((260, 300), dtype=torch.int32, device="cuda")
    f1 = torch.empty((260, 300), dtype=torch.float32, device="cuda")
    u2 = torch.empty((129, 33), dtype=torch.int32, device="cuda")
    device.gemm_batch([
        dict(routine="1x1", a=_T(c1["a"]), b=_T(c1["b"]), k=2000, gamma_a=0.5, gamma_b=3.0,
             units=u1, out=f1),
        dict(routine="1x2", w=_T(c2["a"]), t=_T(c2["t"]), h=_T(c2["h"]), m=_T(c2["mm"]), k=65,
             units=u2),
    ])
    device.status()
    want_u, want_f = orc.gemm_1x1(c1["a"], c1["b"], 2000, c1["wpr"], 0.5, 3.0)
    assert np.array_equal(u1.cpu().numpy(), want_u)
    assert np.array_equal(f1.cpu().numpy(), want_f)
    want2, _ = orc.gemm_1x2(c2["a"], 1.0, c2["t"], c2["h"], c2["mm"], 65, c2["wpr"])
    assert np.array_equal(u2.cpu().numpy(), want2)


def test_batch_errors():
    import torch
    from paper_2306_08960_b200 import device
    rng = np.random.default_rng(2)
    c = _case(rng, 8, 8, 8, 64)
    u = torch.empty((8, 8), dtype=torch.int32, device="cuda")
    f = torch.empty((8, 8), dtype=torch.float32, device="cuda")
    item = dict(routine="1x1", a=_T(c["a"]), b=_T(c["b"]), k=64, units=u, out=f)
    with pytest.raises(ValueError):
        device.gemm_batch([])
    with pytest.raises(ValueError):  # 6 outputs > 4
        device.gemm_batch([item, item, item])
    with pytest.raises(api.InvalidEncoding):
        device.gemm_batch([dict(routine="1x2", w=_T(c["a"]), t=_T(c["t"]), h=_T(c["h"]),
                                m=_T(c["mm"]), k=64, a_scale=0.0, units=u)])
    bad = c["t"].copy()
    bad[0, 0] |= c["h"][0, 0] | 1
    hb = c["h"].copy()
    hb[0, 0] |= 1
    device.gemm_batch([dict(routine="2x2", wt=_T(c["wt"]), wh=_T(c["wh"]), wm=_T(c["wm"]),
                            t=_T(bad), h=_T(hb), m=_T(c["mm"]), k=64, units=u)])
    with pytest.raises(api.InvalidEncoding):
        device.status()
