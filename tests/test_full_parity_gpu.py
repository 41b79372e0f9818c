"""Every output cell at the BASELINE sizes against the unmodified reference (oracle/_ref).

The reference's own GEMM entry points (kernels.cpp:163-275), run with all host threads, give
the float32 result C = scale * float(units); with unit scales that float IS the integer
units, exactly (|units| < 2^24). The GPU units are compared with it cell for cell, tolerance
0 (acceptance.cpp:245-267, verify.cpp:261-287). The per-row / per-column scale epilogue of
config 3 has no reference counterpart (the reference takes scalars): its float output is
checked cell for cell against the documented operation order applied to those verified
units (s = scale * row[r]; s = s * col[c]; C = s * float(units)), and against the C oracle
on sampled rows in test_gemm_gpu.py. Config 4 (APB) is compared on all 3072 rows with the C
oracle (double accumulation as kernels.cpp:300-332), tolerance 1e-5 relative.
"""
import os

import numpy as np
import pytest

from paper_2306_08960_b200 import api, data

pytestmark = pytest.mark.gpu

THREADS = max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count())


def _T(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()


def _ref_units(out_f32):
    u = out_f32.astype(np.int32)
    assert np.array_equal(u.astype(np.float32), out_f32)  # integral, so unit-scale floats are units
    return u


def test_config1_1x1_4096_every_cell(ref):
    import torch
    from paper_2306_08960_b200 import device
    rng = np.random.default_rng(101)
    m = n = k = 4096
    a, wpr = data.random_words(rng, m, k)
    b, _ = data.random_words(rng, n, k)
    u = torch.empty((m, n), dtype=torch.int32, device="cuda")
    device.gemm_1x1(_T(a), _T(b), k, units=u)
    device.status()
    want = _ref_units(ref.gemm_1x1(a, b, k, wpr, threads=THREADS)[0])
    assert np.array_equal(u.cpu().numpy(), want)


def test_config2_2x2_4096_every_cell(ref):
    import torch
    from paper_2306_08960_b200 import device
    rng = np.random.default_rng(102)
    m = n = k = 4096
    wt, wh, wm, wpr = data.random_planes(rng, m, k)
    at, ah, am, _ = data.random_planes(rng, n, k)
    u = torch.empty((m, n), dtype=torch.int32, device="cuda")
    device.gemm_2x2(*(_T(x) for x in (wt, wh, wm, at, ah, am)), k, units=u)
    device.status()
    want = _ref_units(ref.gemm_2x2(wt, wh, wm, at, ah, am, k, wpr, threads=THREADS)[0])
    # the reference's scale is 0.25 * s_w * s_a (kernels.cpp:232): with unit plane scales its
    # float output is units / 4, exact
    assert np.array_equal(u.cpu().numpy(), (want.astype(np.float64) * 4).astype(np.int32))


def test_config3_1x2_every_cell_with_row_col_scales(ref):
    import torch
    from paper_2306_08960_b200 import device
    rng = np.random.default_rng(103)
    m, n, k = 4096, 8192, 4096  # binary weights on the rows, 8192 2-bit activations on the columns
    w, wpr = data.random_words(rng, m, k)
    t, h, mm, _ = data.random_planes(rng, n, k)
    gamma = rng.uniform(0.5, 1.5, m).astype(np.float32)
    beta = rng.uniform(0.5, 1.5, n).astype(np.float32)
    u = torch.empty((m, n), dtype=torch.int32, device="cuda")
    f = torch.empty((m, n), dtype=torch.float32, device="cuda")
    device.gemm_1x2(_T(w), 1.0, _T(t), _T(h), _T(mm), k, row_scale=torch.from_numpy(gamma).cuda(),
                    col_scale=torch.from_numpy(beta).cuda(), units=u, out=f)
    device.status()
    # reference half_scale = 0.5 (kernels.cpp:193): float output = units / 2, exact
    want = ref.gemm_1x2(w, 1.0, t, h, mm, k, wpr, threads=THREADS)[0]
    want_u = (want.astype(np.float64) * 2).astype(np.int32)
    got_u = u.cpu().numpy()
    assert np.array_equal(got_u, want_u)
    s = (np.float32(0.5) * gamma)[:, None]
    s = (s * beta[None, :]).astype(np.float32)
    assert np.array_equal(f.cpu().numpy(), (s * want_u.astype(np.float32)).astype(np.float32))


def test_config4_apb_every_row(orc):
    import torch
    from paper_2306_08960_b200 import device
    rng = np.random.default_rng(104)
    rows, cols, tokens = 3072, 768, 8192
    a, alpha, _ = data.apb_weights(rng, rows, cols)
    layer = api.decompose_apb(a, alpha)
    x = rng.standard_normal((cols, tokens)).astype(np.float32)
    r = layer.residual
    T = lambda v: torch.from_numpy(np.ascontiguousarray(v)).cuda()  # noqa: E731
    out = torch.empty((rows, tokens), dtype=torch.float32, device="cuda")
    device.layer_forward(T(layer.bin.words.view(np.int64)), cols, T(alpha), T(r.row_ptr.view(np.int64)),
                         T(r.col_idx.view(np.int64)), T(r.vals), T(x), out)
    device.status()
    want = orc.layer_forward(rows, cols, 1.0, layer.bin.words, layer.bin.words_per_row(), r.row_ptr,
                             r.col_idx, r.vals, x, row_alpha=alpha).astype(np.float64)
    got = out.cpu().numpy().astype(np.float64)
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert rel <= 1e-5, rel  # tolerance 1e-5 relative Frobenius (BASELINE config 4)
    assert np.max(np.abs(got - want)) <= 1e-5 * np.max(np.abs(want))


def test_config5_1x1_32768_every_cell(ref):
    """32768^3 (the N-shard sweep's problem at N=1): every cell against the reference, in row
    blocks so the host holds one block of the reference's output at a time."""
    import torch
    from paper_2306_08960_b200 import device
    rng = np.random.default_rng(105)
    m = n = k = 32768
    a, wpr = data.random_words(rng, m, k)
    b, _ = data.random_words(rng, n, k)
    u = torch.empty((m, n), dtype=torch.int32, device="cuda")
    device.gemm_1x1(_T(a), _T(b), k, units=u)
    device.status()
    blk = 4096
    for r0 in range(0, m, blk):
        want = _ref_units(ref.gemm_1x1(a[r0:r0 + blk], b, k, wpr, threads=THREADS)[0])
        assert np.array_equal(u[r0:r0 + blk].cpu().numpy(), want), r0
    del u
    torch.cuda.empty_cache()


@pytest.mark.parametrize("k", [1 << 20, (1 << 20) - 77])
def test_random_levels_at_max_shared_dim(orc, k):
    """Mixed random data at K = 2^20: 1/2 and 2/2 against the C oracle cell for cell (the
    all-level-3 case in test_gemm_gpu.py pins the extreme magnitudes)."""
    import torch
    from paper_2306_08960_b200 import device
    rng = np.random.default_rng(k)
    m, n = 16, 64
    w, wpr = data.random_words(rng, m, k)
    wt, wh, wm, _ = data.random_planes(rng, m, k)
    at, ah, am, _ = data.random_planes(rng, n, k)
    u12 = torch.empty((m, n), dtype=torch.int32, device="cuda")
    u22 = torch.empty((m, n), dtype=torch.int32, device="cuda")
    device.gemm_1x2(_T(w), 1.0, _T(at), _T(ah), _T(am), k, units=u12)
    device.gemm_2x2(*(_T(x) for x in (wt, wh, wm, at, ah, am)), k, units=u22)
    device.status()
    assert np.array_equal(u12.cpu().numpy(), orc.gemm_1x2(w, 1.0, at, ah, am, k, wpr)[0])
    assert np.array_equal(u22.cpu().numpy(), orc.gemm_2x2(wt, wh, wm, at, ah, am, k, wpr)[0])
