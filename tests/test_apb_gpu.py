"""GPU parity for the APB layer forward (apb.cpp:158-164), its binary part gemm_1x32_ref
(kernels.cpp:300-332) and spmm_csr (kernels.cpp:334-352).

Tolerance (BASELINE.json north star): fp32 outputs within 1e-5 relative Frobenius error of
the reference's double-accumulated result; the max-abs error is asserted alongside with
a bound of 1e-5 * max|C|. The standalone SpMM evaluates the reference's exact fp32
operation order and is compared bit-exactly."""
import numpy as np
import pytest

from conftest import apb_case
from paper_2306_08960_b200 import api, data

pytestmark = pytest.mark.gpu

REL_TOL = 1e-5


def rel_frob(got, want):
    want = want.astype(np.float64)
    num = np.linalg.norm(got.astype(np.float64) - want)
    den = np.linalg.norm(want)
    return num if den == 0 else num / den


def check_close(got, want):
    rel = rel_frob(got, want)
    max_abs = float(np.max(np.abs(got.astype(np.float64) - want))) if got.size else 0.0
    bound = REL_TOL * float(np.max(np.abs(want))) if want.size else 0.0
    assert rel <= REL_TOL, (rel, max_abs)
    assert max_abs <= max(bound, 1e-30), (rel, max_abs, bound)
    return rel, max_abs


def _layer(c):
    m, k, wpr = c["m"], c["k"], c["wpr"]
    bin_ = api.BitMatrix.from_words(m, k, wpr, c["bin"])
    res = api.CsrMatrix.create(m, k, c["row_ptr"], c["col_idx"], c["vals"])
    alpha = c["alpha_vec"] if "alpha_vec" in c else float(c["alpha_delta"][0])
    return api.ApbLayer(m, k, alpha, bin_, res)


def test_golden_layer_forward(apb_golden):
    for i in range(int(apb_golden["apb_count"])):
        c = apb_case(apb_golden, i)
        layer = _layer(c)
        check_close(api.layer_forward(layer, c["b"]), c["c"])
        if "c1x32" in c:
            check_close(api.gemm_1x32_ref(layer.bin, layer.alpha, c["b"]), c["c1x32"])
            assert np.array_equal(api.spmm_csr(layer.residual, c["b"]), c["cspmm"])


def test_frozen_1x32_and_spmm():
    # test_kernels.cpp:216-220, 235-243
    w = api.pack_signs(np.array([[1.0, -1.0, 1.0]], np.float32))
    assert api.gemm_1x32_ref(w, 2.0, np.array([[1.0], [2.0], [3.0]], np.float32))[0, 0] == 4.0
    a = api.CsrMatrix.create(2, 2, [0, 1, 2], [1, 0], [5.0, 1.0])
    c = api.spmm_csr(a, np.array([[1.0, 2.0], [3.0, 4.0]], np.float32))
    assert np.array_equal(c, np.array([[15.0, 20.0], [1.0, 2.0]], np.float32))
    with pytest.raises(ValueError):
        api.spmm_csr(a, np.zeros((3, 1), np.float32))


def test_decompose_then_forward_matches_dense(orc):
    # test_apb.cpp:181-197 / acceptance.cpp:335-387 pattern on random layers
    rng = np.random.default_rng(7)
    worst = 0.0
    for _ in range(20):
        m, k, n = int(rng.integers(1, 128)), int(rng.integers(1, 512)), int(rng.integers(1, 300))
        w = rng.uniform(-2, 2, (m, k)).astype(np.float32)
        alpha, delta = float(rng.uniform(0.2, 1.0)), float(rng.uniform(0.05, 0.5))
        fwd = orc.apb_forward(w, alpha, delta)
        layer = api.decompose_apb(fwd, alpha)
        b = rng.uniform(-1, 1, (k, n)).astype(np.float32)
        got = api.layer_forward(layer, b)
        bw, wpr, rp, ci, v = orc.decompose_apb(fwd, alpha)
        want = orc.layer_forward(m, k, alpha, bw, wpr, rp, ci, v, b)
        rel, _ = check_close(got, want)
        worst = max(worst, rel)
        dense = fwd.astype(np.float64) @ b.astype(np.float64)
        assert rel_frob(got, dense) <= 1e-4  # the reference's own bound vs the dense product


def test_config4_full_size_sampled(orc):
    """BASELINE config 4: out N=3072, K=768, tokens 8192, per-row alpha, top-2% residual."""
    import torch
    from paper_2306_08960_b200 import device
    rng = np.random.default_rng(4)
    rows, cols, tokens = 3072, 768, 8192
    a, alpha, keep = data.apb_weights(rng, rows, cols)
    layer = api.decompose_apb(a, alpha)
    x = rng.standard_normal((cols, tokens)).astype(np.float32)
    r = layer.residual
    T = lambda v: torch.from_numpy(v).cuda()  # noqa: E731
    out = torch.empty((rows, tokens), dtype=torch.float32, device="cuda")
    device.layer_forward(T(layer.bin.words.view(np.int64)), cols, T(alpha), T(r.row_ptr.view(np.int64)),
                         T(r.col_idx.view(np.int64)), T(r.vals), T(x), out)
    device.status()
    got = out.cpu().numpy()
    sample = np.sort(rng.choice(rows, 48, replace=False))
    rp = r.row_ptr
    sub_rp = [0]
    ci, vv = [], []
    for s in sample:
        lo, hi = int(rp[s]), int(rp[s + 1])
        ci.append(r.col_idx[lo:hi])
        vv.append(r.vals[lo:hi])
        sub_rp.append(sub_rp[-1] + hi - lo)
    want = orc.layer_forward(len(sample), cols, 1.0, layer.bin.words[sample], layer.bin.words_per_row(),
                             np.asarray(sub_rp, np.uint64), np.concatenate(ci).astype(np.uint64),
                             np.concatenate(vv).astype(np.float32), x, row_alpha=alpha[sample])
    check_close(got[sample], want)
    assert int(r.nnz()) == rows * keep or int(r.nnz()) >= rows * keep  # exact-|alpha| ties aside


def test_spmm_bit_exact_random(orc):
    rng = np.random.default_rng(13)
    for (rows, cols, n, dens) in [(50, 70, 33, 0.1), (300, 768, 1000, 0.02), (7, 5, 300, 0.5)]:
        mask = rng.random((rows, cols)) < dens
        vals = rng.uniform(-1, 1, (rows, cols)).astype(np.float32)
        r_idx, c_idx = np.nonzero(mask)
        rp = np.zeros(rows + 1, np.uint64)
        rp[1:] = np.cumsum(np.bincount(r_idx, minlength=rows))
        csr = api.CsrMatrix.create(rows, cols, rp, c_idx.astype(np.uint64), vals[mask])
        b = rng.standard_normal((cols, n)).astype(np.float32)
        got = api.spmm_csr(csr, b)
        want = orc.spmm_csr(rows, csr.row_ptr, csr.col_idx, csr.vals, b)
        assert np.array_equal(got, want)


def test_layer_forward_empty_residual_and_odd_shapes(orc):
    rng = np.random.default_rng(21)
    for (m, k, n) in [(1, 1, 1), (3, 65, 5), (129, 64, 257), (130, 130, 3)]:
        w = rng.standard_normal((m, k)).astype(np.float32)
        alpha = 0.5
        fwd = np.where(w >= 0, alpha, -alpha).astype(np.float32)  # fully binarized: nnz = 0
        layer = api.decompose_apb(fwd, alpha)
        assert layer.residual.nnz() == 0
        b = rng.standard_normal((k, n)).astype(np.float32)
        got = api.layer_forward(layer, b)
        want = orc.gemm_1x32(layer.bin.words, k, layer.bin.words_per_row(), alpha, b)
        check_close(got, want)


@pytest.mark.parametrize("fold", ["same-stage", "sep"])
@pytest.mark.parametrize("k", [900, 1000, 4096])
def test_large_k_layer_forward(orc, k, fold, monkeypatch):
    """K past the one-pass X split (x_token_scale + split_x_f16) and K=4096, where split
    accumulators keep the tensor-core fp32 accumulation within tolerance. Both placements of
    the folded residual's W'_lo . X_hi products: in the main K loop's stages (default) and as
    a separate phase after it (BITMM_APB_FOLD=sep)."""
    if fold == "sep":
        monkeypatch.setenv("BITMM_APB_FOLD", "sep")
    else:
        monkeypatch.delenv("BITMM_APB_FOLD", raising=False)
    rng = np.random.default_rng(k)
    rows, tokens = 96, 200
    a, alpha, _ = data.apb_weights(rng, rows, k)
    layer = api.decompose_apb(a, alpha)
    x = rng.standard_normal((k, tokens)).astype(np.float32)
    got = api.layer_forward(layer, x)
    r = layer.residual
    want = orc.layer_forward(rows, k, 1.0, layer.bin.words, layer.bin.words_per_row(), r.row_ptr,
                             r.col_idx, r.vals, x, row_alpha=alpha)
    check_close(got, want)


@pytest.mark.parametrize("v1", ["0", "1"])
def test_spmm_exact_odd_shapes(orc, monkeypatch, v1):
    # ragged columns (N % 4 != 0), empty rows, rows with > 8 nonzeros, single column, K past the
    # 64-token kernel's shared memory (1000) — through the 64-token persistent kernel and the
    # 32-token chunk kernel (BITMM_SPMM_V1=1)
    monkeypatch.setenv("BITMM_SPMM_V1", v1)
    rng = np.random.default_rng(99)
    for (rows, cols, n) in [(5, 3, 1), (33, 700, 37), (7, 64, 130), (300, 50, 33), (70, 1000, 200),
                            (129, 864, 64)]:
        dens = rng.uniform(0.0, 0.6)
        mask = rng.random((rows, cols)) < dens
        mask[0] = False  # an empty row
        vals = rng.standard_normal((rows, cols)).astype(np.float32)
        r_idx, c_idx = np.nonzero(mask)
        rp = np.zeros(rows + 1, np.uint64)
        rp[1:] = np.cumsum(np.bincount(r_idx, minlength=rows))
        csr = api.CsrMatrix.create(rows, cols, rp, c_idx.astype(np.uint64), vals[mask])
        b = rng.standard_normal((cols, n)).astype(np.float32)
        assert np.array_equal(api.spmm_csr(csr, b), orc.spmm_csr(rows, csr.row_ptr, csr.col_idx,
                                                                 csr.vals, b))


def test_token_magnitude_range(orc):
    """The fp16 split scales every token by a power of two before splitting: tokens spanning
    1e-30 .. 1e30 (beyond fp16's range either way), an all-zero token, and a token with one
    large outlier keep the 1e-5 tolerance column by column."""
    rng = np.random.default_rng(5)
    rows, k, tokens = 64, 300, 9
    a, alpha, _ = data.apb_weights(rng, rows, k)
    layer = api.decompose_apb(a, alpha)
    x = rng.standard_normal((k, tokens)).astype(np.float32)
    scales = np.array([1e-30, 1e-12, 1e-4, 1.0, 7e4, 1e12, 1e30, 0.0, 1.0], np.float32)
    x *= scales[None, :]
    x[17, 8] = 3e5  # one outlier in an otherwise unit-scale token
    got = api.layer_forward(layer, x)
    r = layer.residual
    want = orc.layer_forward(rows, k, 1.0, layer.bin.words, layer.bin.words_per_row(), r.row_ptr,
                             r.col_idx, r.vals, x, row_alpha=alpha)
    assert np.all(got[:, 7] == 0.0)
    for j in range(tokens):
        if j != 7:
            check_close(got[:, j], want[:, j])


def test_folded_residual_edge_rows(orc):
    """layer_forward folds the residual into the fp16 operand as W' = s + v/alpha_r
    (apb_fold_kernel). Rows that cannot take that form use m_r = max(|alpha_r|, max|v|):
    alpha_r = 0, an alpha_r far below the residual (v/alpha_r past fp16), a negative alpha_r.
    Also a row with a repeated column (spmm_csr sums both), a row with more than 32 nonzeros
    (the warp's lanes loop), and an empty row."""
    rng = np.random.default_rng(404)
    m, k, n = 12, 200, 77
    wpr = (k + 511) // 512 * 8
    signs = rng.random((m, k)) < 0.5
    words = np.zeros((m, wpr), np.uint64)
    for r in range(m):
        for c in np.nonzero(signs[r])[0]:
            words[r, c // 64] |= np.uint64(1) << np.uint64(c % 64)
    alpha = rng.uniform(0.01, 0.03, m).astype(np.float32)
    alpha[0] = 0.0
    alpha[1] = 1e-9
    alpha[2] = -0.02
    rows_c, rows_v = [], []
    for r in range(m):
        nnz = {5: 0, 6: 60}.get(r, 4)
        cols = np.sort(rng.choice(k, nnz, replace=False)).astype(np.uint64)
        rows_c.append(cols)
        rows_v.append((rng.standard_normal(len(cols)) * 0.05).astype(np.float32))
    rp = np.zeros(m + 1, np.uint64)
    rp[1:] = np.cumsum([len(c) for c in rows_c])
    ci, vv = np.concatenate(rows_c), np.concatenate(rows_v)
    layer = api.ApbLayer(m, k, alpha, api.BitMatrix.from_words(m, k, wpr, words),
                         api.CsrMatrix.create(m, k, rp, ci, vv))
    x = rng.standard_normal((k, n)).astype(np.float32)
    got = api.layer_forward(layer, x)
    want = orc.layer_forward(m, k, 1.0, words, wpr, rp, ci, vv, x, row_alpha=alpha)
    for r in range(m):
        check_close(got[r], want[r])
    # a repeated column (only the device-pointer entry point accepts one; the host flavour
    # validates strictly increasing columns like CsrMatrix::validate): both entries count
    import torch
    from paper_2306_08960_b200 import device
    rows_c[3] = np.array([10, 10, 50, 199, 10], np.uint64)
    rows_v[3] = np.array([0.05, -0.02, 0.01, 0.03, 0.04], np.float32)
    rp[1:] = np.cumsum([len(c) for c in rows_c])
    ci, vv = np.concatenate(rows_c), np.concatenate(rows_v)
    T = lambda v: torch.from_numpy(np.ascontiguousarray(v)).cuda()  # noqa: E731
    out = torch.empty((m, n), dtype=torch.float32, device="cuda")
    device.layer_forward(T(words.view(np.int64)), k, T(alpha), T(rp.view(np.int64)),
                         T(ci.view(np.int64)), T(vv), T(x), out)
    device.status()
    want = orc.layer_forward(m, k, 1.0, words, wpr, rp, ci, vv, x, row_alpha=alpha)
    got = out.cpu().numpy()
    for r in range(m):
        check_close(got[r], want[r])
