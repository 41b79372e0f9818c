"""APB with 2-bit activations.

The layer is the composition of reference calls gemm_1x2(bin, alpha, planes) +
spmm_csr(residual, dequant(planes)) added as layer_forward adds (apb.cpp:161-162).
CPU: the oracle restatement is pinned against that composition run on the UNMODIFIED
reference library (oracle/_ref). GPU: the CUDA path is bit-identical to the oracle.
"""
import numpy as np
import pytest

from paper_2306_08960_b200 import api, data


def _layer(rng, rows, cols, keep_frac=0.02, lane=512):
    """The layer from the oracle's decompose_apb (apb.cpp:119-142), so the CPU tests need no GPU."""
    import oracle
    a, alpha, _ = data.apb_weights(rng, rows, cols, keep_frac=keep_frac)
    bw, wpr, rp, ci, v = oracle.Oracle().decompose_apb(a, alpha, lane)
    layer = api.ApbLayer(rows, cols, alpha, api.BitMatrix.from_words(rows, cols, wpr, bw),
                         api.CsrMatrix.create(rows, cols, rp, ci, v))
    return layer, alpha


def _planes(rng, tokens, cols, lane=512):
    t, h, m, wpr = data.random_planes(rng, tokens, cols, lane)
    return t, h, m, wpr


def _thm(t, h, m, cols, s=1.0, g=None):
    rows, wpr = t.shape
    bm = lambda w: api.BitMatrix.from_words(rows, cols, wpr, w)  # noqa: E731
    return api.ThmPlanes(bm(t), bm(h), bm(m), scale=s, gamma=g)


def _ref_composition(ref, layer, alpha_rows, t, h, m, s, g):
    """gemm_1x2 per row (alpha_r as gamma) + spmm_csr over the dequantized planes."""
    k, wpr = layer.cols, layer.bin.words_per_row()
    tokens = t.shape[0]
    bin_part = np.empty((layer.rows, tokens), np.float32)
    for r in range(layer.rows):
        o, _ = ref.gemm_1x2(layer.bin.words[r:r + 1], float(alpha_rows[r]), t, h, m, k, wpr,
                            a_scale=s, a_gamma=g)
        bin_part[r] = o[0]
    lv = data.levels_from_planes(t, h, m, k).astype(np.float32)  # tokens x k
    sg = np.float32(np.float32(s) * np.float32(1.0 if g is None else g))
    d = np.ascontiguousarray((lv * sg).T.astype(np.float32))    # k x tokens
    rr = layer.residual
    res, _ = ref.spmm_csr(layer.rows, k, rr.row_ptr, rr.col_idx, rr.vals, d)
    return (bin_part + res).astype(np.float32)


@pytest.mark.parametrize("rows,cols,tokens,g", [(40, 96, 33, None), (17, 600, 70, 0.75),
                                                 (64, 1100, 9, None)])
def test_oracle_pinned_to_reference_composition(orc, ref, rows, cols, tokens, g):
    rng = np.random.default_rng(rows + cols)
    layer, alpha = _layer(rng, rows, cols)
    t, h, m, wpr = _planes(rng, tokens, cols)
    s = 0.37
    rr = layer.residual
    want = _ref_composition(ref, layer, alpha, t, h, m, s, g)
    got = orc.layer_forward_2bit(rows, cols, 1.0, layer.bin.words, wpr, rr.row_ptr, rr.col_idx,
                                 rr.vals, t, h, m, a_scale=s, a_gamma=g, row_alpha=alpha)
    assert np.array_equal(got, want)
    # scalar alpha follows the same path
    got_s = orc.layer_forward_2bit(rows, cols, float(alpha[0]), layer.bin.words, wpr, rr.row_ptr,
                                   rr.col_idx, rr.vals, t, h, m, a_scale=s, a_gamma=g)
    want_s = _ref_composition(ref, layer, np.full(rows, alpha[0], np.float32), t, h, m, s, g)
    assert np.array_equal(got_s, want_s)


# ------------------------------------------------------------------ GPU
def _gpu_vs_oracle(orc, rows, cols, tokens, lane=512, g=None, keep_frac=0.02, per_row=True, seed=0):
    rng = np.random.default_rng(seed + rows * 7 + cols)
    layer, alpha = _layer(rng, rows, cols, keep_frac=keep_frac, lane=lane)
    t, h, m, wpr = _planes(rng, tokens, cols, lane)
    s = 0.125 + rng.random()
    if not per_row:
        layer.alpha = float(alpha[0])
    planes = _thm(t, h, m, cols, s, g)
    got = api.layer_forward_2bit(layer, planes)
    rr = layer.residual
    want = orc.layer_forward_2bit(rows, cols, 1.0 if per_row else float(alpha[0]), layer.bin.words,
                                  wpr, rr.row_ptr, rr.col_idx, rr.vals, t, h, m, a_scale=s,
                                  a_gamma=g, row_alpha=alpha if per_row else None)
    assert np.array_equal(got, want), np.max(np.abs(got - want))
    return got


@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols,tokens", [(1, 1, 1), (300, 768, 333), (256, 256, 256),
                                              (513, 130, 1000), (64, 5000, 70)])
def test_gpu_bit_exact(orc, rows, cols, tokens):
    _gpu_vs_oracle(orc, rows, cols, tokens)


@pytest.mark.gpu
def test_gpu_scalar_alpha_gamma_lane64(orc):
    _gpu_vs_oracle(orc, 200, 700, 150, lane=64, g=0.5, per_row=False)


@pytest.mark.gpu
def test_gpu_empty_residual(orc):
    # keep_frac -> 1 kept weight per row minimum; also a layer with no residual at all
    rng = np.random.default_rng(5)
    rows, cols, tokens = 128, 256, 96
    alpha = np.float32(0.5)
    a = np.where(rng.random((rows, cols)) < 0.5, alpha, -alpha).astype(np.float32)
    layer = api.decompose_apb(a, float(alpha))
    assert layer.residual.nnz() == 0
    t, h, m, wpr = _planes(rng, tokens, cols)
    planes = _thm(t, h, m, cols)
    got = api.layer_forward_2bit(layer, planes)
    rr = layer.residual
    want = orc.layer_forward_2bit(rows, cols, float(alpha), layer.bin.words, wpr, rr.row_ptr,
                                  rr.col_idx, rr.vals, t, h, m)
    assert np.array_equal(got, want)


@pytest.mark.gpu
def test_gpu_illegal_planes_raise(orc):
    rng = np.random.default_rng(6)
    layer, _ = _layer(rng, 32, 128)
    t, h, m, wpr = _planes(rng, 16, 128)
    h = h.copy()
    h[3, 0] |= t[3, 0] | 1  # t and h both set -> illegal state
    t = t.copy()
    t[3, 0] |= 1
    planes = _thm(t, h, m, 128)
    with pytest.raises(api.InvalidEncoding):
        api.layer_forward_2bit(layer, planes)
    # the C ABI latches the same error from the device-side plane check
    import ctypes as C
    from paper_2306_08960_b200 import _lib
    P = lambda x: x.ctypes.data_as(C.c_void_p)  # noqa: E731
    rr = layer.residual
    out = np.empty((32, 16), np.float32)
    rc = _lib.load().bitmm_layer_forward_2bit_host(
        32, 128, 1.0, None, P(layer.bin.words), wpr, P(rr.row_ptr), P(rr.col_idx), P(rr.vals),
        rr.nnz(), P(t), P(h), P(m), 16, 1.0, 0, 1.0, P(out), 16)
    assert rc == _lib.ERR_INVALID_ENCODING


@pytest.mark.gpu
def test_gpu_device_path_config4_shape(orc):
    """Config-4 shape (3072 x 768, 8192 tokens) through the device entry point, rows sampled."""
    import torch
    from paper_2306_08960_b200 import device
    rng = np.random.default_rng(44)
    rows, cols, tokens = 3072, 768, 8192
    layer, alpha = _layer(rng, rows, cols)
    t, h, m, wpr = _planes(rng, tokens, cols)
    T = lambda v: torch.from_numpy(np.ascontiguousarray(v)).cuda()  # noqa: E731
    rr = layer.residual
    out = torch.empty((rows, tokens), dtype=torch.float32, device="cuda")
    device.layer_forward_2bit(T(layer.bin.words.view(np.int64)), cols, T(alpha),
                              T(rr.row_ptr.view(np.int64)), T(rr.col_idx.view(np.int64)), T(rr.vals),
                              T(t.view(np.int64)), T(h.view(np.int64)), T(m.view(np.int64)), out,
                              a_scale=0.5)
    device.status()
    got = out.cpu().numpy()
    sample = np.sort(rng.choice(rows, 24, replace=False))
    rp = rr.row_ptr
    sub_rp, ci, vv = [0], [], []
    for r in sample:
        lo, hi = int(rp[r]), int(rp[r + 1])
        ci.append(rr.col_idx[lo:hi])
        vv.append(rr.vals[lo:hi])
        sub_rp.append(sub_rp[-1] + hi - lo)
    want = orc.layer_forward_2bit(len(sample), cols, 1.0, layer.bin.words[sample], wpr,
                                  np.asarray(sub_rp, np.uint64), np.concatenate(ci).astype(np.uint64),
                                  np.concatenate(vv).astype(np.float32), t, h, m, a_scale=0.5,
                                  row_alpha=alpha[sample])
    assert np.array_equal(got[sample], want)


@pytest.mark.gpu
@pytest.mark.parametrize("g", [1e-39, 3.0e36])
def test_gpu_fused_extreme_scales(orc, monkeypatch, g):
    """The fused layer's L8 chunks rebuild d = fl(p * s * g) as fma(p + 4, sg, -4 sg): exact also
    when sg is subnormal (g = 1e-39) or large (4 sg near the top of the fp32 range)."""
    monkeypatch.setenv("BITMM_APB2_FUSED", "1")
    _gpu_vs_oracle(orc, 300, 768, 200, g=g, seed=5)


@pytest.mark.gpu
@pytest.mark.parametrize("form", ["fused", "fused-bf16", "two-pass", "two-pass-fp32"])
@pytest.mark.parametrize("rows,cols,tokens", [(300, 768, 332), (513, 130, 1000), (257, 973, 64), (33, 974, 8),
                                              (64, 1100, 68), (1000, 256, 4)])
def test_gpu_every_form_bit_exact(orc, monkeypatch, form, rows, cols, tokens):
    """The device forms of the layer — residual fused into the GEMM epilogue
    (apb2_fused_kernel, with L8 or bf16 level chunks), GEMM then the bf16-level SpMM (spmm_levels_kernel), GEMM then the
    fp32-level SpMM (spmm_xchunk_kernel<LEVELS>) — each bit-identical to the oracle, at shapes
    with ragged row blocks, token blocks and K (cols 1100 exceeds the fused kernel's shared
    memory and falls back to the two-pass form)."""
    from paper_2306_08960_b200 import _lib
    lib = _lib.load()
    monkeypatch.setenv("BITMM_APB2_FUSED", "1" if form.startswith("fused") else "0")
    monkeypatch.setenv("BITMM_APB2_L8", "0" if form == "fused-bf16" else "1")
    monkeypatch.setenv("BITMM_SPMM_LEVELS_V1", "1" if form == "two-pass-fp32" else "0")
    lib.bitmm_profile_reset()
    lib.bitmm_profile_enable(1)
    try:
        _gpu_vs_oracle(orc, rows, cols, tokens, seed=3)
        assert lib.bitmm_profile_collect() == 0
        ran = {lib.bitmm_profile_kernel_name(i).decode() for i in range(lib.bitmm_profile_kernel_count())
               if lib.bitmm_profile_kernel_launches(i) > 0}
    finally:
        lib.bitmm_profile_enable(0)
        lib.bitmm_profile_reset()
    # the form the switches and the shape select is the one that ran
    if form.startswith("fused") and cols <= 973:
        assert "apb2_fused" in ran, ran
    elif form == "two-pass-fp32":
        assert "apb2_fused" not in ran and "spmm_levels" not in ran, ran
    else:
        assert "apb2_fused" not in ran and "spmm_levels" in ran, ran


@pytest.mark.gpu
def test_gpu_fused_repeated_and_concurrent(orc):
    """The fused kernel's pipeline (TMA/MMA/epilogue/residual handshakes, level reloads at token
    block changes) under repetition and concurrency: two host threads on two streams run layers of
    different shapes 40 times each; every result must equal the oracle's bit for bit."""
    import threading

    import torch
    from paper_2306_08960_b200 import device
    shapes = [(300, 768, 332), (1000, 960, 1000)]
    cases = []
    for i, (rows, cols, tokens) in enumerate(shapes):
        rng = np.random.default_rng(100 + i)
        layer, alpha = _layer(rng, rows, cols)
        t, h, m, wpr = _planes(rng, tokens, cols)
        rr = layer.residual
        want = orc.layer_forward_2bit(rows, cols, 1.0, layer.bin.words, wpr, rr.row_ptr, rr.col_idx, rr.vals,
                                      t, h, m, a_scale=0.75, row_alpha=alpha)
        T = lambda v: torch.from_numpy(np.ascontiguousarray(v)).cuda()  # noqa: E731
        d = [T(layer.bin.words.view(np.int64)), T(alpha), T(rr.row_ptr.view(np.int64)),
             T(rr.col_idx.view(np.int64)), T(rr.vals), T(t.view(np.int64)), T(h.view(np.int64)),
             T(m.view(np.int64))]
        cases.append((rows, cols, tokens, d, want))
    errors = []

    def worker(ci):
        rows, cols, tokens, d, want = cases[ci]
        stream = torch.cuda.Stream()
        try:
            with torch.cuda.stream(stream):
                out = torch.empty((rows, tokens), dtype=torch.float32, device="cuda")
                for _ in range(40):
                    out.fill_(float("nan"))
                    device.layer_forward_2bit(d[0], cols, d[1], d[2], d[3], d[4], d[5], d[6], d[7], out,
                                              a_scale=0.75, stream=stream)
                    device.status(stream)
                    if not np.array_equal(out.cpu().numpy(), want):
                        errors.append(ci)
                        return
        except Exception as e:  # pragma: no cover
            errors.append((ci, repr(e)))

    threads = [threading.Thread(target=worker, args=(i,)) for i in range(len(cases))]
    for th in threads:
        th.start()
    for th in threads:
        th.join(timeout=600)
    assert not any(th.is_alive() for th in threads), "a worker hung"
    assert not errors, errors
