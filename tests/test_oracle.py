"""CPU: pin the C restatement (oracle/bitmm_oracle.c) before trusting it.

* against the reference's frozen known-answer cases (test_kernels.cpp:41-143),
* against golden outputs of the unmodified reference (tests/golden/, make_golden.py),
* against the live reference library when it is built here (oracle/_ref).
"""
import numpy as np
import pytest

from conftest import apb_case, gemm_case
from paper_2306_08960_b200 import data


def _planes(levels, lane=512):
    return data.planes_from_levels(np.asarray(levels, np.uint8).reshape(1, -1), lane)


# ---------------------------------------------------------------- frozen cases
def test_frozen_dot_and_mbm(orc):
    # test_kernels.cpp:41-69
    u = np.array([0b101], np.uint64)
    v = np.array([0b100], np.uint64)
    w = np.array([0], np.uint64)
    assert orc.dot_binary(u, u, 3) == 3
    assert orc.dot_binary(u, v, 3) == 1
    assert orc.dot_binary(u, w, 3) == -1
    assert orc.dot_binary(np.array([0b1111], np.uint64), w, 4) == -4
    x, y, z = (np.array([b], np.uint64) for b in (0b110, 0b101, 0b011))
    assert orc.mbm(x, y, z) == -2
    assert orc.mbm(x, x, np.array([0b111], np.uint64)) == 3
    assert orc.mbm(x, y, np.array([0], np.uint64)) == 0
    assert orc.mbm(x, y, np.array([0b100], np.uint64)) == 1


def test_frozen_1x1(orc):
    # test_kernels.cpp:89-99: [+1,-1,+1] . [+1,+1,+1] = 1, scaled by gamma_a*gamma_b
    a, wpr = data.pack_bits(np.array([[1, 0, 1]], np.uint8))
    b, _ = data.pack_bits(np.array([[1, 1, 1]], np.uint8))
    assert orc.gemm_1x1(a, b, 3, wpr)[1][0, 0] == 1.0
    assert orc.gemm_1x1(a, b, 3, wpr, 0.5, 2.0)[1][0, 0] == 1.0
    assert orc.gemm_1x1(a, b, 3, wpr, 2.0, 3.0)[1][0, 0] == 6.0


def test_frozen_1x2(orc):
    # test_kernels.cpp:107-119: signs [+1,-1,+1,+1] x levels [0,1,2,3] = 4
    w, wpr = data.pack_bits(np.array([[1, 0, 1, 1]], np.uint8))
    t, h, m, _ = _planes([0, 1, 2, 3])
    assert orc.gemm_1x2(w, 1.0, t, h, m, 4, wpr)[1][0, 0] == 4.0
    assert orc.gemm_1x2(w, 2.0, t, h, m, 4, wpr)[1][0, 0] == 8.0
    assert orc.gemm_1x2(w, 2.0, t, h, m, 4, wpr, a_gamma=0.5)[1][0, 0] == 4.0


def test_frozen_2x2(orc):
    # test_kernels.cpp:125-139
    wt, wh, wm, wpr = _planes([3, 1])
    at, ah, am, _ = _planes([0, 2])
    assert orc.gemm_2x2(wt, wh, wm, at, ah, am, 2, wpr)[1][0, 0] == 2.0
    t3, h3, m3, wpr1 = _planes([3])
    assert orc.gemm_2x2(t3, h3, m3, t3, h3, m3, 1, wpr1)[1][0, 0] == 9.0
    assert orc.gemm_2x2(t3, h3, m3, t3, h3, m3, 1, wpr1, w_scale=0.5, a_scale=0.25)[1][0, 0] == 1.125


def test_frozen_1x32_and_spmm(orc):
    # test_kernels.cpp:216-220, 235-242
    w, wpr = data.pack_bits(np.array([[1, 0, 1]], np.uint8))
    b = np.array([[1.0], [2.0], [3.0]], np.float32)
    assert orc.gemm_1x32(w, 3, wpr, 2.0, b)[0, 0] == 4.0
    rp = np.array([0, 1, 2], np.uint64)
    ci = np.array([1, 0], np.uint64)
    v = np.array([5.0, 1.0], np.float32)
    bb = np.array([[1.0, 2.0], [3.0, 4.0]], np.float32)
    assert np.array_equal(orc.spmm_csr(2, rp, ci, v, bb), np.array([[15, 20], [1, 2]], np.float32))


# ---------------------------------------------------------------- golden (reference outputs)
def test_oracle_matches_reference_gemm_golden(orc, gemm_golden):
    for i in range(int(gemm_golden["gemm_count"])):
        c = gemm_case(gemm_golden, i)
        k, wpr, lane = c["k"], c["wpr"], c["lane"]
        wt, wh, wm, _ = data.planes_from_levels(c["lw"], lane)
        at, ah, am, _ = data.planes_from_levels(c["la"], lane)
        _, o11 = orc.gemm_1x1(c["a"], c["b"], k, wpr, c["g_a"], c["g_b"])
        _, o12 = orc.gemm_1x2(c["a"], c["g_w"], at, ah, am, k, wpr, c["s_a"], c["g_a"])
        _, o22 = orc.gemm_2x2(wt, wh, wm, at, ah, am, k, wpr, c["s_w"], c["s_a"], None, c["g_a"])
        assert np.array_equal(o11, c["c11"]), i
        assert np.array_equal(o12, c["c12"]), i
        assert np.array_equal(o22, c["c22"]), i


def test_oracle_integer_units_match_decoded_dense(orc, gemm_golden):
    # test_kernels.cpp:145-183: units equal plain integer sums of decoded operands
    for i in range(0, int(gemm_golden["gemm_count"]), 5):
        c = gemm_case(gemm_golden, i)
        k, wpr, lane = c["k"], c["wpr"], c["lane"]
        sa = 2 * data.unpack_bits(c["a"], k).astype(np.int64) - 1
        sb = 2 * data.unpack_bits(c["b"], k).astype(np.int64) - 1
        lw, la = c["lw"].astype(np.int64), c["la"].astype(np.int64)
        at, ah, am, _ = data.planes_from_levels(c["la"], lane)
        wt, wh, wm, _ = data.planes_from_levels(c["lw"], lane)
        assert np.array_equal(orc.gemm_1x1(c["a"], c["b"], k, wpr)[0], sa @ sb.T)
        assert np.array_equal(orc.gemm_1x2(c["a"], 1.0, at, ah, am, k, wpr)[0], 2 * (sa @ la.T))
        assert np.array_equal(orc.gemm_2x2(wt, wh, wm, at, ah, am, k, wpr)[0], 4 * (lw @ la.T))


def test_oracle_matches_reference_apb_golden(orc, apb_golden):
    for i in range(int(apb_golden["apb_count"])):
        c = apb_case(apb_golden, i)
        m, k, wpr = c["m"], c["k"], c["wpr"]
        if "alpha_vec" in c:
            out = orc.layer_forward(m, k, 1.0, c["bin"], wpr, c["row_ptr"], c["col_idx"], c["vals"],
                                    c["b"], row_alpha=c["alpha_vec"])
            bin_, _, rp, ci, v = orc.decompose_apb(c["fwd"], c["alpha_vec"])
        else:
            alpha = float(c["alpha_delta"][0])
            fwd = orc.apb_forward(c["w"], alpha, float(c["alpha_delta"][1]))
            assert np.array_equal(fwd, c["fwd"])
            bin_, _, rp, ci, v = orc.decompose_apb(c["fwd"], alpha)
            out = orc.layer_forward(m, k, alpha, c["bin"], wpr, c["row_ptr"], c["col_idx"],
                                    c["vals"], c["b"])
            assert np.array_equal(orc.gemm_1x32(c["bin"], k, wpr, alpha, c["b"]), c["c1x32"])
            assert np.array_equal(orc.spmm_csr(m, c["row_ptr"], c["col_idx"], c["vals"], c["b"]),
                                  c["cspmm"])
        assert np.array_equal(bin_, c["bin"]) and np.array_equal(rp, c["row_ptr"])
        assert np.array_equal(ci, c["col_idx"]) and np.array_equal(v, c["vals"])
        assert np.array_equal(out, c["c"]), i


def test_oracle_matches_reference_packing_golden(orc, packing_golden):
    g = packing_golden
    for i in range(int(g["pack_count"])):
        p = f"p{i:03d}_"
        rows, cols, lane, wpr = (int(x) for x in g[p + "shape"])
        words, w2 = orc.pack_signs(g[p + "a"], lane)
        assert w2 == wpr and np.array_equal(words, g[p + "signs"])
        lv = orc.quantize_2bit(g[p + "x"], 0.5)
        assert np.array_equal(lv, g[p + "levels"])
        t, h, m, _ = orc.decompose_thm(lv, lane)
        assert np.array_equal(t, g[p + "t"]) and np.array_equal(h, g[p + "h"])
        assert np.array_equal(m, g[p + "m"])
    for j in range(int(g["row_count"])):
        p = f"r{j:03d}_"
        n = int(g[p + "n"])
        assert orc.dot_binary(g[p + "u"], g[p + "v"], n) == int(g[p + "dot"])
        assert orc.mbm(g[p + "u"], g[p + "v"], g[p + "z"]) == int(g[p + "mbm"])


# ---------------------------------------------------------------- live reference (here only)
def test_oracle_matches_live_reference_random(orc, ref):
    rng = np.random.default_rng(77)
    for _ in range(25):
        m, n = int(rng.integers(1, 24)), int(rng.integers(1, 24))
        k = int(rng.integers(1, 700))
        a, wpr = data.random_words(rng, m, k)
        b, _ = data.random_words(rng, n, k)
        at, ah, am, _ = data.random_planes(rng, n, k)
        wt, wh, wm, _ = data.random_planes(rng, m, k)
        assert np.array_equal(orc.gemm_1x1(a, b, k, wpr, 0.7, 1.25)[1],
                              ref.gemm_1x1(a, b, k, wpr, 0.7, 1.25)[0])
        assert np.array_equal(orc.gemm_1x2(a, 1.25, at, ah, am, k, wpr, 0.3, 2.0)[1],
                              ref.gemm_1x2(a, 1.25, at, ah, am, k, wpr, 0.3, 2.0)[0])
        assert np.array_equal(orc.gemm_2x2(wt, wh, wm, at, ah, am, k, wpr, 0.75, 0.5, 0.5, None)[1],
                              ref.gemm_2x2(wt, wh, wm, at, ah, am, k, wpr, 0.75, 0.5, 0.5, None)[0])


def test_reference_backends_agree(ref):
    """test_simd_equivalence.cpp:85-125 pattern: scalar and avx512 reference backends agree,
    so the golden vectors do not depend on which ISA the GPU box's host runs."""
    rng = np.random.default_rng(5)
    a, wpr = data.random_words(rng, 9, 777)
    b, _ = data.random_words(rng, 11, 777)
    saved = ref.active_simd()
    outs = []
    for level in ("scalar", "avx2", "avx512"):
        try:
            ref.set_simd(level)
        except Exception:
            continue
        outs.append(ref.gemm_1x1(a, b, 777, wpr)[0])
    ref.set_simd(saved)
    assert len(outs) >= 1 and all(np.array_equal(outs[0], o) for o in outs)


@pytest.mark.parametrize("n", [1, 2, 3, 12])
def test_exhaustive_small_dot(orc, n):
    # acceptance.cpp:97-105 (exhaustive plain dot up to 12 positions; sampled here for n=12)
    lim = 1 << n
    rng = np.random.default_rng(n)
    us = range(lim) if n <= 6 else rng.integers(0, lim, 200)
    vs = range(lim) if n <= 6 else rng.integers(0, lim, 200)
    for u in us:
        for v in vs:
            want = sum((1 if (u >> i) & 1 else -1) * (1 if (v >> i) & 1 else -1) for i in range(n))
            got = orc.dot_binary(np.array([u], np.uint64), np.array([v], np.uint64), n)
            assert got == want
