"""CPU: host-side mirror of the reference interface — packing, decomposition and
validation — against the oracle and the reference's golden vectors."""
import numpy as np
import pytest

from conftest import apb_case
from paper_2306_08960_b200 import api, data


def test_bitmatrix_frozen_packing():
    # test_tensor.cpp:17-30: [+1,-1,+1] -> 0b101, 8 words per row at 512-bit lanes
    b = api.pack_signs(np.array([[1.0, -1.0, 1.0]], np.float32))
    assert int(b.words[0, 0]) == 0b101
    assert b.words_per_row() == 8
    assert b.bit(0, 0) and not b.bit(0, 1) and b.bit(0, 2)
    assert api.pack_signs(np.array([[0.0, -0.0]], np.float32)).words[0, 0] == 0b11  # sign(0)=+1


def test_from_words_rejects_padding():
    # test_tensor.cpp:81-91
    with pytest.raises(ValueError):
        api.BitMatrix.from_words(1, 3, 1, [0b1000])
    with pytest.raises(ValueError):
        api.BitMatrix.from_words(1, 65, 1, [0])
    with pytest.raises(ValueError):
        api.BitMatrix.from_words(2, 3, 1, [0])
    assert api.BitMatrix.from_words(1, 3, 1, [0b111]).padding_is_zero()


def test_packing_matches_golden(orc, packing_golden):
    g = packing_golden
    for i in range(int(g["pack_count"])):
        p = f"p{i:03d}_"
        rows, cols, lane, wpr = (int(x) for x in g[p + "shape"])
        b = api.pack_signs(g[p + "a"], lane)
        assert b.words_per_row() == wpr and np.array_equal(b.words, g[p + "signs"])
        q = api.quantize_uniform_2bit(g[p + "x"], 0.5)
        assert np.array_equal(q.levels.reshape(rows, cols), g[p + "levels"])
        tp = api.decompose_thm(q, lane_bits=lane)
        assert np.array_equal(tp.t.words, g[p + "t"]) and np.array_equal(tp.h.words, g[p + "h"])
        assert np.array_equal(tp.m.words, g[p + "m"])
        tp.validate()
        assert np.array_equal(data.levels_from_planes(tp.t.words, tp.h.words, tp.m.words, cols),
                              g[p + "levels"])


def test_random_planes_are_legal_uniform():
    rng = np.random.default_rng(0)
    t, h, m, wpr = data.random_planes(rng, 64, 1000)
    tp = api.ThmPlanes(*(api.BitMatrix.from_words(64, 1000, wpr, x) for x in (t, h, m)))
    tp.validate()
    lv = data.levels_from_planes(t, h, m, 1000)
    counts = np.bincount(lv.reshape(-1), minlength=4) / lv.size
    assert np.all(np.abs(counts - 0.25) < 0.01)


def test_thm_validate_errors():
    # test_tensor.cpp:123-148
    def planes(t, h, m):
        return api.ThmPlanes(*(api.BitMatrix.from_words(1, 1, 8, [v] + [0] * 7) for v in (t, h, m)))
    for t, h, m in [(1, 1, 0), (1, 0, 0), (0, 1, 1), (1, 1, 1)]:
        with pytest.raises(api.InvalidEncoding):
            planes(t, h, m).validate()
    for t, h, m in [(0, 0, 1), (0, 0, 0), (0, 1, 0), (1, 0, 1)]:
        planes(t, h, m).validate()


def test_decompose_apb_matches_golden(apb_golden):
    for i in range(int(apb_golden["apb_count"])):
        c = apb_case(apb_golden, i)
        alpha = c["alpha_vec"] if "alpha_vec" in c else float(c["alpha_delta"][0])
        layer = api.decompose_apb(c["fwd"], alpha)
        assert np.array_equal(layer.bin.words, c["bin"])
        assert np.array_equal(layer.residual.row_ptr, c["row_ptr"])
        assert np.array_equal(layer.residual.col_idx, c["col_idx"])
        assert np.array_equal(layer.residual.vals, c["vals"])


def test_decompose_apb_tie_rounding_matches_oracle(orc):
    # apb.cpp:35-46: non-dyadic thresholds exercise the ties-away-from-zero fixup
    rng = np.random.default_rng(8)
    for alpha, delta in [(0.75, 0.5), (0.7, 0.4), (0.3, 0.45)]:
        w = rng.uniform(-3, 3, (8, 90)).astype(np.float32)
        fwd = orc.apb_forward(w, alpha, delta)
        layer = api.decompose_apb(fwd, alpha)
        bw, wpr, rp, ci, v = orc.decompose_apb(fwd, alpha)
        assert np.array_equal(layer.bin.words, bw) and np.array_equal(layer.residual.vals, v)
        assert np.array_equal(layer.residual.col_idx, ci)
    with pytest.raises(ValueError):
        api.decompose_apb(np.ones((1, 1), np.float32), 0.0)


def test_csr_validation():
    # test_tensor.cpp:101-121
    api.CsrMatrix.create(2, 2, [0, 1, 2], [1, 0], [5.0, 1.0])
    with pytest.raises(ValueError):
        api.CsrMatrix.create(2, 2, [0, 1], [1], [5.0])
    with pytest.raises(ValueError):
        api.CsrMatrix.create(1, 2, [1, 1], [], [])
    with pytest.raises(ValueError):
        api.CsrMatrix.create(1, 2, [0, 2], [1, 1], [1.0, 2.0])
    with pytest.raises(ValueError):
        api.CsrMatrix.create(1, 2, [0, 1], [2], [1.0])
    with pytest.raises(ValueError):
        api.CsrMatrix.create(1, 2, [0, 1], [0], [np.inf])
    with pytest.raises(ValueError):
        api.CsrMatrix.create(2, 2, [0, 2, 1], [0, 1], [1.0, 1.0])


def test_quantizer_frozen():
    # test_transform.cpp:15-35: lround halves away from zero, clamp to [0, 3]
    q = api.quantize_uniform_2bit(np.array([[-1.0, 0.24, 0.25, 0.74, 0.75, 1.3, 9.0]], np.float32), 0.5)
    assert list(q.levels) == [0, 0, 1, 1, 2, 3, 3]
    with pytest.raises(ValueError):
        api.quantize_uniform_2bit(np.zeros((1, 1), np.float32), 0.0)


def test_apb_weights_generator_shape():
    rng = np.random.default_rng(1)
    a, alpha, keep = data.apb_weights(rng, 16, 768)
    assert keep == 15  # 2% of 768, the survey's C4 residual count
    layer = api.decompose_apb(a, alpha)
    assert layer.residual.nnz() == 16 * 15


def test_init_alpha_delta_matches_reference(tmp_path):
    """init_alpha_delta (apb.cpp:191-210): the host mirror's sequential double sums give the
    reference's alpha and delta bit for bit, including the 1e-8 delta floor."""
    import oracle
    ref = oracle.load_ref()
    if ref is None:
        pytest.skip("reference library not built")
    rng = np.random.default_rng(3)
    cases = [rng.normal(0.0, 0.02, (64, 300)).astype(np.float32),
             rng.uniform(-3, 3, (7, 1001)).astype(np.float32),
             np.full((3, 5), 0.25, np.float32)]  # zero variance: delta floor
    for w in cases:
        alpha, delta = api.init_alpha_delta(w)
        ra, rd = ref.pack_apb(w, str(tmp_path / "p"))
        assert np.float32(alpha) == np.float32(ra) and np.float32(delta) == np.float32(rd)
    with pytest.raises(ValueError):
        api.init_alpha_delta(np.zeros((0, 4), np.float32))
