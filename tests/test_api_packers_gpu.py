"""GPU: the packers of the Python mirror of the reference interface (api.pack_signs,
api.decompose_thm, api.decompose_apb run on the GPU through the host ABI) against the
reference's golden vectors, its frozen test cases and the oracle."""
import numpy as np
import pytest

from conftest import apb_case
from paper_2306_08960_b200 import api, data

pytestmark = pytest.mark.gpu


def test_bitmatrix_frozen_packing():
    # test_tensor.cpp:17-30: [+1,-1,+1] -> 0b101, 8 words per row at 512-bit lanes
    b = api.pack_signs(np.array([[1.0, -1.0, 1.0]], np.float32))
    assert int(b.words[0, 0]) == 0b101
    assert b.words_per_row() == 8
    assert b.bit(0, 0) and not b.bit(0, 1) and b.bit(0, 2)
    assert api.pack_signs(np.array([[0.0, -0.0]], np.float32)).words[0, 0] == 0b11  # sign(0)=+1


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


