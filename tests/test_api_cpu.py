"""CPU: host-side parts of the mirror of the reference interface — layouts, validation, the
levels quantizer — and the CLI's fenced training-side helper, against the oracle and the
reference's golden vectors. The packers themselves run on the GPU (test_api_packers_gpu.py)."""
import numpy as np
import pytest

from paper_2306_08960_b200 import api, data


def test_from_words_rejects_padding():
    # test_tensor.cpp:81-91
    with pytest.raises(ValueError):
        api.BitMatrix.from_words(1, 3, 1, [0b1000])
    with pytest.raises(ValueError):
        api.BitMatrix.from_words(1, 65, 1, [0])
    with pytest.raises(ValueError):
        api.BitMatrix.from_words(2, 3, 1, [0])
    assert api.BitMatrix.from_words(1, 3, 1, [0b111]).padding_is_zero()


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
    import oracle
    _, _, rp, _, _ = oracle.Oracle().decompose_apb(a, alpha)
    assert int(rp[-1]) == 16 * 15


def test_init_alpha_delta_matches_reference(tmp_path):
    """init_alpha_delta (apb.cpp:191-210), the CLI's fenced training-side helper: its sequential
    double sums give the reference's alpha and delta bit for bit, including the 1e-8 floor."""
    from paper_2306_08960_b200 import cli
    import oracle
    ref = oracle.load_ref()
    if ref is None:
        pytest.skip("reference library not built")
    rng = np.random.default_rng(3)
    cases = [rng.normal(0.0, 0.02, (64, 300)).astype(np.float32),
             rng.uniform(-3, 3, (7, 1001)).astype(np.float32),
             np.full((3, 5), 0.25, np.float32)]  # zero variance: delta floor
    for w in cases:
        alpha, delta = cli.init_alpha_delta(w)
        ra, rd = ref.pack_apb(w, str(tmp_path / "p"))
        assert np.float32(alpha) == np.float32(ra) and np.float32(delta) == np.float32(rd)
    with pytest.raises(ValueError):
        cli.init_alpha_delta(np.zeros((0, 4), np.float32))
