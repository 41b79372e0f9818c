"""Batched row ops on the GPU (dot_binary / mbm, kernels.cpp:120-140) vs the reference's own
golden values (tests/golden/packing_cases.npz, from oracle/_ref) and the oracle."""
import numpy as np
import pytest

from paper_2306_08960_b200 import data

pytestmark = pytest.mark.gpu


def _T(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint64).view(np.int64)).cuda()


def test_golden_row_ops(packing_golden):
    from paper_2306_08960_b200 import device
    g = packing_golden
    import re
    ids = sorted({k.split("_")[0] for k in g if re.match(r"r\d{3}_", k)})
    assert ids
    for i in ids:
        u, v, z = (np.atleast_2d(g[f"{i}_{x}"]) for x in ("u", "v", "z"))
        n = int(g[f"{i}_n"])
        d = device.dot_binary_rows(_T(u), _T(v), n).cpu().numpy()
        mm = device.mbm_rows(_T(u), _T(v), _T(z)).cpu().numpy()
        assert d[0] == int(g[f"{i}_dot"]), i
        assert mm[0] == int(g[f"{i}_mbm"]), i


@pytest.mark.parametrize("count,cols", [(1, 1), (1000, 64), (37, 4096), (5, 100000)])
def test_random_rows_vs_oracle(orc, count, cols):
    from paper_2306_08960_b200 import device
    rng = np.random.default_rng(count + cols)
    u, words = data.random_words(rng, count, cols)
    v, _ = data.random_words(rng, count, cols)
    z, _ = data.random_words(rng, count, cols)
    d = device.dot_binary_rows(_T(u), _T(v), cols).cpu().numpy()
    m = device.mbm_rows(_T(u), _T(v), _T(z)).cpu().numpy()
    for r in range(count):
        assert d[r] == orc.dot_binary(u[r], v[r], cols)
        assert m[r] == orc.mbm(u[r], v[r], z[r])


def test_row_op_errors():
    from paper_2306_08960_b200 import device
    u = np.zeros((2, 1), np.uint64)
    with pytest.raises(ValueError):
        device.dot_binary_rows(_T(u), _T(u), 65)  # words_for(65) = 2 > 1 (kernels.cpp:122)
