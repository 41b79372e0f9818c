"""The flat bulk-copy expansion (unpack.cuh, unpack_flat_kernel; BITMM_UNPACK_FLAT=1, measured and
not the default): taken for e2m1 operands whose rows hold no padding (K = 64 * words_per_row, a
multiple of 256). Results bit-exact against the
oracle and identical to the per-slice kernel (BITMM_UNPACK_FLAT=0), illegal plane triples
reported, chunk boundaries and ragged operand sizes covered."""
import numpy as np
import pytest
import torch

import oracle
from paper_2306_08960_b200 import api, data, device

pytestmark = pytest.mark.gpu
orc = oracle.Oracle()


def T(x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()


# (m, n, k, lane bits): lane 64 gives wpr = K / 64 for any K multiple of 64; K must be a
# multiple of 256 for the flat path (kpad = K); rows * words not a multiple of the 2048-word chunk
SHAPES = [(1, 1, 256, 64), (300, 517, 512, 64), (129, 70, 4096, 512), (1000, 333, 8192, 512),
          (64, 2050, 768, 256), (513, 257, 1280, 256)]


@pytest.mark.parametrize("m,n,k,lane", SHAPES)
@pytest.mark.parametrize("flat", ["1", "0"])
def test_flat_expansion_bit_exact(monkeypatch, m, n, k, lane, flat):
    monkeypatch.setenv("BITMM_UNPACK_FLAT", flat)
    rng = np.random.default_rng(m * 7 + k)
    a, wpr = data.random_words(rng, m, k, lane)
    b, _ = data.random_words(rng, n, k, lane)
    t, h, mm, _ = data.random_planes(rng, n, k, lane)
    wt, wh, wm, _ = data.random_planes(rng, m, k, lane)
    assert (wpr * 64 == k) == (k % lane == 0)
    u = torch.empty((m, n), dtype=torch.int32, device="cuda")
    device.gemm_1x1(T(a), T(b), k, units=u)
    assert np.array_equal(u.cpu().numpy(), orc.gemm_1x1(a, b, k, wpr)[0])
    device.gemm_1x2(T(a), 1.0, T(t), T(h), T(mm), k, units=u)
    assert np.array_equal(u.cpu().numpy(), orc.gemm_1x2(a, 1.0, t, h, mm, k, wpr)[0])
    device.gemm_2x2(T(wt), T(wh), T(wm), T(t), T(h), T(mm), k, units=u)
    assert np.array_equal(u.cpu().numpy(), orc.gemm_2x2(wt, wh, wm, t, h, mm, k, wpr)[0])
    device.status()


def test_flat_expansion_reports_illegal_planes(monkeypatch):
    monkeypatch.setenv("BITMM_UNPACK_FLAT", "1")
    rng = np.random.default_rng(2)
    m, n, k = 70, 2100, 4096  # the activation planes span two chunks
    a, wpr = data.random_words(rng, m, k)
    for row, word, bit in ((0, 0, 0), (n - 1, wpr - 1, 63), (1000, 17, 31)):
        t, h, mm, _ = data.random_planes(rng, n, k)
        t[row, word] |= np.uint64(1) << np.uint64(bit)  # t without m: illegal
        mm[row, word] &= ~(np.uint64(1) << np.uint64(bit))
        u = torch.empty((m, n), dtype=torch.int32, device="cuda")
        device.gemm_1x2(T(a), 1.0, T(t), T(h), T(mm), k, units=u)
        with pytest.raises(api.InvalidEncoding):
            device.status()
    # a legal call afterwards
    t, h, mm, _ = data.random_planes(rng, n, k)
    device.gemm_1x2(T(a), 1.0, T(t), T(h), T(mm), k, units=u)
    device.status()
