"""Dev diagnostic: where does the APB binary-part error come from? (not a pytest module)"""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2306_08960_b200 import api, data
rng = np.random.default_rng(0)
for (m, k, n) in [(256, 768, 512), (256, 4096, 512), (256, 64, 512)]:
    bits = rng.integers(0, 2, (m, k), dtype=np.uint8)
    w, wpr = data.pack_bits(bits)
    bm = api.BitMatrix.from_words(m, k, wpr, w)
    s = (2 * bits.astype(np.float64) - 1)
    x = rng.standard_normal((k, n)).astype(np.float32)
    # bf16-exact x: error only from accumulation
    xb = (x.view(np.uint32) & np.uint32(0xFFFF0000)).view(np.float32)
    for name, xx in [("bf16-exact x", xb), ("fp32 x", x)]:
        got = api.gemm_1x32_ref(bm, 1.0, xx)
        want = s @ xx.astype(np.float64)
        rel = np.linalg.norm(got - want) / np.linalg.norm(want)
        mx = np.max(np.abs(got - want)) / np.max(np.abs(want))
        bias = np.mean((got - want) * np.sign(want))
        print(f"m={m} k={k} n={n} {name}: rel_frob={rel:.3e} max_abs/max={mx:.3e} signed_bias={bias:.3e}")
