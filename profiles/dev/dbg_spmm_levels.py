import sys, os
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
import oracle
from paper_2306_08960_b200 import api
import test_apb2 as T
orc = oracle.Oracle()
rows, cols, tokens = 300, 768, 333
rng = np.random.default_rng(0 + rows * 7 + cols)
layer, alpha = T._layer(rng, rows, cols, keep_frac=0.02, lane=512)
t, h, m, wpr = T._planes(rng, tokens, cols, 512)
s = 0.125 + rng.random()
planes = T._thm(t, h, m, cols, s, None)
got = api.layer_forward_2bit(layer, planes)
rr = layer.residual
want = orc.layer_forward_2bit(rows, cols, 1.0, layer.bin.words, wpr, rr.row_ptr, rr.col_idx, rr.vals, t, h, m,
                              a_scale=s, a_gamma=None, row_alpha=alpha)
d = np.argwhere(got != want)
print("ndiff", len(d), "of", got.size)
print("rows", np.unique(d[:, 0])[:20], "cols", np.unique(d[:, 1])[:40])
for r, c in d[:5]:
    print(r, c, got[r, c], want[r, c], got[r, c] - want[r, c])
