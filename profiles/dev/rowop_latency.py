"""Per-call cost of one dot_binary / mbm row pair: the GPU host flavour (count = 1, what the
drop-in's BITMM_DROPIN_ROWOPS_GPU binding calls) vs the reference's AVX-512 row op
(oracle/_ref) and the batched device call per row. python profiles/dev/rowop_latency.py"""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2306_08960_b200 import _lib  # noqa: E402

lib = _lib.load()
ref = oracle.load_ref()
P = lambda x: x.ctypes.data_as(C.c_void_p)  # noqa: E731
rng = np.random.default_rng(3)
for words in (1, 8, 64):
    n = words * 64
    u = rng.integers(0, 2**63, words, dtype=np.uint64)
    v = rng.integers(0, 2**63, words, dtype=np.uint64)
    out = np.zeros(1, np.int64)
    for _ in range(20):
        lib.bitmm_dot_binary_host(P(u), P(v), 1, words, n, P(out))
    t0 = time.perf_counter()
    reps = 2000
    for _ in range(reps):
        lib.bitmm_dot_binary_host(P(u), P(v), 1, words, n, P(out))
    gpu = (time.perf_counter() - t0) / reps
    t0 = time.perf_counter()
    for _ in range(reps):
        ref.dot_binary(u, v, n)
    cpu = (time.perf_counter() - t0) / reps
    # batched: 65536 row pairs in one host call
    U = rng.integers(0, 2**63, (65536, words), dtype=np.uint64)
    V = rng.integers(0, 2**63, (65536, words), dtype=np.uint64)
    O = np.zeros(65536, np.int64)
    lib.bitmm_dot_binary_host(P(U), P(V), 65536, words, n, P(O))
    t0 = time.perf_counter()
    lib.bitmm_dot_binary_host(P(U), P(V), 65536, words, n, P(O))
    batch = (time.perf_counter() - t0) / 65536
    print(f"dot_binary {n:5d} bits: GPU per call {gpu * 1e6:7.1f} us, reference CPU (via ctypes) "
          f"{cpu * 1e6:6.2f} us, GPU batched {batch * 1e9:7.1f} ns per row pair")
