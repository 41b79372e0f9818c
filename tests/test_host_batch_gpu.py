"""Host-flavour GEMM group (`bitmm_gemm_batch_host`): the *_host calls of several items, with
their wire pipelines merged into one when every output takes the 16-bit wire. Results must be
bit-identical to the single host calls (themselves pinned to the oracle elsewhere) and to the
oracle on sampled rows; a device-detected encoding error in any item must be reported."""
import ctypes as C

import numpy as np
import pytest

import oracle
from paper_2306_08960_b200 import _lib, data

pytestmark = pytest.mark.gpu

lib = _lib.load()
orc = oracle.Oracle()
P = lambda x: None if x is None else x.ctypes.data_as(C.c_void_p)  # noqa: E731


def _items(rng, shapes, ldc_pad=0):
    """One item per (routine, m, n, k); host operands and fresh outputs (units and fp32)."""
    arr = (_lib.GemmItem * len(shapes))()
    keep = []
    for it, (routine, m, n, k) in zip(arr, shapes):
        if routine == 0:
            a, wpr = data.random_words(rng, m, k)
            b, _ = data.random_words(rng, n, k)
            ops = dict(a0=a, b0=b)
            it.a_scale, it.b_scale = 0.5, 1.5
        elif routine == 1:
            w, wpr = data.random_words(rng, m, k)
            t, h, mm, _ = data.random_planes(rng, n, k)
            ops = dict(a0=w, b0=t, b1=h, b2=mm)
            it.a_scale, it.b_scale, it.has_b_gamma, it.b_gamma = 0.75, 0.5, 1, 1.25
            rs = rng.uniform(0.5, 1.5, m).astype(np.float32)
            cs = rng.uniform(0.5, 1.5, n).astype(np.float32)
            ops.update(row_scale=rs, col_scale=cs)
        else:
            wt, wh, wm, wpr = data.random_planes(rng, m, k)
            t, h, mm, _ = data.random_planes(rng, n, k)
            ops = dict(a0=wt, a1=wh, a2=wm, b0=t, b1=h, b2=mm)
            it.a_scale, it.b_scale = 0.5, 2.0
        ldc = n + ldc_pad
        ops["u"] = np.full((m, ldc), -7, np.int32)
        ops["c"] = np.full((m, ldc), -7.0, np.float32)
        for name, v in ops.items():
            if name in ("u", "c"):
                continue
            setattr(it, name, v.ctypes.data)
        it.routine, it.m, it.n, it.k, it.wpr, it.ldc = routine, m, n, k, wpr, ldc
        it.c_units, it.c = ops["u"].ctypes.data, ops["c"].ctypes.data
        keep.append(ops)
    return arr, keep


def _single(it, u, c):
    """The same item through its own *_host call."""
    f = lambda name: getattr(it, name)  # noqa: E731
    if it.routine == 0:
        return lib.bitmm_gemm_1x1_host(f("a0"), it.m, f("b0"), it.n, it.k, it.wpr, it.a_scale, it.b_scale, P(u),
                                       P(c), it.ldc)
    if it.routine == 1:
        return lib.bitmm_gemm_1x2_host(f("a0"), it.m, it.a_scale, f("b0"), f("b1"), f("b2"), it.n, it.k, it.wpr,
                                       it.b_scale, it.has_b_gamma, it.b_gamma, f("row_scale"), f("col_scale"),
                                       P(u), P(c), it.ldc)
    return lib.bitmm_gemm_2x2_host(f("a0"), f("a1"), f("a2"), it.m, it.a_scale, it.has_a_gamma, it.a_gamma, f("b0"),
                                   f("b1"), f("b2"), it.n, it.k, it.wpr, it.b_scale, it.has_b_gamma, it.b_gamma,
                                   f("row_scale"), f("col_scale"), P(u), P(c), it.ldc)


# every output >= 32 MB (merged pipeline; slices of rows for 1/1 and 2/2, of columns for 1/2),
# and a batch with a small item (run one after the other)
CASES = {
    "merged": [(0, 2304, 4096, 520), (1, 1100, 8200, 700), (2, 2100, 4100, 300)],
    "merged-pad": [(2, 2048, 4500, 130), (0, 2600, 3300, 1000)],
    "mixed": [(0, 2304, 4096, 520), (1, 300, 500, 777)],
}


@pytest.mark.parametrize("case", list(CASES))
def test_batch_host_matches_single_calls(case):
    rng = np.random.default_rng(len(case))
    arr, keep = _items(rng, CASES[case], ldc_pad=3 if case == "merged-pad" else 0)
    assert lib.bitmm_gemm_batch_host(arr, len(arr)) == 0, _lib.last_error()
    for it, ops in zip(arr, keep):
        u = np.full_like(ops["u"], -7)
        c = np.full_like(ops["c"], -7.0)
        assert _single(it, u, c) == 0, _lib.last_error()
        assert np.array_equal(ops["u"], u) and np.array_equal(ops["c"], c), (case, it.routine)
    # and the 1/1 item against the oracle on sampled rows
    it, ops = arr[0], keep[0]
    if it.routine == 0:
        rows = rng.choice(it.m, 16, replace=False)
        wu, _ = orc.gemm_1x1(ops["a0"][rows], ops["b0"], it.k, it.wpr, it.a_scale, it.b_scale)
        assert np.array_equal(ops["u"][rows, :it.n], wu)


def test_batch_host_merged_and_sequential_agree(monkeypatch):
    rng = np.random.default_rng(3)
    arr, keep = _items(rng, CASES["merged"])
    assert lib.bitmm_gemm_batch_host(arr, len(arr)) == 0, _lib.last_error()
    merged_bytes = lib.bitmm_last_d2h_bytes()
    monkeypatch.setenv("BITMM_HOST_BATCH", "0")
    arr2, keep2 = _items(np.random.default_rng(3), CASES["merged"])
    assert lib.bitmm_gemm_batch_host(arr2, len(arr2)) == 0, _lib.last_error()
    # the same parts cross PCIe either way (12-bit where the columns allow, else 16-bit words)
    assert lib.bitmm_last_d2h_bytes() == merged_bytes <= sum(it.m * it.n * 2 for it in arr)
    for a, b in zip(keep, keep2):
        assert np.array_equal(a["u"], b["u"]) and np.array_equal(a["c"], b["c"])


def test_batch_host_errors():
    rng = np.random.default_rng(4)
    arr, keep = _items(rng, CASES["merged"])
    # an illegal plane triple in the 2/2 item's activations: InvalidEncoding from the device
    bad_t = keep[2]["b0"].copy()
    bad_h = keep[2]["b1"].copy()
    bad_t[7, 1] |= np.uint64(1) << np.uint64(3)
    bad_h[7, 1] |= np.uint64(1) << np.uint64(3)
    keep[2]["b0"], keep[2]["b1"] = bad_t, bad_h
    arr[2].b0, arr[2].b1 = bad_t.ctypes.data, bad_h.ctypes.data
    assert lib.bitmm_gemm_batch_host(arr, len(arr)) == 2
    # argument errors before any work
    assert lib.bitmm_gemm_batch_host(arr, 0) == 1
    assert lib.bitmm_gemm_batch_host(arr, 5) == 1
    arr[0].routine = 7
    assert lib.bitmm_gemm_batch_host(arr, 1) == 1
    # a valid batch afterwards (the latched status was consumed)
    arr, keep = _items(rng, CASES["merged"][:2])
    assert lib.bitmm_gemm_batch_host(arr, len(arr)) == 0, _lib.last_error()
