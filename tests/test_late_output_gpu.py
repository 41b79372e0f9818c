"""Late-output host calls (`bitmm_gemm_host_late`) and the staged small-output path.

The reference's gemm_1x1 / 1x2 / 2x2 return a fresh DenseMatrix (kernels.cpp:163-275); the
drop-in builds it inside the library's callback while the device works. Outputs below the
pipelining threshold travel through the lease's pinned staging and are copied into the
destination by the host pool (run_staged); larger ones resolve the destination up front and
take the sliced / 16-bit wire paths. Every result must equal the oracle bit for bit, cells
outside the requested block must stay untouched, and device-detected errors must be reported
without writing the destination."""
import ctypes as C

import numpy as np
import pytest

import oracle
from paper_2306_08960_b200 import _lib, data

pytestmark = pytest.mark.gpu

lib = _lib.load()
orc = oracle.Oracle()
SENT = -123456789
P = lambda x: None if x is None else x.ctypes.data_as(C.c_void_p)  # noqa: E731


class Dest:
    """The callback's side: allocates sentinel-filled buffers with a leading dimension of
    n + pad when called, records how often it was called."""

    def __init__(self, m, n, pad=0, fail=False, null=False):
        self.m, self.n, self.ldc = m, n, n + pad
        self.fail, self.null = fail, null
        self.calls = 0
        self.u = self.c = None
        self.fn = _lib.OUT_FN(self._cb)

    def _cb(self, user, out):
        self.calls += 1
        if self.fail:
            return 7
        assert out.contents.ldc == self.n  # preset to n
        self.u = np.full((self.m, self.ldc), SENT, np.int32)
        self.c = np.full((self.m, self.ldc), np.float32(SENT), np.float32)
        out.contents.c_units = None if self.null else self.u.ctypes.data
        out.contents.c = self.c.ctypes.data
        out.contents.ldc = self.ldc
        return 0


def _item(routine, m, n, k, wpr, ops, scales=(1.0, 1.0)):
    it = _lib.GemmItem()
    it.routine = routine
    names = ("a0", "a1", "a2", "b0", "b1", "b2")
    for name, arr in zip(names, ops):
        if arr is not None:
            setattr(it, name, arr.ctypes.data)
    it.m, it.n, it.k, it.wpr = m, n, k, wpr
    it.a_scale, it.b_scale = scales
    return it


def _case(routine, m, n, k, seed):
    rng = np.random.default_rng(seed)
    if routine == _lib.ROUTINE_1X1:
        a, wpr = data.random_words(rng, m, k)
        b, _ = data.random_words(rng, n, k)
        ops = (a, None, None, b, None, None)
        want = orc.gemm_1x1(a, b, k, wpr, 0.75, 1.25)
        scales = (0.75, 1.25)
    elif routine == _lib.ROUTINE_1X2:
        w, wpr = data.random_words(rng, m, k)
        t, h, mm, _ = data.random_planes(rng, n, k)
        ops = (w, None, None, t, h, mm)
        want = orc.gemm_1x2(w, 0.5, t, h, mm, k, wpr, a_scale=1.5)
        scales = (0.5, 1.5)
    else:
        wt, wh, wm, wpr = data.random_planes(rng, m, k)
        t, h, mm, _ = data.random_planes(rng, n, k)
        ops = (wt, wh, wm, t, h, mm)
        want = orc.gemm_2x2(wt, wh, wm, t, h, mm, k, wpr, w_scale=0.5, a_scale=2.0)
        scales = (0.5, 2.0)
    return ops, wpr, want, scales


# small (staged, ragged), 1024^3 (the acceptance criterion-8 shape), one > 32 MB output
# (destination resolved up front; sliced 16-bit wire)
SHAPES = [(200, 300, 1000), (1024, 1024, 1024), (2112, 4096, 512)]


@pytest.mark.parametrize("routine", [0, 1, 2])
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("want", [1, 2, 3])
@pytest.mark.parametrize("wire_min", [None, "0"])
def test_late_output_bit_exact(routine, shape, want, wire_min, monkeypatch):
    """wire_min "0": every output takes the 16-bit wire (BITMM_WIRE_MIN_BYTES=0), so a late
    destination is resolved before the wire's pipeline starts."""
    if wire_min is not None:
        monkeypatch.setenv("BITMM_WIRE_MIN_BYTES", wire_min)
    m, n, k = shape
    ops, wpr, (wu, wc), scales = _case(routine, m, n, k, seed=m + n + k + routine)
    it = _item(routine, m, n, k, wpr, ops, scales)
    d = Dest(m, n, pad=5 if m < 1024 else 0)
    assert lib.bitmm_gemm_host_late(C.byref(it), want, d.fn, None) == 0, _lib.last_error()
    assert d.calls == 1
    if want & 1:
        assert np.array_equal(d.u[:, :n], wu)
    else:
        assert (d.u == SENT).all()
    if want & 2:
        assert np.array_equal(d.c[:, :n], wc)
    else:
        assert (d.c == np.float32(SENT)).all()
    if d.ldc > n:  # the padding columns are not the output's
        assert (d.u[:, n:] == SENT).all() and (d.c[:, n:] == np.float32(SENT)).all()


@pytest.mark.parametrize("staged", ["1", "0"])
def test_host_call_into_pageable_strided_output(staged, monkeypatch):
    """The plain *_host calls below the pipelining threshold: staged (default for pageable
    destinations) and the direct copy (BITMM_HOST_STAGED=0) give the same bits, ldc > n."""
    monkeypatch.setenv("BITMM_HOST_STAGED", staged)
    m, n, k = 700, 333, 1500
    ops, wpr, (wu, wc), _ = _case(0, m, n, k, seed=4)
    ldc = n + 3
    u = np.full((m, ldc), SENT, np.int32)
    c = np.full((m, ldc), np.float32(SENT), np.float32)
    assert lib.bitmm_gemm_1x1_host(P(ops[0]), m, P(ops[3]), n, k, wpr, 0.75, 1.25, P(u), P(c), ldc) == 0
    assert np.array_equal(u[:, :n], wu) and np.array_equal(c[:, :n], wc)
    assert (u[:, n:] == SENT).all() and (c[:, n:] == np.float32(SENT)).all()
    assert lib.bitmm_last_d2h_bytes() == 2 * m * n * 4


def test_late_output_callback_errors():
    m, n, k = 64, 96, 256
    ops, wpr, _, scales = _case(0, m, n, k, seed=1)
    it = _item(0, m, n, k, wpr, ops, scales)
    d = Dest(m, n, fail=True)
    assert lib.bitmm_gemm_host_late(C.byref(it), 3, d.fn, None) == 1
    assert "callback" in _lib.last_error()
    d = Dest(m, n, null=True)
    assert lib.bitmm_gemm_host_late(C.byref(it), 3, d.fn, None) == 1
    assert "null" in _lib.last_error()
    # bad arguments fail before anything is enqueued: the callback is never called
    d = Dest(m, n)
    assert lib.bitmm_gemm_host_late(C.byref(it), 0, d.fn, None) == 1
    assert lib.bitmm_gemm_host_late(C.byref(it), 4, d.fn, None) == 1
    it.k = 0
    assert lib.bitmm_gemm_host_late(C.byref(it), 3, d.fn, None) == 1
    it.k = k
    it.routine = 9
    assert lib.bitmm_gemm_host_late(C.byref(it), 3, d.fn, None) == 1
    assert d.calls == 0
    # and a valid call afterwards works
    it.routine = 0
    assert lib.bitmm_gemm_host_late(C.byref(it), 3, d.fn, None) == 0 and d.calls == 1


def test_late_output_device_error_leaves_destination_untouched():
    """An illegal plane word is detected on the device (ThmPlanes::validate, tensor.cpp:133-153):
    the call reports InvalidEncoding and writes nothing into the callback's buffers."""
    m, n, k = 128, 80, 700
    ops, wpr, _, scales = _case(1, m, n, k, seed=3)
    t, h, mm = (x.copy() for x in ops[3:])
    t[5, 0] |= np.uint64(1)
    h[5, 0] &= ~np.uint64(1)
    mm[5, 0] &= ~np.uint64(1)
    it = _item(1, m, n, k, wpr, (ops[0], None, None, t, h, mm), scales)
    d = Dest(m, n)
    assert lib.bitmm_gemm_host_late(C.byref(it), 3, d.fn, None) == 2
    assert d.calls == 1
    assert (d.u == SENT).all() and (d.c == np.float32(SENT)).all()
    # the latched status was consumed: the same call on legal planes succeeds
    it = _item(1, m, n, k, wpr, ops, scales)
    assert lib.bitmm_gemm_host_late(C.byref(it), 2, d.fn, None) == 0


def test_other_host_calls_leave_columns_past_n_untouched():
    """gemm_1x32 / layer_forward / spmm_csr / the 2-bit layer, host flavour, into a buffer with
    ldc > n: the same values as with ldc = n, and columns [n, ldc) keep their contents."""
    from paper_2306_08960_b200 import api
    rng = np.random.default_rng(11)
    rows, cols, n = 96, 300, 70
    w, alpha, _ = data.apb_weights(rng, rows, cols)
    layer = api.decompose_apb(w, alpha)
    r = layer.residual
    bw, wpr = layer.bin.words, layer.bin.words_per_row()
    x = rng.standard_normal((cols, n)).astype(np.float32)
    t, h, mm, _ = data.random_planes(rng, n, cols)
    calls = {
        "1x32": lambda c, ldc: lib.bitmm_gemm_1x32_host(P(bw), rows, cols, wpr, 0.5, None, P(x), n, n, P(c), ldc),
        "layer": lambda c, ldc: lib.bitmm_layer_forward_host(rows, cols, 0.5, P(alpha), P(bw), wpr, P(r.row_ptr),
                                                             P(r.col_idx), P(r.vals), len(r.vals), P(x), n, n,
                                                             P(c), ldc),
        "spmm": lambda c, ldc: lib.bitmm_spmm_csr_host(rows, cols, P(r.row_ptr), P(r.col_idx), P(r.vals),
                                                       len(r.vals), P(x), n, n, P(c), ldc),
        "2bit": lambda c, ldc: lib.bitmm_layer_forward_2bit_host(rows, cols, 0.5, P(alpha), P(bw), wpr,
                                                                 P(r.row_ptr), P(r.col_idx), P(r.vals),
                                                                 len(r.vals), P(t), P(h), P(mm), n, 1.25, 0,
                                                                 1.0, P(c), ldc),
    }
    for name, fn in calls.items():
        ref = np.zeros((rows, n), np.float32)
        assert fn(ref, n) == 0, (name, _lib.last_error())
        c = np.full((rows, n + 3), np.float32(SENT), np.float32)
        assert fn(c, n + 3) == 0, (name, _lib.last_error())
        assert np.array_equal(c[:, :n], ref), name
        assert (c[:, n:] == np.float32(SENT)).all(), name
