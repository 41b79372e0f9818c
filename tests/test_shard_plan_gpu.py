"""Single-process multi-GPU 1/1 (bitmm_shard_plan_*): output columns split over
the listed devices, blocks gathered into the root's matrix by the GEMM epilogue (peer memory) or
by NCCL. On a one-GPU box the device list repeats device 0 (blocks run one after another on it),
which exercises the column split, the epilogue's strided stores into the root's matrix and the
plan's bookkeeping; NCCL then needs distinct devices and must refuse. Results bit-exact against
the oracle."""
import ctypes as C

import numpy as np
import pytest

import oracle
from paper_2306_08960_b200 import _lib, data

pytestmark = pytest.mark.gpu
lib = _lib.load()
orc = oracle.Oracle()
P = lambda x: x.ctypes.data_as(C.c_void_p)  # noqa: E731
NONE, PEER, NCCL = 0, 1, 2


def _plan(devs, m, n, k, seed=0):
    rng = np.random.default_rng(seed + m + n + k)
    a, wpr = data.random_words(rng, m, k)
    b, _ = data.random_words(rng, n, k)
    dv = (C.c_int * len(devs))(*devs)
    plan = C.c_void_p()
    assert lib.bitmm_shard_plan_create(dv, len(devs), m, n, k, wpr, C.byref(plan)) == 0, _lib.last_error()
    assert lib.bitmm_shard_plan_upload(plan, P(a), P(b)) == 0, _lib.last_error()
    return plan, a, b, wpr


@pytest.mark.parametrize("devs", [[0], [0, 0], [0, 0, 0]])
@pytest.mark.parametrize("m,n,k", [(300, 1000, 777), (256, 4096, 4096), (1, 96, 64)])
def test_shard_plan_peer_gather_bit_exact(devs, m, n, k):
    if n < 32 * len(devs):
        pytest.skip("fewer than 32 columns per device")
    plan, a, b, wpr = _plan(devs, m, n, k)
    try:
        ms = C.c_double(0)
        for gather in (PEER, NCCL) if len(devs) == 1 else (PEER,):
            out = np.full((m, n + 5), -1, np.int32)
            assert lib.bitmm_shard_run(plan, gather, C.byref(ms)) == 0, _lib.last_error()
            assert ms.value > 0
            assert lib.bitmm_shard_download(plan, 0, m, P(out), n + 5) == 0
            assert np.array_equal(out[:, :n], orc.gemm_1x1(a, b, k, wpr)[0]), gather
            assert (out[:, n:] == -1).all()
        assert lib.bitmm_shard_run(plan, NONE, C.byref(ms)) == 0, _lib.last_error()
        if len(devs) > 1:  # NCCL needs distinct devices
            assert lib.bitmm_shard_run(plan, NCCL, C.byref(ms)) == 3
            assert "distinct" in _lib.last_error()
    finally:
        assert lib.bitmm_shard_plan_destroy(plan) == 0


def test_shard_plan_errors():
    plan = C.c_void_p()
    dv = (C.c_int * 2)(0, 99)
    assert lib.bitmm_shard_plan_create(dv, 2, 64, 256, 512, 8, C.byref(plan)) == 1  # device 99
    dv = (C.c_int * 3)(0, 0, 0)
    assert lib.bitmm_shard_plan_create(dv, 3, 64, 64, 512, 8, C.byref(plan)) == 1  # < 32 columns each
    assert lib.bitmm_shard_plan_create(dv, 0, 64, 256, 512, 8, C.byref(plan)) == 1
    p, *_ = _plan([0], 32, 64, 128)
    try:
        assert lib.bitmm_shard_run(p, 7, None) == 1
        out = np.zeros((32, 10), np.int32)
        assert lib.bitmm_shard_download(p, 0, 32, P(out), 10) == 1  # ldc < n
        assert lib.bitmm_shard_download(p, 30, 3, P(np.zeros((3, 64), np.int32)), 64) == 1  # rows past m
        part = np.zeros((3, 64), np.int32)
        assert lib.bitmm_shard_run(p, 1, None) == 0
        assert lib.bitmm_shard_download(p, 29, 3, P(part), 64) == 0
    finally:
        lib.bitmm_shard_plan_destroy(p)
