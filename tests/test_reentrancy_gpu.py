"""Re-entrancy of the C ABI: concurrent calls from several host threads and streams.

The reference's gemm_1x1 / gemm_1x2 / gemm_2x2 allocate per call and share no state
(kernels.cpp:163-275); callers run them from many std::threads (run_row_blocks,
kernels.cpp:50-68). Here 4 host threads issue {1x1, 1x2, 2x2}_host calls (small outputs and
ones above the 32 MB threshold of the 16-bit pipelined wire) while 2 more threads issue
*_dev calls on two different CUDA streams, 50 iterations each; every result must equal the
oracle bit for bit. A single thread interleaving an asynchronous device call with a host
call (the case a shared workspace or status flag would break) is checked too.
"""
import ctypes as C
import threading

import numpy as np
import pytest

from paper_2306_08960_b200 import _lib, data

pytestmark = pytest.mark.gpu

ITERS = 50


def _p(x):
    return None if x is None else x.ctypes.data_as(C.c_void_p)


@pytest.fixture(scope="module")
def cases(orc):
    rng = np.random.default_rng(77)
    out = []
    for (m, n, k) in [(200, 300, 1000), (96, 64, 4096), (4096, 2048, 256)]:
        a, wpr = data.random_words(rng, m, k)
        b, _ = data.random_words(rng, n, k)
        t, h, mm, _ = data.random_planes(rng, n, k)
        wt, wh, wm, _ = data.random_planes(rng, m, k)
        out.append(dict(m=m, n=n, k=k, wpr=wpr, a=a, b=b, t=t, h=h, mm=mm, wt=wt, wh=wh, wm=wm,
                        u11=orc.gemm_1x1(a, b, k, wpr)[0], u12=orc.gemm_1x2(a, 1.0, t, h, mm, k, wpr)[0],
                        u22=orc.gemm_2x2(wt, wh, wm, t, h, mm, k, wpr)[0]))
    return out


def _host_call(lib, c, routine):
    m, n, k, wpr = c["m"], c["n"], c["k"], c["wpr"]
    u = np.empty((m, n), np.int32)
    if routine == 0:
        rc = lib.bitmm_gemm_1x1_host(_p(c["a"]), m, _p(c["b"]), n, k, wpr, 1.0, 1.0, _p(u), None, n)
        want = c["u11"]
    elif routine == 1:
        rc = lib.bitmm_gemm_1x2_host(_p(c["a"]), m, 1.0, _p(c["t"]), _p(c["h"]), _p(c["mm"]), n, k, wpr, 1.0,
                                     0, 1.0, None, None, _p(u), None, n)
        want = c["u12"]
    else:
        rc = lib.bitmm_gemm_2x2_host(_p(c["wt"]), _p(c["wh"]), _p(c["wm"]), m, 1.0, 0, 1.0, _p(c["t"]),
                                     _p(c["h"]), _p(c["mm"]), n, k, wpr, 1.0, 0, 1.0, None, None, _p(u),
                                     None, n)
        want = c["u22"]
    return rc, np.array_equal(u, want)


def test_concurrent_host_threads_and_device_streams(cases):
    import torch
    from paper_2306_08960_b200 import device
    lib = _lib.load()
    errors = []

    def host_worker(seed):
        rng = np.random.default_rng(seed)
        try:
            for _ in range(ITERS):
                for routine in (0, 1, 2):
                    c = cases[int(rng.integers(len(cases)))]
                    rc, ok = _host_call(lib, c, routine)
                    if rc != 0 or not ok:
                        errors.append(("host", seed, routine, c["m"], rc, _lib.last_error()))
                        return
        except Exception as e:  # pragma: no cover
            errors.append(("host", seed, repr(e)))

    T = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()  # noqa: E731
    dev_inputs = [{k: T(v) for k, v in c.items() if isinstance(v, np.ndarray) and v.dtype == np.uint64}
                  for c in cases]

    def dev_worker(seed):
        torch.cuda.set_device(0)
        stream = torch.cuda.Stream()
        rng = np.random.default_rng(seed)
        try:
            with torch.cuda.stream(stream):
                for _ in range(ITERS):
                    i = int(rng.integers(len(cases)))
                    c, d = cases[i], dev_inputs[i]
                    u11 = torch.empty((c["m"], c["n"]), dtype=torch.int32, device="cuda")
                    u22 = torch.empty_like(u11)
                    device.gemm_1x1(d["a"], d["b"], c["k"], units=u11, stream=stream)
                    device.gemm_2x2(d["wt"], d["wh"], d["wm"], d["t"], d["h"], d["mm"], c["k"], units=u22,
                                    stream=stream)
                    device.status(stream)
                    if not (np.array_equal(u11.cpu().numpy(), c["u11"]) and
                            np.array_equal(u22.cpu().numpy(), c["u22"])):
                        errors.append(("dev", seed, c["m"]))
                        return
        except Exception as e:  # pragma: no cover
            errors.append(("dev", seed, repr(e)))

    threads = [threading.Thread(target=host_worker, args=(s,)) for s in range(4)]
    threads += [threading.Thread(target=dev_worker, args=(100 + s,)) for s in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in threads), "a worker hung"
    assert not errors, errors[:5]


def test_async_device_call_then_host_call_same_thread(cases):
    """An enqueued (not yet synchronised) device call followed by a host call on the same
    thread: separate workspaces and status flags, so neither sees the other's data or errors."""
    import torch
    from paper_2306_08960_b200 import api, device
    lib = _lib.load()
    c = cases[2]
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()  # noqa: E731
    u = torch.empty((c["m"], c["n"]), dtype=torch.int32, device="cuda")
    bad_t = c["t"].copy()
    bad_h = c["h"].copy()
    bad_t[0, 0] |= np.uint64(1)
    bad_h[0, 0] |= np.uint64(1)  # t and h set on one element: illegal
    for _ in range(5):
        device.gemm_1x1(T(c["a"]), T(c["b"]), c["k"], units=u)           # async, default stream
        rc, ok = _host_call(lib, c, 1)                                    # host call meanwhile
        assert rc == 0 and ok
        assert np.array_equal(u.cpu().numpy(), c["u11"])
        # an encoding error latched by an async device call is reported by that stream only
        device.gemm_1x2(T(c["a"]), 1.0, T(bad_t), T(bad_h), T(c["mm"]), c["k"], units=u)
        rc, ok = _host_call(lib, c, 2)
        assert rc == 0 and ok
        with pytest.raises(api.InvalidEncoding):
            device.status()


def test_batched_and_late_host_calls_concurrently(cases):
    """bitmm_gemm_batch_host (the merged wire pipelines, a batch-local lease) and
    bitmm_gemm_host_late (the callback-provided destination) from two threads each, beside
    plain host calls: every result bit-exact, 20 iterations per thread."""
    lib = _lib.load()
    big = cases[2]  # 4096 x 2048: 32 MB of int32, on the 16-bit wire
    m, n, k, wpr = big["m"], big["n"], big["k"], big["wpr"]
    errors = []

    def batch_worker():
        for _ in range(20):
            items = (_lib.GemmItem * 2)()
            u0 = np.empty((m, n), np.int32)
            u1 = np.empty((m, n), np.int32)
            items[0].routine, items[0].a0, items[0].b0 = 0, big["a"].ctypes.data, big["b"].ctypes.data
            items[1].routine, items[1].a0 = 2, big["wt"].ctypes.data
            items[1].a1, items[1].a2 = big["wh"].ctypes.data, big["wm"].ctypes.data
            items[1].b0, items[1].b1, items[1].b2 = big["t"].ctypes.data, big["h"].ctypes.data, big["mm"].ctypes.data
            for it, u in zip(items, (u0, u1)):
                it.m, it.n, it.k, it.wpr, it.ldc = m, n, k, wpr, n
                it.a_scale = it.b_scale = 1.0
                it.c_units = u.ctypes.data
            if lib.bitmm_gemm_batch_host(items, 2) != 0:
                errors.append(_lib.last_error())
                return
            if not (np.array_equal(u0, big["u11"]) and np.array_equal(u1, big["u22"])):
                errors.append("batch mismatch")
                return

    def late_worker():
        c = cases[0]
        keep = {}

        def cb(user, out):
            keep["u"] = np.empty((c["m"], c["n"]), np.int32)
            out.contents.c_units = keep["u"].ctypes.data
            out.contents.ldc = c["n"]
            return 0

        fn = _lib.OUT_FN(cb)
        it = _lib.GemmItem()
        it.routine, it.a0, it.b0 = 0, c["a"].ctypes.data, c["b"].ctypes.data
        it.m, it.n, it.k, it.wpr, it.a_scale, it.b_scale = c["m"], c["n"], c["k"], c["wpr"], 1.0, 1.0
        for _ in range(20):
            if lib.bitmm_gemm_host_late(C.byref(it), _lib.WANT_UNITS, fn, None) != 0:
                errors.append(_lib.last_error())
                return
            if not np.array_equal(keep["u"], c["u11"]):
                errors.append("late mismatch")
                return

    def plain_worker():
        for i in range(20):
            rc, ok = _host_call(lib, cases[i % 2], i % 3)
            if rc != 0 or not ok:
                errors.append(f"plain {rc} {ok}")
                return

    threads = [threading.Thread(target=f) for f in (batch_worker, batch_worker, late_worker, late_worker,
                                                    plain_worker)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
