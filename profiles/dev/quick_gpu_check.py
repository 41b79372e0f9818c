"""First-light GPU check (dev tool, not a pytest module): runs each C-ABI routine once
on small random inputs against a numpy restatement and times the 1/1 4096^3 kernel."""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2306_08960_b200 import _lib  # noqa: E402


def pack(bits, lane=512):
    rows, k = bits.shape
    wpr = ((k + lane - 1) // lane) * (lane // 64) if k else 0
    padded = np.zeros((rows, wpr * 64), np.uint8)
    padded[:, :k] = bits
    return np.packbits(padded, axis=1, bitorder="little").view("<u8").reshape(rows, wpr).copy(), wpr


def planes(levels, lane=512):
    t, wpr = pack((levels == 3).astype(np.uint8), lane)
    h, _ = pack((levels == 2).astype(np.uint8), lane)
    m, _ = pack(((levels == 0) | (levels == 3)).astype(np.uint8), lane)
    return t, h, m, wpr


def ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def main():
    lib = _lib.load()
    print("sms", lib.bitmm_device_sm_count())
    rng = np.random.default_rng(1)
    ok = True
    for (m, n, k) in [(1, 1, 1), (3, 5, 70), (130, 260, 300), (257, 129, 1000), (128, 256, 4096)]:
        a = rng.integers(0, 2, (m, k), dtype=np.uint8)
        b = rng.integers(0, 2, (n, k), dtype=np.uint8)
        aw, wpr = pack(a)
        bw, _ = pack(b)
        want = (2 * a.astype(np.int64) - 1) @ (2 * b.astype(np.int64) - 1).T
        got = np.zeros((m, n), np.int32)
        gotf = np.zeros((m, n), np.float32)
        rc = lib.bitmm_gemm_1x1_host(ptr(aw), m, ptr(bw), n, k, wpr, 0.5, 3.0, ptr(got), ptr(gotf), n)
        e1 = rc == 0 and np.array_equal(got, want) and np.array_equal(gotf, np.float32(1.5) * want.astype(np.float32))
        # 1x2
        lv = rng.integers(0, 4, (n, k), dtype=np.uint8)
        t, h, mm, _ = planes(lv)
        got12 = np.zeros((m, n), np.int32)
        rc2 = lib.bitmm_gemm_1x2_host(ptr(aw), m, 1.0, ptr(t), ptr(h), ptr(mm), n, k, wpr, 1.0, 0, 1.0,
                                      None, None, ptr(got12), None, n)
        want12 = 2 * ((2 * a.astype(np.int64) - 1) @ lv.astype(np.int64).T)
        e2 = rc2 == 0 and np.array_equal(got12, want12)
        # 2x2
        lw = rng.integers(0, 4, (m, k), dtype=np.uint8)
        wt, wh, wm, _ = planes(lw)
        got22 = np.zeros((m, n), np.int32)
        rc3 = lib.bitmm_gemm_2x2_host(ptr(wt), ptr(wh), ptr(wm), m, 1.0, 0, 1.0, ptr(t), ptr(h), ptr(mm), n, k,
                                      wpr, 1.0, 0, 1.0, None, None, ptr(got22), None, n)
        want22 = 4 * (lw.astype(np.int64) @ lv.astype(np.int64).T)
        e3 = rc3 == 0 and np.array_equal(got22, want22)
        # popc
        print(f"m={m} n={n} k={k}: 1x1 {e1} (rc {rc}) 1x2 {e2} (rc {rc2}) 2x2 {e3} (rc {rc3})",
              _lib.last_error() if not (e1 and e2 and e3) else "")
        if not e1:
            bad = np.argwhere(got != want)
            print("  1x1 mismatches", len(bad), bad[:5], got[tuple(bad[0])] if len(bad) else None,
                  want[tuple(bad[0])] if len(bad) else None)
        ok &= e1 and e2 and e3
    # APB small
    for (m, k, n) in [(3, 5, 7), (200, 768, 300)]:
        wbits = rng.integers(0, 2, (m, k), dtype=np.uint8)
        ww, wpr = pack(wbits)
        x = rng.standard_normal((k, n)).astype(np.float32)
        alpha = 0.37
        got = np.zeros((m, n), np.float32)
        rc = lib.bitmm_gemm_1x32_host(ptr(ww), m, k, wpr, alpha, None, ptr(x), n, n, ptr(got), n)
        want = alpha * ((2 * wbits.astype(np.float64) - 1) @ x.astype(np.float64))
        rel = np.linalg.norm(got - want) / np.linalg.norm(want)
        print(f"1x32 m={m} k={k} n={n} rc={rc} rel={rel:.3e}", _lib.last_error() if rc else "")
        ok &= rc == 0 and rel < 1e-5
    print("ALL OK" if ok else "FAILURES")

    import torch
    m = n = k = 4096
    a = torch.randint(0, 2**62, (m, k // 64), dtype=torch.int64, device="cuda")
    b = torch.randint(0, 2**62, (n, k // 64), dtype=torch.int64, device="cuda")
    c = torch.empty((m, n), dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for name, fn in [("tc", lib.bitmm_gemm_1x1_dev), ("popc", lib.bitmm_gemm_1x1_popc_dev)]:
        for _ in range(3):
            fn(a.data_ptr(), m, b.data_ptr(), n, k, k // 64, 1.0, 1.0, c.data_ptr(), None, n, s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record()
        for _ in range(reps):
            fn(a.data_ptr(), m, b.data_ptr(), n, k, k // 64, 1.0, 1.0, c.data_ptr(), None, n, s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"{name} 1x1 4096^3: {ms:.4f} ms  {m*n*k/ms/1e9:.1f} T-upd/s  launches={lib.bitmm_last_launch_count()}")
    c2 = c.clone()
    lib.bitmm_gemm_1x1_dev(a.data_ptr(), m, b.data_ptr(), n, k, k // 64, 1.0, 1.0, c2.data_ptr(), None, n, s)
    lib.bitmm_gemm_1x1_popc_dev(a.data_ptr(), m, b.data_ptr(), n, k, k // 64, 1.0, 1.0, c.data_ptr(), None, n, s)
    torch.cuda.synchronize()
    print("tc == popc at 4096^3:", torch.equal(c, c2))


if __name__ == "__main__":
    main()
