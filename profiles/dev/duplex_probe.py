"""Do host->device and device->host copies on two streams overlap on this box's PCIe link?"""
import torch

n_d2h, n_h2d = 64 << 20, 24 << 20
dd = torch.empty(n_d2h, dtype=torch.uint8, device="cuda")
hd = torch.empty(n_d2h, dtype=torch.uint8).pin_memory()
dh = torch.empty(n_h2d, dtype=torch.uint8, device="cuda")
hh = torch.empty(n_h2d, dtype=torch.uint8).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
print("async engines:", torch.cuda.get_device_properties(0))


def timed(f):
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def d2h():
    with torch.cuda.stream(s1):
        hd.copy_(dd, non_blocking=True)


def h2d():
    with torch.cuda.stream(s2):
        dh.copy_(hh, non_blocking=True)


def both():
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    d2h()
    h2d()
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


def interleaved(parts=8):
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    a, b = n_d2h // parts, n_h2d // parts
    for p in range(parts):
        with torch.cuda.stream(s1):
            hd[p * a:(p + 1) * a].copy_(dd[p * a:(p + 1) * a], non_blocking=True)
        with torch.cuda.stream(s2):
            dh[p * b:(p + 1) * b].copy_(hh[p * b:(p + 1) * b], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


t1, t2, t3, t4 = timed(d2h), timed(h2d), timed(both), timed(interleaved)
print(f"D2H 64 MiB {t1:.3f} ms, H2D 24 MiB {t2:.3f} ms, both on two streams {t3:.3f} ms, "
      f"interleaved in 8 parts {t4:.3f} ms (serial would be {t1 + t2:.3f})")
