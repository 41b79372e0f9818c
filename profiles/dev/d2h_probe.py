"""PCIe device->host copy rate into pinned memory: one copy vs the same bytes in parts."""
import torch

for mib in (32, 64):
    n = mib << 20
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    for parts in (1, 8, 32):
        step = n // parts
        for _ in range(3):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for p in range(parts):
                h[p * step:(p + 1) * step].copy_(d[p * step:(p + 1) * step], non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"D2H {mib} MiB in {parts} parts: {ms:.3f} ms = {n / ms / 1e6:.1f} GB/s")
    for _ in range(3):
        e0.record(); d.copy_(h, non_blocking=True); e1.record(); torch.cuda.synchronize()
    print(f"H2D {mib} MiB: {e0.elapsed_time(e1):.3f} ms = {n / e0.elapsed_time(e1) / 1e6:.1f} GB/s")
