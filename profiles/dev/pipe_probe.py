"""Reproduce the host-call pipeline pattern with plain torch copies: per slice, H2D of the
slice's inputs + a short kernel on stream s, then D2H of its outputs in parts on stream d.
Variants: H2D on s (as the library), H2D on a third stream issued up front."""
import torch

SL, PARTS = 8, 4
n_in, n_out = 24 << 20, 64 << 20
hin = torch.empty(n_in, dtype=torch.uint8).pin_memory()
din = torch.empty(n_in, dtype=torch.uint8, device="cuda")
dout = torch.empty(n_out, dtype=torch.uint8, device="cuda")
hout = torch.empty(n_out, dtype=torch.uint8).pin_memory()
s, d, u = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def run(variant):
    a, b = n_in // SL, n_out // SL
    evs = []
    for i in range(SL):
        if variant == "h2d_on_s":
            with torch.cuda.stream(s):
                for p in range(3):
                    din[i * a + p * a // 3: i * a + (p + 1) * a // 3].copy_(hin[i * a + p * a // 3: i * a + (p + 1) * a // 3], non_blocking=True)
        else:
            with torch.cuda.stream(u):
                din[i * a:(i + 1) * a].copy_(hin[i * a:(i + 1) * a], non_blocking=True)
                e = torch.cuda.Event()
                e.record(u)
            s.wait_event(e)
        with torch.cuda.stream(s):
            torch.cuda._sleep(20000)  # ~10 us of "GEMM"
            e = torch.cuda.Event()
            e.record(s)
        d.wait_event(e)
        with torch.cuda.stream(d):
            for p in range(PARTS):
                o = i * b + p * b // PARTS
                hout[o:o + b // PARTS].copy_(dout[o:o + b // PARTS], non_blocking=True)


for variant in ("h2d_on_s", "h2d_on_u", "h2d_on_s", "h2d_on_u"):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.wait_stream(torch.cuda.current_stream()); u.wait_stream(torch.cuda.current_stream())
    run(variant)
    torch.cuda.current_stream().wait_stream(d)
    e1.record()
    torch.cuda.synchronize()
    print(f"{variant}: {e0.elapsed_time(e1):.3f} ms (D2H alone ~{n_out / 55e6:.3f} ms, H2D alone ~{n_in / 55e6:.3f})")
