"""A library block-scaled FP4 GEMM beside tc_gemm: torch._scaled_mm on e2m1 operands with
E8M0 block scales (cuBLASLt on sm_100), at 4096^3 and 4096 x 8192 x 4096, median of 20
L2-flushed launches. Prints one JSON line per shape (or the error if this build lacks it)."""
import json

import torch


def to_blocked(s):
    """cuBLAS block-scaled layout of a [rows, cols] scale matrix (128 x 4 tiles, 32-4-4 order)."""
    rows, cols = s.shape
    rb, cb = (rows + 127) // 128, (cols + 3) // 4
    p = torch.zeros((rb * 128, cb * 4), dtype=s.dtype, device=s.device)
    p[:rows, :cols] = s
    blocks = p.view(rb, 128, cb, 4).permute(0, 2, 1, 3)
    return blocks.reshape(-1, 4, 32, 4).transpose(1, 2).reshape(-1, 32, 16).flatten()


def run(m, n, k):
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(1)
    a = torch.randint(0, 256, (m, k // 2), dtype=torch.uint8, device=dev, generator=g).view(torch.float4_e2m1fn_x2)
    b = torch.randint(0, 256, (n, k // 2), dtype=torch.uint8, device=dev, generator=g).view(torch.float4_e2m1fn_x2)
    sa = to_blocked(torch.full((m, k // 32), 127, dtype=torch.uint8, device=dev)).view(torch.float8_e8m0fnu)
    sb = to_blocked(torch.full((n, k // 32), 127, dtype=torch.uint8, device=dev)).view(torch.float8_e8m0fnu)
    import torch.nn.functional as F
    try:
        f = lambda: torch._scaled_mm(a, b.t(), sa, sb, out_dtype=torch.bfloat16)  # noqa: E731
        out = f()
        api = "torch._scaled_mm"
    except RuntimeError:
        # torch >= 2.10: the recipe-based entry point (MX block-32 E8M0, cuBLAS 32-4-4 swizzle)
        f = lambda: F.scaled_mm(a, b.t(), sa, F.ScalingType.BlockWise1x32, sb, F.ScalingType.BlockWise1x32,  # noqa: E731
                                swizzle_a=F.SwizzleType.SWIZZLE_32_4_4, swizzle_b=F.SwizzleType.SWIZZLE_32_4_4,
                                output_dtype=torch.bfloat16)
        out = f()
        api = "torch.nn.functional.scaled_mm (BlockWise1x32, SWIZZLE_32_4_4)"
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ts = []
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    return {"library": f"{api} (cuBLASLt) e2m1 x e2m1, E8M0 block-32 scales, bf16 out",
            "m": m, "n": n, "k": k, "ms": ms, "tflops": 2 * m * n * k / (ms * 1e-3) / 1e12,
            "out_dtype": str(out.dtype)}


for shape in ((4096, 4096, 4096), (4096, 8192, 4096), (8192, 8192, 8192)):
    try:
        print(json.dumps(run(*shape)), flush=True)
    except Exception as e:  # the build may not expose FP4 scaled_mm
        print(json.dumps({"shape": shape, "error": repr(e)[:1500]}), flush=True)
