"""GPU flows of the reference CLI (tools/bitmm_main.cpp): `pack` and `bench`.

    python -m paper_2306_08960_b200.cli pack --input w.btsr --output w.bits --mode sign
    python -m paper_2306_08960_b200.cli pack --input x.btsr --output x --mode thm --step 0.5
    python -m paper_2306_08960_b200.cli bench --routine 1x1 --m 4096 --k 4096 --n 4096 --csv out.csv

`pack` (cmd_pack, bitmm_main.cpp:182-222) loads the dense container straight into device memory
(bitmm_btsr_load_dev), packs it with the GPU packers (pack.cuh) and writes the same containers
the reference writes (pack_signs -> store_tensor; quantize_uniform_2bit + decompose_thm ->
store_thm_planes; apb_forward + decompose_apb -> store_apb_layer, on the GPU decompose_apb). `bench` (cmd_bench, bitmm_main.cpp:64-104; bench_routine, bench.cpp:90-185)
times the routines on the GPU with operands resident in HBM and writes the reference's CSV
columns (write_csv_header / write_csv_record, bench.cpp:188-200). The reference's `verify`,
`tpp`, `apb-stats` and `shapes` stay host-side (out of scope).
Exit codes follow the reference: 0 ok, 2 usage, 3 I/O.
"""
from __future__ import annotations

import argparse
import sys

import numpy as np

EXIT_OK, EXIT_USAGE, EXIT_IO = 0, 2, 3
ROUTINES = ("1x1", "1x2", "2x2", "spmm", "1x32_ref")
CSV_HEADER = "routine,m,k,n,reps,warmup,threads,simd,seconds,gops,gflops,tpp_gops,pct_tpp\n"



# ---- CLI-only: the reference CLI's `pack --mode apb` parameter step (bitmm_main.cpp:195-207).
# Training-side APB helpers (apb.cpp:50-55, 191-210), OUT OF SCOPE for the hot path (SURVEY.md
# §2 row 6); kept here, at the one place that needs them, so `pack` writes the same files as
# the reference CLI. Nothing on the GEMM / layer path calls them.
DELTA_MIN = np.float32(1e-8)  # kDeltaMin, apb.hpp:16


def init_alpha_delta(w: np.ndarray):
    """init_alpha_delta (apb.cpp:191-210): alpha = mean |w|, delta = max(3 * population std,
    1e-8), both accumulated in double in storage order (sequential sums, as the reference)."""
    v = np.ascontiguousarray(w, np.float32).reshape(-1).astype(np.float64)
    n = v.size
    if n == 0:
        raise ValueError("empty weight matrix")
    abs_sum = float(np.cumsum(np.abs(v))[-1])  # cumsum: one running sum, element order
    mean = float(np.cumsum(v)[-1]) / n
    var = float(np.cumsum((v - mean) ** 2)[-1]) / n
    alpha = np.float32(abs_sum / n)
    delta = max(np.float32(3.0 * np.sqrt(var)), DELTA_MIN)
    return alpha, np.float32(delta)


def check_apb_params(alpha, delta) -> None:
    """ApbParams::validate (apb.cpp:50-55)."""
    if not alpha > 0.0:
        raise ValueError("alpha must be positive")
    if not delta >= DELTA_MIN:
        raise ValueError("delta must be at least the 1e-8 floor")
    if not (np.isfinite(alpha) and np.isfinite(delta)):
        raise ValueError("alpha and delta must be finite")


def cmd_pack(args) -> int:
    import torch
    from . import api, btsr, device
    d = btsr.load_dev(args.input, "dense")
    x = d["data"]
    rows, cols = x.shape
    if args.mode == "sign":
        words = device.pack_signs(x, args.lane_bits)
        device.status()
        wpr = words.shape[1]
        bm = api.BitMatrix.from_words(rows, cols, wpr, words.cpu().numpy().view(np.uint64))
        btsr.store_tensor(args.output, bm)
        print(f"packed signs: {rows} x {cols} -> {args.output}")
    elif args.mode == "thm":
        if args.step is None:
            raise ValueError("--step is required for thm packing")
        t, h, m = device.quantize_thm(x, args.step, args.lane_bits)
        device.status()
        wpr = t.shape[1]
        bm = lambda w: api.BitMatrix.from_words(rows, cols, wpr, w.cpu().numpy().view(np.uint64))  # noqa: E731
        btsr.store_thm_planes(args.output, api.ThmPlanes(bm(t), bm(h), bm(m), scale=float(args.step)))
        print(f"packed planes: {rows} x {cols} step={args.step:g} -> "
              f"{args.output}.{{t,h,m}}.btsr + {args.output}.json")
    elif args.mode == "apb":
        # bitmm_main.cpp:195-207: params given or init_alpha_delta, apb_forward, decompose_apb
        if (args.alpha is None) != (args.delta is None):
            raise ValueError("--alpha and --delta must be given together")
        if args.alpha is not None:
            alpha, delta = np.float32(args.alpha), np.float32(args.delta)
        else:
            alpha, delta = init_alpha_delta(x.cpu().numpy())
        check_apb_params(alpha, delta)
        bound = np.float32(alpha + delta)  # float add, apb.cpp:59
        sign_alpha = torch.where(x >= 0, torch.tensor(float(alpha), device=x.device),
                                 torch.tensor(-float(alpha), device=x.device))
        fwd = torch.where(x.abs() <= float(bound), sign_alpha, x).contiguous()  # apb_forward
        words, rp, ci, vals = device.decompose_apb(fwd, float(alpha), args.lane_bits)
        device.status()
        wpr = words.shape[1]
        bm = api.BitMatrix.from_words(rows, cols, wpr, words.cpu().numpy().view(np.uint64))
        res = api.CsrMatrix.create(rows, cols, rp.cpu().numpy().view(np.uint64),
                                   ci.cpu().numpy().view(np.uint64), vals.cpu().numpy())
        btsr.store_apb_layer(args.output, bm, res, float(alpha))
        print(f"packed layer: {rows} x {cols} alpha={float(alpha):g} nnz={res.nnz()} -> "
              f"{args.output}.{{bin,res}}.btsr + {args.output}.json")
    else:
        raise ValueError(f"unknown pack mode: {args.mode} (GPU modes: sign|thm|apb)")
    torch.cuda.synchronize()
    return EXIT_OK


def _square(text: str):
    try:
        lo_s, rest = text.split("..")
        hi_s, _, step_s = rest.partition(":")
        lo, hi = int(lo_s), int(hi_s)
        step = int(step_s) if step_s else lo
    except ValueError:
        raise ValueError("--square: expected LO..HI[:STEP]") from None
    if lo <= 0 or hi < lo or step <= 0:
        raise ValueError("--square: range must satisfy 0 < LO <= HI, STEP > 0")
    return list(range(lo, hi + 1, step))


def bench_routine(routine: str, m: int, k: int, n: int, reps: int, warmup: int, seed: int,
                  density: float) -> dict:
    """bench_routine (bench.cpp:90-185) on the GPU: operands built once outside the timed
    region and resident in HBM, output preallocated, median of `reps` CUDA-event timings."""
    import torch
    from . import data, device
    rng = np.random.default_rng(seed)
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()  # noqa: E731
    if routine == "1x1":
        a, _ = data.random_words(rng, m, k)
        b, _ = data.random_words(rng, n, k)
        da, db = T(a), T(b)
        out = torch.empty((m, n), dtype=torch.float32, device="cuda")
        run = lambda: device.gemm_1x1(da, db, k, out=out)  # noqa: E731
    elif routine == "1x2":
        a, _ = data.random_words(rng, m, k)
        t, h, mm, _ = data.random_planes(rng, n, k)
        da, dt, dh, dm = T(a), T(t), T(h), T(mm)
        out = torch.empty((m, n), dtype=torch.float32, device="cuda")
        run = lambda: device.gemm_1x2(da, 1.0, dt, dh, dm, k, a_scale=0.5, out=out)  # noqa: E731
    elif routine == "2x2":
        wt, wh, wm, _ = data.random_planes(rng, m, k)
        t, h, mm, _ = data.random_planes(rng, n, k)
        d = [T(x) for x in (wt, wh, wm, t, h, mm)]
        out = torch.empty((m, n), dtype=torch.float32, device="cuda")
        run = lambda: device.gemm_2x2(*d, k, w_scale=0.25, a_scale=0.5, out=out)  # noqa: E731
    elif routine == "spmm":
        mask = rng.random((m, k)) < density
        r_idx, c_idx = np.nonzero(mask)
        rp = np.zeros(m + 1, np.int64)
        np.add.at(rp, r_idx + 1, 1)
        rp = np.cumsum(rp)
        vals = rng.uniform(-1, 1, r_idx.size).astype(np.float32)
        b = rng.uniform(-1, 1, (k, n)).astype(np.float32)
        drp, dci = torch.from_numpy(rp).cuda(), torch.from_numpy(c_idx.astype(np.int64)).cuda()
        dv, dbm = torch.from_numpy(vals).cuda(), torch.from_numpy(b).cuda()
        out = torch.empty((m, n), dtype=torch.float32, device="cuda")
        run = lambda: device.spmm_csr(m, k, drp, dci, dv, dbm, out)  # noqa: E731
    elif routine == "1x32_ref":
        a, _ = data.random_words(rng, m, k)
        b = rng.uniform(-1, 1, (k, n)).astype(np.float32)
        da, dbm = T(a), torch.from_numpy(b).cuda()
        out = torch.empty((m, n), dtype=torch.float32, device="cuda")
        run = lambda: device.gemm_1x32(da, k, 1.0, dbm, out)  # noqa: E731
    else:
        raise ValueError(f"unknown routine: {routine} (GPU routines: {'|'.join(ROUTINES)})")
    for _ in range(warmup):
        run()
    torch.cuda.synchronize()
    device.status()
    times = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e-3)
    device.status()
    times.sort()
    mid = len(times) // 2
    seconds = times[mid] if len(times) % 2 else 0.5 * (times[mid - 1] + times[mid])  # median()
    gops = m * k * n / seconds / 1e9  # bench.cpp:175
    return dict(routine=routine, m=m, k=k, n=n, reps=reps, warmup=warmup, threads=1,
                simd="b200-tcgen05", seconds=seconds, gops=gops, gflops=2.0 * gops)


def csv_record(rec: dict) -> str:
    """write_csv_record (bench.cpp:192-200); tpp columns stay empty (no CPU SIMD model)."""
    return (f"{rec['routine']},{rec['m']},{rec['k']},{rec['n']},{rec['reps']},{rec['warmup']},"
            f"{rec['threads']},{rec['simd']},{rec['seconds']:g},{rec['gops']:g},{rec['gflops']:g},,\n")


def cmd_bench(args) -> int:
    problems = [(d, d, d) for d in _square(args.square)] if args.square else [(args.m, args.k, args.n)]
    routines = args.routine or ["1x1", "1x2", "2x2"]
    for r in routines:
        if r not in ROUTINES:
            raise ValueError(f"unknown routine: {r}")
    csv = open(args.csv, "w") if args.csv else None
    try:
        if csv:
            csv.write(CSV_HEADER)
        for (m, k, n) in problems:
            for r in routines:
                rec = bench_routine(r, m, k, n, args.reps, args.warmup, args.seed, args.density)
                print(f"{r:<9s} m={m} k={k} n={n} simd={rec['simd']} threads=1 "
                      f"median={rec['seconds']:.6f}s gops={rec['gops']:.3f}")
                if csv:
                    csv.write(csv_record(rec))
    finally:
        if csv:
            csv.close()
    return EXIT_OK


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="bitmm-b200", description="GPU flows of the bitmm CLI")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("pack", help="convert a dense container to a packed form on the GPU")
    p.add_argument("--input", required=True)
    p.add_argument("--output", required=True)
    p.add_argument("--mode", default="sign")
    p.add_argument("--step", type=float)
    p.add_argument("--alpha", type=float)
    p.add_argument("--delta", type=float)
    p.add_argument("--lane-bits", type=int, default=512)
    b = sub.add_parser("bench", help="time routines on the GPU and report gops")
    b.add_argument("--routine", action="append")
    b.add_argument("--m", type=int, default=1024)
    b.add_argument("--k", type=int, default=1024)
    b.add_argument("--n", type=int, default=1024)
    b.add_argument("--square")
    b.add_argument("--reps", type=int, default=9)
    b.add_argument("--warmup", type=int, default=2)
    b.add_argument("--seed", type=int, default=1)
    b.add_argument("--density", type=float, default=0.02)
    b.add_argument("--csv")
    args = ap.parse_args(argv)
    from .api import IoError
    try:
        return cmd_pack(args) if args.cmd == "pack" else cmd_bench(args)
    except IoError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_IO
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
