"""Generate tests/golden/*.npz from the UNMODIFIED reference library.

Run here (where /root/reference exists):  make -C oracle && python tests/golden/make_golden.py
The reference is compiled from /root/reference/proj/src by oracle/Makefile into
oracle/_ref/libbitmm_ref.so and called through oracle/ref_shim.cpp. The fixtures pin
both the C restatement (oracle/bitmm_oracle.c) and the CUDA path.

Case design follows the reference's own acceptance suite (acceptance.cpp:173-267, seed
2024 there; scale/gamma tables at :175-176) and its APB criterion (acceptance.cpp:335-387),
at sizes small enough to commit. Inputs are generated with numpy (seeded) and handed
to the reference as words, so nothing depends on libstdc++ random streams.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

import oracle  # noqa: E402
from paper_2306_08960_b200 import data  # noqa: E402

SCALES = [1.0, 0.5, 0.25, 0.75, 1.25, 0.3]   # acceptance.cpp:175
GAMMAS = [1.0, 0.5, 2.0, 1.25, 0.7]          # acceptance.cpp:176


def gemm_cases(ref: oracle.Ref, rng: np.random.Generator):
    shapes = []
    for _ in range(40):
        shapes.append((int(rng.integers(1, 41)), int(rng.integers(1, 301)), int(rng.integers(1, 41)), 512))
    for _ in range(6):
        shapes.append((int(rng.integers(1, 9)), int(rng.integers(257, 4097)), int(rng.integers(1, 9)), 512))
    for k in (1, 63, 64, 65, 127, 128, 129, 511, 512, 513):  # off-grid K (acceptance.cpp:135-136)
        shapes.append((3, k, 5, 512))
    for k in (1, 63, 70, 200):  # lane-width invariance (test_kernels.cpp:185-196)
        shapes.append((2, k, 2, 64))
    out = {}
    for i, (m, k, n, lane) in enumerate(shapes):
        a, wpr = data.random_words(rng, m, k, lane)
        b, _ = data.random_words(rng, n, k, lane)
        lw = data.random_levels(rng, m, k)
        la = data.random_levels(rng, n, k)
        wt, wh, wm, _ = data.planes_from_levels(lw, lane)
        at, ah, am, _ = data.planes_from_levels(la, lane)
        s_w, s_a = SCALES[rng.integers(6)], SCALES[rng.integers(6)]
        g_a, g_b, g_w = GAMMAS[rng.integers(5)], GAMMAS[rng.integers(5)], GAMMAS[rng.integers(5)]
        c11, _ = ref.gemm_1x1(a, b, k, wpr, g_a, g_b)
        c12, _ = ref.gemm_1x2(a, g_w, at, ah, am, k, wpr, s_a, g_a)
        c22, _ = ref.gemm_2x2(wt, wh, wm, at, ah, am, k, wpr, s_w, s_a, None, g_a)
        p = f"g{i:03d}_"
        out.update({
            p + "shape": np.array([m, k, n, wpr, lane], np.int64),
            p + "params": np.array([s_w, s_a, g_a, g_b, g_w], np.float32),
            p + "a": a, p + "b": b, p + "lw": lw, p + "la": la,
            p + "c11": c11, p + "c12": c12, p + "c22": c22,
        })
    out["gemm_count"] = np.array(len(shapes))
    return out


def apb_cases(ref: oracle.Ref, rng: np.random.Generator):
    out = {}
    count = 0
    for i in range(12):  # acceptance.cpp:344-379 at committed sizes
        m = int(rng.integers(1, 49))
        k = int(rng.integers(1, 201))
        n = int(rng.integers(1, 33))
        w = rng.uniform(-2.0, 2.0, (m, k)).astype(np.float32)
        alpha = np.float32(rng.uniform(0.2, 1.0))
        delta = np.float32(rng.uniform(0.05, 0.5))
        fwd = ref.apb_forward(w, float(alpha), float(delta))
        bin_, wpr, rp, ci, v = ref.decompose_apb(fwd, float(alpha))
        b = rng.uniform(-1.0, 1.0, (k, n)).astype(np.float32)
        c, _ = ref.layer_forward(m, k, float(alpha), bin_, wpr, rp, ci, v, b)
        c1x32, _ = ref.gemm_1x32(bin_, k, wpr, float(alpha), b)
        csp, _ = ref.spmm_csr(m, k, rp, ci, v, b)
        p = f"a{i:03d}_"
        out.update({
            p + "shape": np.array([m, k, n, wpr], np.int64),
            p + "alpha_delta": np.array([alpha, delta], np.float32),
            p + "w": w, p + "fwd": fwd, p + "bin": bin_, p + "row_ptr": rp, p + "col_idx": ci,
            p + "vals": v, p + "b": b, p + "c": c, p + "c1x32": c1x32, p + "cspmm": csp,
        })
        count += 1
    # per-row alpha (BASELINE config 4 shape family): rows are independent in the
    # reference (kernels.cpp:312-330, 341-350), so row r is a 1-row layer with alpha_r.
    for j in range(2):
        i = count
        m, k, n = 24, 96, 16
        a, alpha_vec, _ = data.apb_weights(rng, m, k, std=0.02, keep_frac=0.05)
        b = rng.standard_normal((k, n)).astype(np.float32)
        rows = []
        bins, rps, cis, vs = [], [0], [], []
        for r in range(m):
            bin_r, wpr, rp_r, ci_r, v_r = ref.decompose_apb(a[r:r + 1], float(alpha_vec[r]))
            c_r, _ = ref.layer_forward(1, k, float(alpha_vec[r]), bin_r, wpr, rp_r, ci_r, v_r, b)
            rows.append(c_r)
            bins.append(bin_r)
            cis.append(ci_r)
            vs.append(v_r)
            rps.append(rps[-1] + int(rp_r[-1]))
        p = f"a{i:03d}_"
        out.update({
            p + "shape": np.array([m, k, n, wpr], np.int64),
            p + "alpha_vec": alpha_vec.astype(np.float32), p + "fwd": a,
            p + "bin": np.concatenate(bins, 0), p + "row_ptr": np.asarray(rps, np.uint64),
            p + "col_idx": np.concatenate(cis).astype(np.uint64),
            p + "vals": np.concatenate(vs).astype(np.float32), p + "b": b,
            p + "c": np.concatenate(rows, 0),
        })
        count += 1
    out["apb_count"] = np.array(count)
    return out


def packing_cases(ref: oracle.Ref, rng: np.random.Generator):
    out = {}
    for i, (rows, cols, lane) in enumerate([(3, 5, 512), (7, 130, 512), (4, 70, 64), (2, 1000, 512)]):
        a = rng.standard_normal((rows, cols)).astype(np.float32)
        a[0, 0] = 0.0  # sign(0) = +1 (tensor.cpp:161)
        a[0, -1] = -0.0
        words, wpr = ref.pack_signs(a, lane)
        x = (rng.uniform(-0.2, 2.0, (rows, cols)) * 1.0).astype(np.float32)
        x[0, 0] = 0.25  # exact half-step tie (lround away from zero)
        x[-1, -1] = 0.75
        lv = ref.quantize_2bit(x, 0.5)
        t, h, m, _ = ref.decompose_thm(lv, 0.5, lane)
        p = f"p{i:03d}_"
        out.update({p + "shape": np.array([rows, cols, lane, wpr], np.int64), p + "a": a,
                    p + "signs": words, p + "x": x, p + "levels": lv, p + "t": t, p + "h": h,
                    p + "m": m})
    out["pack_count"] = np.array(4)
    # row ops (kernels.cpp:120-140)
    dots = []
    for n in (1, 3, 63, 64, 65, 200):
        words = (n + 63) // 64
        u, _ = data.random_words(rng, 1, n, 64)
        v, _ = data.random_words(rng, 1, n, 64)
        z, _ = data.random_words(rng, 1, n, 64)
        dots.append((n, u[0], v[0], z[0], ref.dot_binary(u[0], v[0], n), ref.mbm(u[0], v[0], z[0])))
        assert u.shape[1] == words
    for j, (n, u, v, z, d, mb) in enumerate(dots):
        p = f"r{j:03d}_"
        out.update({p + "n": np.array(n), p + "u": u, p + "v": v, p + "z": z,
                    p + "dot": np.array(d), p + "mbm": np.array(mb)})
    out["row_count"] = np.array(len(dots))
    return out


def main():
    ref = oracle.Ref()
    rng = np.random.default_rng(2024)
    np.savez_compressed(os.path.join(HERE, "gemm_cases.npz"), **gemm_cases(ref, rng))
    np.savez_compressed(os.path.join(HERE, "apb_cases.npz"), **apb_cases(ref, rng))
    np.savez_compressed(os.path.join(HERE, "packing_cases.npz"), **packing_cases(ref, rng))
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)), "bytes")


if __name__ == "__main__":
    main()
