"""Parity checkers for the sm_100a bitwise-GEMM path — TEST INFRASTRUCTURE ONLY.

Two independent CPU implementations, both loaded through ctypes:

* `Oracle`  — oracle/liboracle.so, the plain-C restatement in bitmm_oracle.c (every
  function cites the reference file:line it follows).
* `Ref`     — oracle/_ref/libbitmm_ref.so, the UNMODIFIED reference library compiled
  from /root/reference/proj/src by oracle/Makefile, behind ref_shim.cpp's C ABI.
  Present wherever it was built (here, and on the GPU box as a prebuilt file).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference`
legs may import this package. The product path (paper_2306_08960_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libbitmm_ref.so")

_p = C.c_void_p
_i64 = C.c_int64
_f = C.c_float
_i = C.c_int


def _ptr(a):
    return None if a is None else np.ascontiguousarray(a).ctypes.data_as(C.c_void_p)


def build(force: bool = False) -> None:
    """Compile liboracle.so (always) and _ref/ (only when /root/reference exists)."""
    args = ["make", "-C", HERE, "-s"]
    if force:
        args.append("-B")
    subprocess.run(args, check=True)


class Oracle:
    """ctypes view of bitmm_oracle.c."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        lib = C.CDLL(path)
        sig = {
            "oracle_gemm_1x1": (None, [_p, _i64, _p, _i64, _i64, _i64, _f, _f, _p, _p]),
            "oracle_gemm_1x2": (None, [_p, _i64, _f, _p, _p, _p, _i64, _i64, _i64, _f, _i, _f,
                                       _p, _p, _p, _p]),
            "oracle_gemm_2x2": (None, [_p, _p, _p, _i64, _f, _i, _f, _p, _p, _p, _i64, _i64,
                                       _i64, _f, _i, _f, _p, _p, _p, _p]),
            "oracle_gemm_1x32": (None, [_p, _i64, _i64, _i64, _f, _p, _p, _i64, _i64, _p]),
            "oracle_spmm_csr": (None, [_i64, _p, _p, _p, _p, _i64, _i64, _p]),
            "oracle_layer_forward": (None, [_i64, _i64, _f, _p, _p, _i64, _p, _p, _p, _p, _i64,
                                            _i64, _p]),
            "oracle_layer_forward_2bit": (None, [_i64, _i64, _f, _p, _p, _i64, _p, _p, _p, _p,
                                                 _p, _p, _i64, _f, _i, _f, _p]),
            "oracle_padded_words": (_i64, [_i64, _i]),
            "oracle_pack_signs": (None, [_p, _i64, _i64, _i64, _p]),
            "oracle_decompose_thm": (None, [_p, _i64, _i64, _i64, _p, _p, _p]),
            "oracle_quantize_2bit": (None, [_p, _i64, _f, _p]),
            "oracle_apb_forward": (None, [_p, _i64, _f, _f, _p]),
            "oracle_decompose_apb": (_i64, [_p, _i64, _i64, _f, _i64, _p, _p, _p, _p]),
            "oracle_dot_binary": (_i64, [_p, _p, _i64, _i64]),
            "oracle_mbm": (_i64, [_p, _p, _p, _i64]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        self.lib = lib

    # ---- GEMMs: return (int32 units, float32 out) ----
    def gemm_1x1(self, a, b, k, wpr, gamma_a=1.0, gamma_b=1.0):
        m, n = a.shape[0], b.shape[0]
        u = np.empty((m, n), np.int32)
        o = np.empty((m, n), np.float32)
        self.lib.oracle_gemm_1x1(_ptr(a), m, _ptr(b), n, k, wpr, gamma_a, gamma_b, _ptr(u), _ptr(o))
        return u, o

    def gemm_1x2(self, w, gamma, t, h, mm, k, wpr, a_scale=1.0, a_gamma=None, row_scale=None,
                 col_scale=None):
        m, n = w.shape[0], t.shape[0]
        u = np.empty((m, n), np.int32)
        o = np.empty((m, n), np.float32)
        self.lib.oracle_gemm_1x2(_ptr(w), m, gamma, _ptr(t), _ptr(h), _ptr(mm), n, k, wpr,
                                 a_scale, int(a_gamma is not None),
                                 1.0 if a_gamma is None else a_gamma,
                                 _ptr(None if row_scale is None else row_scale.astype(np.float32)),
                                 _ptr(None if col_scale is None else col_scale.astype(np.float32)),
                                 _ptr(u), _ptr(o))
        return u, o

    def gemm_2x2(self, wt, wh, wm, at, ah, am, k, wpr, w_scale=1.0, a_scale=1.0, w_gamma=None,
                 a_gamma=None, row_scale=None, col_scale=None):
        m, n = wt.shape[0], at.shape[0]
        u = np.empty((m, n), np.int32)
        o = np.empty((m, n), np.float32)
        self.lib.oracle_gemm_2x2(_ptr(wt), _ptr(wh), _ptr(wm), m, w_scale, int(w_gamma is not None),
                                 1.0 if w_gamma is None else w_gamma, _ptr(at), _ptr(ah), _ptr(am),
                                 n, k, wpr, a_scale, int(a_gamma is not None),
                                 1.0 if a_gamma is None else a_gamma,
                                 _ptr(None if row_scale is None else row_scale.astype(np.float32)),
                                 _ptr(None if col_scale is None else col_scale.astype(np.float32)),
                                 _ptr(u), _ptr(o))
        return u, o

    def gemm_1x32(self, w, k, wpr, gamma, b, row_gamma=None):
        m, n = w.shape[0], b.shape[1]
        o = np.empty((m, n), np.float32)
        rg = None if row_gamma is None else np.ascontiguousarray(row_gamma, np.float32)
        self.lib.oracle_gemm_1x32(_ptr(w), m, k, wpr, gamma, _ptr(rg), _ptr(b), n, b.shape[1],
                                  _ptr(o))
        return o

    def spmm_csr(self, rows, row_ptr, col_idx, vals, b):
        n = b.shape[1]
        o = np.empty((rows, n), np.float32)
        self.lib.oracle_spmm_csr(rows, _ptr(row_ptr), _ptr(col_idx), _ptr(vals), _ptr(b), n, n,
                                 _ptr(o))
        return o

    def layer_forward(self, rows, cols, alpha, bin_words, wpr, row_ptr, col_idx, vals, b,
                      row_alpha=None):
        n = b.shape[1]
        o = np.empty((rows, n), np.float32)
        ra = None if row_alpha is None else np.ascontiguousarray(row_alpha, np.float32)
        self.lib.oracle_layer_forward(rows, cols, alpha, _ptr(ra), _ptr(bin_words), wpr,
                                      _ptr(row_ptr), _ptr(col_idx), _ptr(vals), _ptr(b), n, n,
                                      _ptr(o))
        return o

    # ---- packing ----
    def layer_forward_2bit(self, rows, cols, alpha, bin_words, wpr, row_ptr, col_idx, vals, t, h,
                           mm, a_scale=1.0, a_gamma=None, row_alpha=None):
        n = t.shape[0]
        o = np.empty((rows, n), np.float32)
        ra = None if row_alpha is None else np.ascontiguousarray(row_alpha, np.float32)
        self.lib.oracle_layer_forward_2bit(rows, cols, alpha, _ptr(ra), _ptr(bin_words), wpr,
                                           _ptr(row_ptr), _ptr(col_idx), _ptr(vals), _ptr(t),
                                           _ptr(h), _ptr(mm), n, a_scale,
                                           int(a_gamma is not None),
                                           1.0 if a_gamma is None else a_gamma, _ptr(o))
        return o

    def pack_signs(self, a, lane_bits=512):
        rows, cols = a.shape
        wpr = self.lib.oracle_padded_words(cols, lane_bits)
        w = np.zeros((rows, wpr), np.uint64)
        self.lib.oracle_pack_signs(_ptr(np.ascontiguousarray(a, np.float32)), rows, cols, wpr, _ptr(w))
        return w, wpr

    def decompose_thm(self, levels, lane_bits=512):
        rows, cols = levels.shape
        wpr = self.lib.oracle_padded_words(cols, lane_bits)
        t, h, m = (np.zeros((rows, wpr), np.uint64) for _ in range(3))
        self.lib.oracle_decompose_thm(_ptr(np.ascontiguousarray(levels, np.uint8)), rows, cols, wpr,
                                      _ptr(t), _ptr(h), _ptr(m))
        return t, h, m, wpr

    def quantize_2bit(self, a, s):
        a = np.ascontiguousarray(a, np.float32)
        out = np.empty(a.shape, np.uint8)
        self.lib.oracle_quantize_2bit(_ptr(a), a.size, s, _ptr(out))
        return out

    def apb_forward(self, w, alpha, delta):
        w = np.ascontiguousarray(w, np.float32)
        out = np.empty_like(w)
        self.lib.oracle_apb_forward(_ptr(w), w.size, alpha, delta, _ptr(out))
        return out

    def decompose_apb(self, a, alpha, lane_bits=512):
        """Returns (bin words, wpr, row_ptr, col_idx, vals); alpha scalar or per-row."""
        a = np.ascontiguousarray(a, np.float32)
        rows, cols = a.shape
        wpr = self.lib.oracle_padded_words(cols, lane_bits)
        if np.ndim(alpha) == 0:
            bin_ = np.zeros((rows, wpr), np.uint64)
            rp = np.zeros(rows + 1, np.uint64)
            nnz = self.lib.oracle_decompose_apb(_ptr(a), rows, cols, float(alpha), wpr, _ptr(bin_),
                                                _ptr(rp), None, None)
            ci = np.zeros(max(nnz, 1), np.uint64)
            v = np.zeros(max(nnz, 1), np.float32)
            self.lib.oracle_decompose_apb(_ptr(a), rows, cols, float(alpha), wpr, _ptr(bin_),
                                          _ptr(rp), _ptr(ci), _ptr(v))
            return bin_, wpr, rp, ci[:nnz], v[:nnz]
        # per-row alpha: split each row with its own alpha (rows are independent)
        bins, rps, cis, vs = [], [0], [], []
        for r in range(rows):
            b_r, _, rp_r, ci_r, v_r = self.decompose_apb(a[r:r + 1], float(alpha[r]), lane_bits)
            bins.append(b_r)
            cis.append(ci_r)
            vs.append(v_r)
            rps.append(rps[-1] + int(rp_r[-1]))
        return (np.concatenate(bins, 0), wpr, np.asarray(rps, np.uint64),
                np.concatenate(cis).astype(np.uint64), np.concatenate(vs).astype(np.float32))

    def dot_binary(self, u, v, n):
        return self.lib.oracle_dot_binary(_ptr(u), _ptr(v), u.size, n)

    def mbm(self, x, y, z):
        return self.lib.oracle_mbm(_ptr(x), _ptr(y), _ptr(z), x.size)


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"reference error {code}: {msg}")
        self.code = code


class Ref:
    """ctypes view of the unmodified reference library (ref_shim.cpp). Each GEMM returns
    (float32 out, seconds spent inside the reference call)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        lib = C.CDLL(path)
        pd = C.POINTER(C.c_double)
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_set_simd": (_i, [C.c_char_p]),
            "ref_active_simd": (C.c_char_p, []),
            "ref_gemm_1x1": (_i, [_p, _i64, _p, _i64, _i64, _i64, _f, _f, _i, _p, pd]),
            "ref_gemm_1x2": (_i, [_p, _i64, _f, _p, _p, _p, _i64, _i64, _i64, _f, _i, _f, _i, _p, pd]),
            "ref_gemm_2x2": (_i, [_p, _p, _p, _i64, _f, _i, _f, _p, _p, _p, _i64, _i64, _i64, _f, _i,
                                  _f, _i, _p, pd]),
            "ref_gemm_1x32": (_i, [_p, _i64, _i64, _i64, _f, _p, _i64, _i, _p, pd]),
            "ref_spmm_csr": (_i, [_i64, _i64, _p, _p, _p, _i64, _p, _i64, _i, _p, pd]),
            "ref_layer_forward": (_i, [_i64, _i64, _f, _p, _i64, _p, _p, _p, _i64, _p, _i64, _i, _p, pd]),
            "ref_apb_forward": (_i, [_p, _i64, _i64, _f, _f, _p]),
            "ref_pack_apb": (_i, [_p, _i64, _i64, _i, C.POINTER(_f), C.POINTER(_f), C.c_char_p]),
            "ref_decompose_apb": (_i, [_p, _i64, _i64, _f, _i, _p, C.POINTER(_i64), _p, _p, _p,
                                       C.POINTER(_i64)]),
            "ref_pack_signs": (_i, [_p, _i64, _i64, _i, _p, C.POINTER(_i64)]),
            "ref_store_dense": (_i, [C.c_char_p, _p, _i64, _i64]),
            "ref_store_bit": (_i, [C.c_char_p, _p, _i64, _i64, _i64]),
            "ref_store_csr": (_i, [C.c_char_p, _i64, _i64, _p, _p, _p, _i64]),
            "ref_store_thm_planes": (_i, [C.c_char_p, _p, _p, _p, _i64, _i64, _i64, _f, _i, _f]),
            "ref_load_check": (_i, [C.c_char_p, _i]),
            "ref_decompose_thm": (_i, [_p, _i64, _i64, _f, _i, _p, _p, _p, C.POINTER(_i64)]),
            "ref_quantize_2bit": (_i, [_p, _i64, _i64, _f, _p]),
            "ref_dot_binary": (_i, [_p, _p, _i64, _i64, C.POINTER(_i64)]),
            "ref_mbm": (_i, [_p, _p, _p, _i64, C.POINTER(_i64)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        self.lib = lib

    def _check(self, rc):
        if rc != 0:
            raise RefError(rc, self.lib.ref_last_error().decode())

    def set_simd(self, level: str) -> None:
        self._check(self.lib.ref_set_simd(level.encode()))

    def active_simd(self) -> str:
        return self.lib.ref_active_simd().decode()

    def gemm_1x1(self, a, b, k, wpr, gamma_a=1.0, gamma_b=1.0, threads=1):
        m, n = a.shape[0], b.shape[0]
        o = np.empty((m, n), np.float32)
        s = C.c_double(0)
        self._check(self.lib.ref_gemm_1x1(_ptr(a), m, _ptr(b), n, k, wpr, gamma_a, gamma_b, threads,
                                          _ptr(o), C.byref(s)))
        return o, s.value

    def gemm_1x2(self, w, gamma, t, h, mm, k, wpr, a_scale=1.0, a_gamma=None, threads=1):
        m, n = w.shape[0], t.shape[0]
        o = np.empty((m, n), np.float32)
        s = C.c_double(0)
        self._check(self.lib.ref_gemm_1x2(_ptr(w), m, gamma, _ptr(t), _ptr(h), _ptr(mm), n, k, wpr,
                                          a_scale, int(a_gamma is not None),
                                          1.0 if a_gamma is None else a_gamma, threads, _ptr(o),
                                          C.byref(s)))
        return o, s.value

    def gemm_2x2(self, wt, wh, wm, at, ah, am, k, wpr, w_scale=1.0, a_scale=1.0, w_gamma=None,
                 a_gamma=None, threads=1):
        m, n = wt.shape[0], at.shape[0]
        o = np.empty((m, n), np.float32)
        s = C.c_double(0)
        self._check(self.lib.ref_gemm_2x2(_ptr(wt), _ptr(wh), _ptr(wm), m, w_scale,
                                          int(w_gamma is not None), 1.0 if w_gamma is None else w_gamma,
                                          _ptr(at), _ptr(ah), _ptr(am), n, k, wpr, a_scale,
                                          int(a_gamma is not None), 1.0 if a_gamma is None else a_gamma,
                                          threads, _ptr(o), C.byref(s)))
        return o, s.value

    def gemm_1x32(self, w, k, wpr, gamma, b, threads=1):
        m, n = w.shape[0], b.shape[1]
        o = np.empty((m, n), np.float32)
        s = C.c_double(0)
        self._check(self.lib.ref_gemm_1x32(_ptr(w), m, k, wpr, gamma, _ptr(b), n, threads, _ptr(o),
                                           C.byref(s)))
        return o, s.value

    def spmm_csr(self, rows, cols, row_ptr, col_idx, vals, b, threads=1):
        n = b.shape[1]
        o = np.empty((rows, n), np.float32)
        s = C.c_double(0)
        self._check(self.lib.ref_spmm_csr(rows, cols, _ptr(row_ptr), _ptr(col_idx), _ptr(vals),
                                          int(row_ptr[-1]), _ptr(b), n, threads, _ptr(o), C.byref(s)))
        return o, s.value

    def layer_forward(self, rows, cols, alpha, bin_words, wpr, row_ptr, col_idx, vals, b, threads=1):
        n = b.shape[1]
        o = np.empty((rows, n), np.float32)
        s = C.c_double(0)
        self._check(self.lib.ref_layer_forward(rows, cols, alpha, _ptr(bin_words), wpr, _ptr(row_ptr),
                                               _ptr(col_idx), _ptr(vals), int(row_ptr[-1]), _ptr(b),
                                               n, threads, _ptr(o), C.byref(s)))
        return o, s.value

    def apb_forward(self, w, alpha, delta):
        w = np.ascontiguousarray(w, np.float32)
        o = np.empty_like(w)
        self._check(self.lib.ref_apb_forward(_ptr(w), w.shape[0], w.shape[1], alpha, delta, _ptr(o)))
        return o

    def decompose_apb(self, a, alpha, lane_bits=512):
        a = np.ascontiguousarray(a, np.float32)
        rows, cols = a.shape
        wpr = _i64(0)
        nnz = _i64(0)
        self._check(self.lib.ref_decompose_apb(_ptr(a), rows, cols, alpha, lane_bits, None,
                                               C.byref(wpr), None, None, None, C.byref(nnz)))
        bin_ = np.zeros((rows, wpr.value), np.uint64)
        rp = np.zeros(rows + 1, np.uint64)
        ci = np.zeros(max(nnz.value, 1), np.uint64)
        v = np.zeros(max(nnz.value, 1), np.float32)
        self._check(self.lib.ref_decompose_apb(_ptr(a), rows, cols, alpha, lane_bits, _ptr(bin_),
                                               C.byref(wpr), _ptr(rp), _ptr(ci), _ptr(v),
                                               C.byref(nnz)))
        return bin_, wpr.value, rp, ci[:nnz.value], v[:nnz.value]

    def pack_signs(self, a, lane_bits=512):
        a = np.ascontiguousarray(a, np.float32)
        wpr = _i64(0)
        self._check(self.lib.ref_pack_signs(_ptr(a), a.shape[0], a.shape[1], lane_bits, None,
                                            C.byref(wpr)))
        w = np.zeros((a.shape[0], wpr.value), np.uint64)
        self._check(self.lib.ref_pack_signs(_ptr(a), a.shape[0], a.shape[1], lane_bits, _ptr(w),
                                            C.byref(wpr)))
        return w, wpr.value

    def decompose_thm(self, levels, scale=1.0, lane_bits=512):
        levels = np.ascontiguousarray(levels, np.uint8)
        rows, cols = levels.shape
        wpr = _i64(0)
        self._check(self.lib.ref_decompose_thm(_ptr(levels), rows, cols, scale, lane_bits, None, None,
                                               None, C.byref(wpr)))
        t, h, m = (np.zeros((rows, wpr.value), np.uint64) for _ in range(3))
        self._check(self.lib.ref_decompose_thm(_ptr(levels), rows, cols, scale, lane_bits, _ptr(t),
                                               _ptr(h), _ptr(m), C.byref(wpr)))
        return t, h, m, wpr.value

    def quantize_2bit(self, a, s):
        a = np.ascontiguousarray(a, np.float32)
        out = np.empty(a.shape, np.uint8)
        self._check(self.lib.ref_quantize_2bit(_ptr(a), a.shape[0], a.shape[1], s, _ptr(out)))
        return out

    def dot_binary(self, u, v, n):
        out = _i64(0)
        self._check(self.lib.ref_dot_binary(_ptr(u), _ptr(v), u.size, n, C.byref(out)))
        return out.value

    def mbm(self, x, y, z):
        out = _i64(0)
        self._check(self.lib.ref_mbm(_ptr(x), _ptr(y), _ptr(z), x.size, C.byref(out)))
        return out.value

    # ---- BTSR containers through the reference writer / reader ----
    def store_dense(self, path, a):
        a = np.ascontiguousarray(a, np.float32)
        self._check(self.lib.ref_store_dense(path.encode(), _ptr(a), a.shape[0], a.shape[1]))

    def store_bit(self, path, words, rows, cols):
        w = np.ascontiguousarray(words, np.uint64)
        self._check(self.lib.ref_store_bit(path.encode(), _ptr(w), rows, cols, w.shape[1] if w.ndim == 2 else 0))

    def store_csr(self, path, rows, cols, row_ptr, col_idx, vals):
        rp = np.ascontiguousarray(row_ptr, np.uint64)
        ci = np.ascontiguousarray(col_idx, np.uint64)
        v = np.ascontiguousarray(vals, np.float32)
        self._check(self.lib.ref_store_csr(path.encode(), rows, cols, _ptr(rp), _ptr(ci), _ptr(v), ci.size))

    def pack_apb(self, w, prefix, alpha=None, delta=None):
        """The reference CLI's `pack --mode apb` (store_apb_layer files under `prefix`);
        returns the (alpha, delta) it used."""
        w = np.ascontiguousarray(w, np.float32)
        a, d = _f(0.0 if alpha is None else alpha), _f(0.0 if delta is None else delta)
        self._check(self.lib.ref_pack_apb(_ptr(w), w.shape[0], w.shape[1], int(alpha is not None),
                                          C.byref(a), C.byref(d), prefix.encode()))
        return a.value, d.value

    def store_thm_planes(self, prefix, t, h, m, cols, scale, gamma=None):
        t, h, m = (np.ascontiguousarray(x, np.uint64) for x in (t, h, m))
        self._check(self.lib.ref_store_thm_planes(prefix.encode(), _ptr(t), _ptr(h), _ptr(m), t.shape[0],
                                                  cols, t.shape[1], scale, int(gamma is not None),
                                                  0.0 if gamma is None else gamma))

    def load_check(self, path, kind=-1):
        """(error class, message) of the reference reader on `path`; (0, '') when it loads."""
        rc = self.lib.ref_load_check(path.encode(), kind)
        return rc, (self.lib.ref_last_error().decode() if rc else "")


def load_ref() -> Optional[Ref]:
    try:
        return Ref()
    except OSError:
        return None
