"""Python mirror of the reference's kernel-layer interface (namespace bitmm).

Same names, argument meaning and error behaviour as
/root/reference/proj/include/bitmm/{tensor,kernels,apb}.hpp, backed by the sm_100a
library through the C ABI (include/bitmm_b200.h, `*_host` flavour: host arrays in,
host float32 DenseMatrix out). Exception mapping:
    std::invalid_argument  -> ValueError
    bitmm::InvalidEncoding -> InvalidEncoding (a RuntimeError, like the reference's)
There is no CPU fallback: without the CUDA library or a device every GEMM raises.

DenseMatrix is a C-contiguous float32 numpy array [rows, cols].
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .data import LANE_BITS, padded_words, tail_mask_words

MAX_SHARED_DIM = 1 << 20  # kMaxSharedDim, tensor.hpp:21


class IoError(RuntimeError):
    """errors.hpp:14 — container format / file errors (BITMM_ERR_IO)."""


class InvalidEncoding(RuntimeError):
    """bitmm::InvalidEncoding (errors.hpp:20-23)."""


def _raise(rc: int) -> None:
    if rc == _lib.OK:
        return
    msg = _lib.last_error()
    if rc == _lib.ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == _lib.ERR_INVALID_ENCODING:
        raise InvalidEncoding(msg)
    if rc == _lib.ERR_IO:
        raise IoError(msg)
    raise _lib.BitmmError(f"bitmm_b200 error {rc}: {msg}")


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# --------------------------------------------------------------------------- types
class BitMatrix:
    """tensor.hpp:59-112 — row-major packed bits, bit 1 <-> +1, zero padding."""

    def __init__(self, rows: int, cols: int, lane_bits: int = LANE_BITS):
        if rows < 0 or cols < 0:
            raise ValueError("matrix dimensions must be non-negative")
        self._rows, self._cols = rows, cols
        self._wpr = padded_words(cols, lane_bits)
        self.words = np.zeros((rows, self._wpr), dtype=np.uint64)

    @staticmethod
    def from_words(rows: int, cols: int, words_per_row: int, words) -> "BitMatrix":
        """tensor.cpp:62-76."""
        if rows < 0 or cols < 0:
            raise ValueError("matrix dimensions must be non-negative")
        if words_per_row * 64 < cols:
            raise ValueError("words_per_row too small for the column count")
        w = np.ascontiguousarray(np.asarray(words, dtype=np.uint64))
        if w.size != rows * words_per_row:
            raise ValueError("bit payload size does not match rows*words_per_row")
        b = BitMatrix.__new__(BitMatrix)
        b._rows, b._cols, b._wpr = rows, cols, words_per_row
        b.words = w.reshape(rows, words_per_row)
        if not b.padding_is_zero():
            raise ValueError("bit matrix padding must be zero")
        return b

    def rows(self) -> int:
        return self._rows

    def cols(self) -> int:
        return self._cols

    def words_per_row(self) -> int:
        return self._wpr

    def bit(self, r: int, i: int) -> bool:
        return bool((int(self.words[r, i >> 6]) >> (i & 63)) & 1)

    def set_bit(self, r: int, i: int, value: bool) -> None:
        m = np.uint64(1 << (i & 63))
        if value:
            self.words[r, i >> 6] |= m
        else:
            self.words[r, i >> 6] &= ~m

    def padding_is_zero(self) -> bool:
        if self._rows == 0 or self._wpr == 0:
            return True
        keep = tail_mask_words(self._cols, self._wpr)
        return not np.any(self.words & ~keep[None, :])

    def __eq__(self, other) -> bool:
        return (isinstance(other, BitMatrix) and self._rows == other._rows
                and self._cols == other._cols and self._wpr == other._wpr
                and np.array_equal(self.words, other.words))


@dataclass
class ThmPlanes:
    """tensor.hpp:134-145 — ternary planes of a 2-bit operand."""

    t: BitMatrix
    h: BitMatrix
    m: BitMatrix
    scale: float = 1.0
    gamma: Optional[float] = None

    def rows(self) -> int:
        return self.t.rows()

    def cols(self) -> int:
        return self.t.cols()

    def _same_shapes(self) -> bool:
        def same(a, b):
            return (a.rows() == b.rows() and a.cols() == b.cols()
                    and a.words_per_row() == b.words_per_row())
        return same(self.t, self.h) and same(self.t, self.m)

    def validate(self) -> None:
        """tensor.cpp:133-153 (host-side; the GEMMs re-check legality on the device)."""
        if not self._same_shapes():
            raise InvalidEncoding("plane shapes differ")
        if not self.scale > 0.0:
            raise InvalidEncoding("plane scale must be positive")
        if not (self.t.padding_is_zero() and self.h.padding_is_zero() and self.m.padding_is_zero()):
            raise InvalidEncoding("plane padding must be zero")
        t, h, m = self.t.words, self.h.words, self.m.words
        if np.any(t & h):
            raise InvalidEncoding("t and h set on the same element")
        if np.any(t & ~m):
            raise InvalidEncoding("t requires m")
        if np.any(h & m):
            raise InvalidEncoding("h requires m clear")


@dataclass
class TwoBitMatrix:
    """transform.hpp:16-27 — unsigned levels p in {0..3}, value p*scale."""

    rows: int
    cols: int
    levels: np.ndarray
    scale: float = 1.0

    def level(self, r: int, c: int) -> int:
        return int(self.levels.reshape(self.rows, self.cols)[r, c])


@dataclass
class CsrMatrix:
    """tensor.hpp:115-128."""

    rows: int = 0
    cols: int = 0
    row_ptr: np.ndarray = field(default_factory=lambda: np.zeros(1, np.uint64))
    col_idx: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    vals: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))

    @staticmethod
    def create(rows, cols, row_ptr, col_idx, vals) -> "CsrMatrix":
        m = CsrMatrix(rows, cols, np.ascontiguousarray(row_ptr, dtype=np.uint64),
                      np.ascontiguousarray(col_idx, dtype=np.uint64),
                      np.ascontiguousarray(vals, dtype=np.float32))
        m.validate()
        return m

    def nnz(self) -> int:
        return 0 if self.row_ptr.size == 0 else int(self.row_ptr[-1])

    def validate(self) -> None:
        """tensor.cpp:104-123."""
        if self.rows < 0 or self.cols < 0:
            raise ValueError("matrix dimensions must be non-negative")
        rp = self.row_ptr
        if rp.size != self.rows + 1:
            raise ValueError("csr row_ptr must have rows+1 entries")
        if rp[0] != 0:
            raise ValueError("csr row_ptr must start at 0")
        if np.any(rp[1:] < rp[:-1]):
            raise ValueError("csr row_ptr must be monotone")
        if self.col_idx.size != rp[-1] or self.vals.size != rp[-1]:
            raise ValueError("csr payload sizes must match nnz")
        if self.col_idx.size and np.any(self.col_idx >= np.uint64(self.cols)):
            raise ValueError("csr column index out of range")
        if self.col_idx.size > 1:
            inc = self.col_idx[1:].astype(np.int64) - self.col_idx[:-1].astype(np.int64)
            starts = np.zeros(self.col_idx.size, bool)
            starts[rp[:-1][rp[:-1] < rp[1:]].astype(np.int64)] = True
            if np.any((inc <= 0) & ~starts[1:]):
                raise ValueError("csr column indices must be strictly increasing per row")
        if not np.all(np.isfinite(self.vals)):
            raise ValueError("csr values must be finite")

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.rows, self.cols), np.float32)
        for r in range(self.rows):
            s, e = int(self.row_ptr[r]), int(self.row_ptr[r + 1])
            d[r, self.col_idx[s:e].astype(np.int64)] = self.vals[s:e]
        return d


@dataclass
class ApbLayer:
    """apb.hpp:45-54. `alpha` may be a scalar (reference) or a per-row vector (BASELINE
    config 4's alpha per output column of the weight)."""

    rows: int
    cols: int
    alpha: object
    bin: BitMatrix
    residual: CsrMatrix


# --------------------------------------------------------------------------- packing
# The packers run on the GPU through the host ABI (bitmm_pack_signs_host, ...); there is no
# host implementation of them here.
def pack_signs(m: np.ndarray, lane_bits: int = LANE_BITS) -> BitMatrix:
    """tensor.cpp:155-164 — sign(0) counts as +1 (GPU packer, bitmm_pack_signs_host)."""
    m = np.ascontiguousarray(m, dtype=np.float32)
    rows, cols = m.shape
    b = BitMatrix(rows, cols, lane_bits)  # the reference's dimension checks
    if rows == 0 or b.words_per_row() == 0:
        return b
    _raise(_lib.load().bitmm_pack_signs_host(_ptr(m), rows, cols, cols, _ptr(b.words), b.words_per_row()))
    return b


def decompose_thm(q: TwoBitMatrix, gamma: Optional[float] = None,
                  lane_bits: int = LANE_BITS) -> ThmPlanes:
    """transform.cpp:47-75 (GPU packer, bitmm_decompose_thm_host): a level above 3 raises
    ValueError ("2-bit level out of range")."""
    lv = np.ascontiguousarray(np.asarray(q.levels, dtype=np.uint8).reshape(q.rows, q.cols))
    t, h, m = (BitMatrix(q.rows, q.cols, lane_bits) for _ in range(3))
    if q.rows > 0 and t.words_per_row() > 0:
        _raise(_lib.load().bitmm_decompose_thm_host(_ptr(lv), q.rows, q.cols, _ptr(t.words), _ptr(h.words),
                                                    _ptr(m.words), t.words_per_row()))
    return ThmPlanes(t, h, m, q.scale, gamma)


def quantize_uniform_2bit(m: np.ndarray, s: float) -> TwoBitMatrix:
    """transform.cpp:21-36 — lround (halves away from zero), clamp to [0,3]. The levels view a
    TwoBitMatrix carries; device pipelines quantize and decompose in one GPU pass
    (bitmm_quantize_thm_*)."""
    if not s > 0.0:
        raise ValueError("quantization step must be positive")
    m = np.asarray(m, dtype=np.float32)
    x = (m / np.float32(s)).astype(np.float32)
    p = np.sign(x) * np.floor(np.abs(x).astype(np.float64) + 0.5)
    p = np.clip(p, 0, 3).astype(np.uint8)
    return TwoBitMatrix(m.shape[0], m.shape[1], p.reshape(-1), float(s))


def decompose_apb(a: np.ndarray, alpha, lane_bits: int = LANE_BITS) -> ApbLayer:
    """apb.cpp:119-142 (GPU packer, bitmm_decompose_apb_host). bin = pack_signs(a) at every
    position; residual = a - alpha*sign(a) wherever |a| != alpha (membership by exact value),
    computed in double and rounded with ties away from zero. `alpha` may also be a per-row
    vector (each row split with its own alpha)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    rows, cols = a.shape
    per_row = np.ndim(alpha) != 0
    al = np.ascontiguousarray(np.asarray(alpha, np.float32).reshape(-1)) if per_row else None
    a_scalar = 1.0 if per_row else float(alpha)
    if (per_row and not np.all(al > 0.0)) or (not per_row and not a_scalar > 0.0):
        raise ValueError("alpha must be positive")
    bin_ = BitMatrix(rows, cols, lane_bits)
    row_ptr = np.zeros(rows + 1, np.uint64)
    nnz = C.c_int64(0)
    lib = _lib.load()
    wpr = bin_.words_per_row()
    _raise(lib.bitmm_decompose_apb_host(_ptr(a), rows, cols, cols, a_scalar, _ptr(al), _ptr(bin_.words), wpr,
                                        _ptr(row_ptr), None, None, 0, C.byref(nnz)))
    col_idx = np.zeros(max(nnz.value, 1), np.uint64)
    vals = np.zeros(max(nnz.value, 1), np.float32)
    if nnz.value > 0:
        _raise(lib.bitmm_decompose_apb_host(_ptr(a), rows, cols, cols, a_scalar, _ptr(al), _ptr(bin_.words),
                                            wpr, _ptr(row_ptr), _ptr(col_idx), _ptr(vals), nnz.value,
                                            C.byref(nnz)))
    res = CsrMatrix.create(rows, cols, row_ptr, col_idx[:nnz.value], vals[:nnz.value])
    return ApbLayer(rows, cols, alpha if not per_row else np.asarray(alpha, np.float32), bin_, res)


# --------------------------------------------------------------------------- GEMMs
def _check_threads(threads: int) -> None:
    if threads < 1:
        raise ValueError("thread count must be at least 1")


def _planes_args(p: ThmPlanes):
    return (p.t.words, p.h.words, p.m.words)


def gemm_1x1(a: BitMatrix, b_packed: BitMatrix, gamma_a: float = 1.0, gamma_b: float = 1.0,
             threads: int = 1) -> np.ndarray:
    """kernels.hpp:47-48 / kernels.cpp:163-183."""
    if a.cols() != b_packed.cols() or a.words_per_row() != b_packed.words_per_row():
        raise ValueError("gemm dimension mismatch (packed rows must share K and padding)")
    _check_gemm(a.rows(), a.cols(), b_packed.rows())
    _check_threads(threads)
    m, n = a.rows(), b_packed.rows()
    out = np.empty((m, n), np.float32)
    _raise(_lib.load().bitmm_gemm_1x1_host(_ptr(a.words), m, _ptr(b_packed.words), n, a.cols(),
                                           a.words_per_row(), gamma_a, gamma_b, None, _ptr(out), n))
    return out


def _check_gemm(m: int, k: int, n: int) -> None:
    """GemmProblem::validate (kernels.cpp:115-118)."""
    if m <= 0 or k <= 0 or n <= 0:
        raise ValueError("gemm dimensions must be positive")
    if k > MAX_SHARED_DIM:
        raise ValueError("shared dimension exceeds the 2^20 accumulator bound")


def gemm_1x2(w: BitMatrix, gamma: float, a_packed: ThmPlanes, threads: int = 1,
             row_scale: Optional[np.ndarray] = None,
             col_scale: Optional[np.ndarray] = None) -> np.ndarray:
    """kernels.hpp:55 / kernels.cpp:185-221. Plane legality is checked on the device and
    still takes precedence over shape errors, as a_packed.validate() does in the reference."""
    if not a_packed._same_shapes():
        raise InvalidEncoding("plane shapes differ")
    m, n = w.rows(), a_packed.rows()
    if w.cols() != a_packed.cols() or w.words_per_row() != a_packed.t.words_per_row():
        # shape error; surface plane errors first like the reference
        a_packed.validate()
        raise ValueError("gemm dimension mismatch (packed rows must share K and padding)")
    _check_threads_after = threads
    out = np.empty((max(m, 0), max(n, 0)), np.float32)
    t, h, mm = _planes_args(a_packed)
    rs = None if row_scale is None else np.ascontiguousarray(row_scale, np.float32)
    cs = None if col_scale is None else np.ascontiguousarray(col_scale, np.float32)
    _raise(_lib.load().bitmm_gemm_1x2_host(
        _ptr(w.words), m, gamma, _ptr(t), _ptr(h), _ptr(mm), n, w.cols(), w.words_per_row(),
        a_packed.scale, int(a_packed.gamma is not None),
        1.0 if a_packed.gamma is None else a_packed.gamma, _ptr(rs), _ptr(cs), None, _ptr(out),
        max(n, 1)))
    _check_threads(_check_threads_after)
    return out


def gemm_2x2(w: ThmPlanes, a_packed: ThmPlanes, threads: int = 1,
             row_scale: Optional[np.ndarray] = None,
             col_scale: Optional[np.ndarray] = None) -> np.ndarray:
    """kernels.hpp:62 / kernels.cpp:223-275."""
    if not w._same_shapes() or not a_packed._same_shapes():
        raise InvalidEncoding("plane shapes differ")
    m, n = w.rows(), a_packed.rows()
    if w.cols() != a_packed.cols() or w.t.words_per_row() != a_packed.t.words_per_row():
        w.validate()
        a_packed.validate()
        raise ValueError("gemm dimension mismatch (packed rows must share K and padding)")
    out = np.empty((max(m, 0), max(n, 0)), np.float32)
    rs = None if row_scale is None else np.ascontiguousarray(row_scale, np.float32)
    cs = None if col_scale is None else np.ascontiguousarray(col_scale, np.float32)
    wt, wh, wm = _planes_args(w)
    at, ah, am = _planes_args(a_packed)
    _raise(_lib.load().bitmm_gemm_2x2_host(
        _ptr(wt), _ptr(wh), _ptr(wm), m, w.scale, int(w.gamma is not None),
        1.0 if w.gamma is None else w.gamma, _ptr(at), _ptr(ah), _ptr(am), n, w.cols(),
        w.t.words_per_row(), a_packed.scale, int(a_packed.gamma is not None),
        1.0 if a_packed.gamma is None else a_packed.gamma, _ptr(rs), _ptr(cs), None, _ptr(out),
        max(n, 1)))
    _check_threads(threads)
    return out


def gemm_1x32_ref(w: BitMatrix, gamma, b: np.ndarray, threads: int = 1) -> np.ndarray:
    """kernels.hpp:73 / kernels.cpp:300-332. `gamma` may be a per-row vector."""
    b = np.ascontiguousarray(b, dtype=np.float32)
    if w.cols() != b.shape[0]:
        raise ValueError("gemm dimension mismatch")
    _check_gemm(w.rows(), w.cols(), b.shape[1])
    _check_threads(threads)
    m, n = w.rows(), b.shape[1]
    g_vec = None if np.ndim(gamma) == 0 else np.ascontiguousarray(gamma, np.float32)
    out = np.empty((m, n), np.float32)
    _raise(_lib.load().bitmm_gemm_1x32_host(
        _ptr(w.words), m, w.cols(), w.words_per_row(), float(gamma) if g_vec is None else 1.0,
        _ptr(g_vec), _ptr(b), n, n, _ptr(out), n))
    return out


def spmm_csr(a: CsrMatrix, b: np.ndarray, threads: int = 1) -> np.ndarray:
    """kernels.hpp:76 / kernels.cpp:334-352."""
    b = np.ascontiguousarray(b, dtype=np.float32)
    if a.cols != b.shape[0]:
        raise ValueError("gemm dimension mismatch")
    if a.rows <= 0 or b.shape[1] <= 0 or a.cols <= 0:
        raise ValueError("gemm dimensions must be positive")
    if a.cols > MAX_SHARED_DIM:
        raise ValueError("shared dimension exceeds the 2^20 accumulator bound")
    _check_threads(threads)
    n = b.shape[1]
    out = np.empty((a.rows, n), np.float32)
    _raise(_lib.load().bitmm_spmm_csr_host(a.rows, a.cols, _ptr(a.row_ptr), _ptr(a.col_idx),
                                           _ptr(a.vals), a.nnz(), _ptr(b), n, n, _ptr(out), n))
    return out


def layer_forward(l: ApbLayer, b: np.ndarray, threads: int = 1) -> np.ndarray:
    """apb.hpp:65 / apb.cpp:158-164: alpha*sign(bin).b + residual.b, one fused GPU pass."""
    b = np.ascontiguousarray(b, dtype=np.float32)
    if l.bin.cols() != b.shape[0] or l.residual.cols != b.shape[0]:
        raise ValueError("gemm dimension mismatch")
    _check_gemm(l.bin.rows(), l.bin.cols(), b.shape[1])
    _check_threads(threads)
    m, n = l.rows, b.shape[1]
    a_vec = None if np.ndim(l.alpha) == 0 else np.ascontiguousarray(l.alpha, np.float32)
    out = np.empty((m, n), np.float32)
    r = l.residual
    _raise(_lib.load().bitmm_layer_forward_host(
        m, l.cols, float(l.alpha) if a_vec is None else 1.0, _ptr(a_vec), _ptr(l.bin.words),
        l.bin.words_per_row(), _ptr(r.row_ptr), _ptr(r.col_idx), _ptr(r.vals), r.nnz(), _ptr(b),
        n, n, _ptr(out), n))
    return out


def layer_forward_2bit(l: ApbLayer, a_packed: ThmPlanes, threads: int = 1) -> np.ndarray:
    """APB inference with 2-bit activations: the composition
    gemm_1x2(bin, alpha, a_packed) + spmm_csr(residual, dequant(a_packed)) of reference calls
    (kernels.cpp:185-221, 334-352; added as in apb.cpp:161-162). a_packed holds one row per
    token, K-packed; the result is rows x tokens, bit-identical to that composition."""
    a_packed.validate()
    if l.bin.cols() != a_packed.cols() or l.bin.words_per_row() != a_packed.t.words_per_row():
        raise ValueError("gemm dimension mismatch (packed rows must share K and padding)")
    _check_gemm(l.bin.rows(), l.bin.cols(), a_packed.rows())
    _check_threads(threads)
    m, n = l.rows, a_packed.rows()
    a_vec = None if np.ndim(l.alpha) == 0 else np.ascontiguousarray(l.alpha, np.float32)
    out = np.empty((m, n), np.float32)
    r = l.residual
    _raise(_lib.load().bitmm_layer_forward_2bit_host(
        m, l.cols, float(l.alpha) if a_vec is None else 1.0, _ptr(a_vec), _ptr(l.bin.words),
        l.bin.words_per_row(), _ptr(r.row_ptr), _ptr(r.col_idx), _ptr(r.vals), r.nnz(),
        _ptr(a_packed.t.words), _ptr(a_packed.h.words), _ptr(a_packed.m.words), n,
        float(a_packed.scale), int(a_packed.gamma is not None),
        1.0 if a_packed.gamma is None else float(a_packed.gamma), _ptr(out), n))
    return out
