"""Device-resident entry points: torch CUDA tensors in, results written in place.

Thin wrappers over the `*_dev` C ABI (include/bitmm_b200.h). PyTorch is plumbing here
(device memory, the current stream); all compute is the sm_100a library. Packed words
travel as int64 tensors (a bit-identical view of the reference's uint64 words).
Encoding errors detected on the device are latched; `status()` synchronises the
stream and raises them (InvalidEncoding / ValueError) like the host flavour does.
"""
from __future__ import annotations

from typing import Optional

import torch

from . import _lib
from .api import _raise


def _stream(stream: Optional[torch.cuda.Stream]):
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError("device entry points need contiguous CUDA tensors")
    return t.data_ptr()


def status(stream: Optional[torch.cuda.Stream] = None) -> None:
    _raise(_lib.load().bitmm_device_status(_stream(stream)))


def launch_count() -> int:
    """Kernels launched by the most recent compute call on this thread."""
    return _lib.load().bitmm_last_launch_count()


def reserve_workspace(routine: int, m: int, n: int, k: int) -> None:
    lib = _lib.load()
    _raise(lib.bitmm_reserve_workspace(lib.bitmm_workspace_bytes(routine, m, n, k)))


def gemm_1x1(a: torch.Tensor, b_packed: torch.Tensor, k: int, gamma_a: float = 1.0,
             gamma_b: float = 1.0, units: Optional[torch.Tensor] = None,
             out: Optional[torch.Tensor] = None, stream=None, popc: bool = False) -> None:
    m, wpr = a.shape
    n = b_packed.shape[0]
    ldc = (units if units is not None else out).shape[1]
    fn = _lib.load().bitmm_gemm_1x1_popc_dev if popc else _lib.load().bitmm_gemm_1x1_dev
    _raise(fn(_ptr(a), m, _ptr(b_packed), n, k, wpr, gamma_a, gamma_b, _ptr(units), _ptr(out),
              ldc, _stream(stream)))


def gemm_1x2(w: torch.Tensor, gamma: float, t: torch.Tensor, h: torch.Tensor, mm: torch.Tensor,
             k: int, a_scale: float = 1.0, a_gamma: Optional[float] = None,
             row_scale: Optional[torch.Tensor] = None, col_scale: Optional[torch.Tensor] = None,
             units: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
             stream=None) -> None:
    m, wpr = w.shape
    n = t.shape[0]
    ldc = (units if units is not None else out).shape[1]
    _raise(_lib.load().bitmm_gemm_1x2_dev(
        _ptr(w), m, gamma, _ptr(t), _ptr(h), _ptr(mm), n, k, wpr, a_scale,
        int(a_gamma is not None), 1.0 if a_gamma is None else a_gamma, _ptr(row_scale),
        _ptr(col_scale), _ptr(units), _ptr(out), ldc, _stream(stream)))


def gemm_2x2(wt, wh, wm, at, ah, am, k: int, w_scale: float = 1.0, a_scale: float = 1.0,
             w_gamma: Optional[float] = None, a_gamma: Optional[float] = None,
             row_scale=None, col_scale=None, units=None, out=None, stream=None) -> None:
    m, wpr = wt.shape
    n = at.shape[0]
    ldc = (units if units is not None else out).shape[1]
    _raise(_lib.load().bitmm_gemm_2x2_dev(
        _ptr(wt), _ptr(wh), _ptr(wm), m, w_scale, int(w_gamma is not None),
        1.0 if w_gamma is None else w_gamma, _ptr(at), _ptr(ah), _ptr(am), n, k, wpr, a_scale,
        int(a_gamma is not None), 1.0 if a_gamma is None else a_gamma, _ptr(row_scale),
        _ptr(col_scale), _ptr(units), _ptr(out), ldc, _stream(stream)))


def gemm_1x32(w: torch.Tensor, k: int, gamma: float, b: torch.Tensor, out: torch.Tensor,
              row_gamma: Optional[torch.Tensor] = None, stream=None) -> None:
    m, wpr = w.shape
    n = b.shape[1]
    _raise(_lib.load().bitmm_gemm_1x32_dev(_ptr(w), m, k, wpr, gamma, _ptr(row_gamma), _ptr(b), n,
                                           b.shape[1], _ptr(out), out.shape[1], _stream(stream)))


def spmm_csr(rows: int, cols: int, row_ptr, col_idx, vals, b: torch.Tensor, out: torch.Tensor,
             stream=None) -> None:
    n = b.shape[1]
    _raise(_lib.load().bitmm_spmm_csr_dev(rows, cols, _ptr(row_ptr), _ptr(col_idx), _ptr(vals),
                                          _ptr(b), n, b.shape[1], _ptr(out), out.shape[1],
                                          _stream(stream)))


def layer_forward(bin_words: torch.Tensor, cols: int, alpha, row_ptr, col_idx, vals,
                  b: torch.Tensor, out: torch.Tensor, stream=None) -> None:
    """alpha: python float (reference scalar) or a CUDA float32 tensor [rows]."""
    rows, wpr = bin_words.shape
    n = b.shape[1]
    if isinstance(alpha, torch.Tensor):
        a_scalar, a_vec = 1.0, alpha
    else:
        a_scalar, a_vec = float(alpha), None
    _raise(_lib.load().bitmm_layer_forward_dev(
        rows, cols, a_scalar, _ptr(a_vec), _ptr(bin_words), wpr, _ptr(row_ptr), _ptr(col_idx),
        _ptr(vals), _ptr(b), n, b.shape[1], _ptr(out), out.shape[1], _stream(stream)))


def gemm_batch(items, stream=None) -> None:
    """One grouped launch for several GEMMs (bitmm_gemm_batch_dev). `items`: dicts with
    routine ('1x1' | '1x2' | '2x2'), the operand tensors (a / w / wt,wh,wm and b / t,h,m),
    k, optional scales (gamma_a, gamma_b, gamma, a_scale, w_scale, a_gamma, w_gamma,
    row_scale, col_scale) and outputs (units, out) — the keywords of gemm_1x1/1x2/2x2."""
    arr = (_lib.GemmItem * len(items))()
    for it, d in zip(arr, items):
        r = d["routine"]
        if r == "1x1":
            it.routine, a, b = _lib.ROUTINE_1X1, [d["a"]], [d["b"]]
            it.a_scale, it.b_scale = d.get("gamma_a", 1.0), d.get("gamma_b", 1.0)
        elif r == "1x2":
            it.routine, a, b = _lib.ROUTINE_1X2, [d["w"]], [d["t"], d["h"], d["m"]]
            it.a_scale, it.b_scale = d.get("gamma", 1.0), d.get("a_scale", 1.0)
        else:
            it.routine, a, b = _lib.ROUTINE_2X2, [d["wt"], d["wh"], d["wm"]], [d["t"], d["h"], d["m"]]
            it.a_scale, it.b_scale = d.get("w_scale", 1.0), d.get("a_scale", 1.0)
            if d.get("w_gamma") is not None:
                it.has_a_gamma, it.a_gamma = 1, d["w_gamma"]
        if r != "1x1" and d.get("a_gamma") is not None:
            it.has_b_gamma, it.b_gamma = 1, d["a_gamma"]
        it.a0, it.a1, it.a2 = (_ptr(a[i]) if i < len(a) else None for i in range(3))
        it.b0, it.b1, it.b2 = (_ptr(b[i]) if i < len(b) else None for i in range(3))
        it.m, it.wpr = a[0].shape
        it.n = b[0].shape[0]
        it.k = d["k"]
        it.row_scale, it.col_scale = _ptr(d.get("row_scale")), _ptr(d.get("col_scale"))
        u, o = d.get("units"), d.get("out")
        it.c_units, it.c = _ptr(u), _ptr(o)
        it.ldc = (u if u is not None else o).shape[1]
    _raise(_lib.load().bitmm_gemm_batch_dev(arr, len(items), _stream(stream)))


def layer_forward_2bit(bin_words: torch.Tensor, cols: int, alpha, row_ptr, col_idx, vals,
                       t: torch.Tensor, h: torch.Tensor, m: torch.Tensor, out: torch.Tensor,
                       a_scale: float = 1.0, a_gamma: Optional[float] = None, stream=None) -> None:
    """APB with 2-bit activations: out[rows][tokens] = gemm_1x2(bin, alpha, planes) +
    spmm_csr(residual, dequant(planes)); planes are tokens x wpr."""
    rows, wpr = bin_words.shape
    if isinstance(alpha, torch.Tensor):
        a_scalar, a_vec = 1.0, alpha
    else:
        a_scalar, a_vec = float(alpha), None
    _raise(_lib.load().bitmm_layer_forward_2bit_dev(
        rows, cols, a_scalar, _ptr(a_vec), _ptr(bin_words), wpr, _ptr(row_ptr), _ptr(col_idx),
        _ptr(vals), _ptr(t), _ptr(h), _ptr(m), t.shape[0], a_scale, int(a_gamma is not None),
        1.0 if a_gamma is None else a_gamma, _ptr(out), out.shape[1], _stream(stream)))


def pack_signs(a: torch.Tensor, lane_bits: int = 512, out: Optional[torch.Tensor] = None,
               stream=None) -> torch.Tensor:
    """GPU pack_signs (tensor.cpp:155-164): fp32 [rows, cols] -> int64 view of the BitMatrix
    words [rows, wpr], wpr = ceil(cols / lane_bits) * lane_bits / 64, zero padding."""
    from .data import padded_words
    rows, cols = a.shape
    wpr = padded_words(cols, lane_bits)
    if out is None:
        out = torch.empty((rows, wpr), dtype=torch.int64, device=a.device)
    _raise(_lib.load().bitmm_pack_signs_dev(_ptr(a), rows, cols, a.stride(0), _ptr(out), wpr,
                                            _stream(stream)))
    return out


def quantize_thm(a: torch.Tensor, s: float, lane_bits: int = 512, stream=None):
    """GPU quantize_uniform_2bit + decompose_thm (transform.cpp:21-36, 47-75): fp32 ->
    (t, h, m) int64 views of the plane words [rows, wpr]."""
    from .data import padded_words
    rows, cols = a.shape
    wpr = padded_words(cols, lane_bits)
    t, h, m = (torch.empty((rows, wpr), dtype=torch.int64, device=a.device) for _ in range(3))
    _raise(_lib.load().bitmm_quantize_thm_dev(_ptr(a), rows, cols, a.stride(0), s, _ptr(t), _ptr(h),
                                              _ptr(m), wpr, _stream(stream)))
    return t, h, m


def decompose_thm(levels: torch.Tensor, lane_bits: int = 512, stream=None):
    """GPU decompose_thm (transform.cpp:47-75): uint8 levels [rows, cols] (TwoBitMatrix) ->
    (t, h, m) int64 views of the plane words [rows, wpr]. A level above 3 is reported by
    status() as ValueError ("2-bit level out of range")."""
    from .data import padded_words
    rows, cols = levels.shape
    levels = levels.contiguous()
    wpr = padded_words(cols, lane_bits)
    t, h, m = (torch.empty((rows, wpr), dtype=torch.int64, device=levels.device) for _ in range(3))
    _raise(_lib.load().bitmm_decompose_thm_dev(_ptr(levels), rows, cols, _ptr(t), _ptr(h), _ptr(m),
                                               wpr, _stream(stream)))
    return t, h, m


def decompose_apb(a: torch.Tensor, alpha, lane_bits: int = 512, stream=None):
    """GPU decompose_apb (apb.cpp:119-142): fp32 [rows, cols] and a positive alpha (a float,
    or a per-row fp32 tensor) -> (bin words [rows, wpr] int64, row_ptr [rows+1], col_idx [nnz]
    as int64 views of the u64 arrays, vals [nnz] fp32). Bit-identical to the reference."""
    import ctypes as C
    from .data import padded_words
    rows, cols = a.shape
    wpr = padded_words(cols, lane_bits)
    dev = a.device
    row_alpha = alpha if isinstance(alpha, torch.Tensor) else None
    scalar = 1.0 if row_alpha is not None else float(alpha)
    bin_ = torch.empty((rows, wpr), dtype=torch.int64, device=dev)
    row_ptr = torch.empty(rows + 1, dtype=torch.int64, device=dev)
    nnz = C.c_int64(0)
    lib = _lib.load()
    args = (_ptr(a), rows, cols, a.stride(0), scalar, _ptr(row_alpha), _ptr(bin_), wpr, _ptr(row_ptr))
    _raise(lib.bitmm_decompose_apb_dev(*args, None, None, 0, C.byref(nnz), _stream(stream)))
    col_idx = torch.empty(nnz.value, dtype=torch.int64, device=dev)
    vals = torch.empty(nnz.value, dtype=torch.float32, device=dev)
    if nnz.value:
        _raise(lib.bitmm_decompose_apb_dev(*args, _ptr(col_idx), _ptr(vals), nnz.value, C.byref(nnz),
                                           _stream(stream)))
    return bin_, row_ptr, col_idx, vals


def dot_binary_rows(u: torch.Tensor, v: torch.Tensor, n: int, stream=None) -> torch.Tensor:
    """dot_binary (kernels.cpp:120-129) for every row pair of u, v [count, words] (int64 views
    of the packed words): n - 2*popc(u ^ v)."""
    count, words = u.shape
    out = torch.empty(count, dtype=torch.int64, device=u.device)
    _raise(_lib.load().bitmm_dot_binary_dev(_ptr(u), _ptr(v), count, words, n, _ptr(out), _stream(stream)))
    return out


def mbm_rows(x: torch.Tensor, y: torch.Tensor, z: torch.Tensor, stream=None) -> torch.Tensor:
    """mbm (kernels.cpp:131-140) for every row triple: popc(z) - 2*popc((x ^ y) & z)."""
    count, words = x.shape
    out = torch.empty(count, dtype=torch.int64, device=x.device)
    _raise(_lib.load().bitmm_mbm_dev(_ptr(x), _ptr(y), _ptr(z), count, words, _ptr(out), _stream(stream)))
    return out
