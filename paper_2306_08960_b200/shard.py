"""Multi-GPU N-sharding of the bitwise GEMMs.

The output-column dimension N is split into contiguous ranges, one per rank: rank g
owns rows [lo_g, hi_g) of the packed b operand (row c of b_packed is output column c,
kernels.hpp:44-46), so no operand crosses ranks and there is no K reduction. The only
cross-GPU step is gathering the result blocks to the root — one collective
(torch.distributed gather; NCCL over NVLink on B200, gloo in the CPU tests).

Two ways to bring the blocks to the root:

* `PeerOutput` (GPUs in one box, the default): the root's M x N output is shared with every
  rank through CUDA IPC (bitmm_ipc_get_handle / bitmm_ipc_open) and each rank's GEMM writes its
  column block straight into it with ldc = N: the epilogue's stores cross NVLink tile by tile
  while the next tiles multiply, so the gather is fused into the GEMM and no collective runs
  after it. The root's matrix is complete after the ranks' kernels and one barrier.
* `run_sharded` (any backend, NCCL or gloo): computes the rank's block in row chunks and
  gathers each chunk asynchronously while the next chunk computes, then (on the root) re-lays
  the blocks out into the reference's row-major M x N matrix. For 1/1 the units K - 2x carry
  K's parity, so the popcount x = (K - units)/2 in [0, K] travels as uint16 when K < 2^16 —
  lossless, half the link bytes — and is expanded back on the root.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Optional

import torch
import torch.distributed as dist


def column_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous column block of `rank`: ceil-sized blocks, the last one possibly short."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid rank/world")
    per = (n + world - 1) // world
    lo = min(n, rank * per)
    return lo, min(n, lo + per)


def shard_width(n: int, world: int) -> int:
    return (n + world - 1) // world


@dataclass
class Wire:
    """How a block travels: `encode` maps the computed block to the transport tensor and
    `decode` maps it back on the root (both identity by default)."""

    dtype: torch.dtype
    encode: Callable[[torch.Tensor], torch.Tensor] = staticmethod(lambda t: t)
    decode: Callable[[torch.Tensor], torch.Tensor] = staticmethod(lambda t: t)


def popcount_wire(k: int) -> Wire:
    """1/1 int32 units u = K - 2x  <->  uint16 popcount x (exact for K < 65536)."""
    if not 0 < k < (1 << 16):
        raise ValueError("popcount wire needs 0 < K < 65536")
    return Wire(
        dtype=torch.int16,
        encode=lambda u: ((k - u) >> 1).to(torch.int16),
        decode=lambda x: k - 2 * (x.to(torch.int32) & 0xFFFF),
    )


def _bytes(t: torch.Tensor) -> torch.Tensor:
    return t.contiguous().view(torch.uint8)


def run_sharded(m: int, n: int, out_dtype: torch.dtype,
                compute: Callable[[int, int, int, int, torch.Tensor], None],
                device: torch.device, group=None, dst: int = 0,
                chunk_rows: Optional[int] = None, wire: Optional[Wire] = None,
                out: Optional[torch.Tensor] = None,
                comm_device: Optional[torch.device] = None) -> Optional[torch.Tensor]:
    """Compute this rank's column block of an M x N result and gather it to `dst`.

    compute(col_lo, col_hi, row_lo, row_hi, block) must fill `block`
    ([row_hi-row_lo, col_hi-col_lo], out_dtype, contiguous) with those output cells.
    Returns the assembled row-major M x N tensor on `dst`, None elsewhere. With a single
    rank it is just compute() into `out`. `comm_device`: where the gathered payloads live when
    the backend cannot move `device` tensors (gloo with CUDA compute); default `device`.
    """
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = column_range(n, rank, world)
    width = shard_width(n, world)
    chunk = chunk_rows or m
    if out is None and rank == dst:
        out = torch.empty((m, n), dtype=out_dtype, device=device)
    if world == 1:
        compute(0, n, 0, m, out)
        return out
    wire = wire or Wire(out_dtype)
    pending: List[tuple] = []

    def finish(item):
        work, r0, r1, parts = item
        work.wait()
        if rank == dst:
            for g, part in enumerate(parts):
                glo, ghi = column_range(n, g, world)
                if ghi > glo:
                    blk = part.view(wire.dtype).view(r1 - r0, width)[:, : ghi - glo].to(out.device)
                    out[r0:r1, glo:ghi].copy_(wire.decode(blk))

    for r0 in range(0, m, chunk):
        r1 = min(m, r0 + chunk)
        block = torch.empty((r1 - r0, width), dtype=out_dtype, device=device)
        if hi > lo:
            view = block[:, : hi - lo]
            if width == hi - lo:
                compute(lo, hi, r0, r1, view)
            else:  # short last shard: compute into a contiguous block, pad the rest
                tmp = torch.empty((r1 - r0, hi - lo), dtype=out_dtype, device=device)
                compute(lo, hi, r0, r1, tmp)
                view.copy_(tmp)
        if width > hi - lo:
            block[:, hi - lo:].zero_()
        payload = _bytes(wire.encode(block))
        if comm_device is not None:
            payload = payload.to(comm_device)
        parts = [torch.empty_like(payload) for _ in range(world)] if rank == dst else None
        work = dist.gather(payload, parts, dst=dst, group=group, async_op=True)
        pending.append((work, r0, r1, parts))
        # keep at most one gather in flight behind the compute of the next chunk
        while len(pending) > 1:
            finish(pending.pop(0))
    while pending:
        finish(pending.pop(0))
    return out if rank == dst else None


class PeerOutput:
    """The root rank's row-major M x N output, mapped into every rank of the group.

    The root allocates it; the others open its CUDA IPC handle. `block_ptr(col_lo)` is the
    device address of column col_lo in row 0 (leading dimension N), what a rank passes to a
    `bitmm_*_dev` call as its output so its column block lands in the root's matrix (SURVEY.md
    §8(e): no operand exchange, the output gathered over NVLink). Call `close()` on every rank
    when done; `tensor` is the matrix on the root, None elsewhere.
    """

    def __init__(self, m: int, n: int, dtype: torch.dtype, device: torch.device, group=None,
                 root: int = 0):
        import ctypes as C

        from . import _lib
        from .api import _raise
        lib = _lib.load()
        self._lib = lib
        self.rank = dist.get_rank(group)
        self.root = root
        self.n = n
        self.elem = torch.empty((), dtype=dtype).element_size()
        self.tensor = None
        self._opened = None
        payload = [None]
        if self.rank == root:
            self.tensor = torch.empty((m, n), dtype=dtype, device=device)
            handle = (C.c_uint8 * 64)()
            off = C.c_uint64(0)
            _raise(lib.bitmm_ipc_get_handle(C.c_void_p(self.tensor.data_ptr()), C.cast(handle, C.c_void_p),
                                            C.byref(off)))
            payload = [(bytes(handle), int(off.value))]
            self.ptr = self.tensor.data_ptr()
        dist.broadcast_object_list(payload, src=root, group=group)
        if self.rank != root:
            handle, off = payload[0]
            base = C.c_void_p()
            buf = (C.c_uint8 * 64).from_buffer_copy(handle)
            _raise(lib.bitmm_ipc_open(C.cast(buf, C.c_void_p), C.byref(base)))
            self._opened = base.value
            self.ptr = base.value + off

    def block_ptr(self, col_lo: int) -> int:
        return self.ptr + col_lo * self.elem

    def close(self) -> None:
        if self._opened is not None:
            from .api import _raise
            _raise(self._lib.bitmm_ipc_close(self._opened))
            self._opened = None
