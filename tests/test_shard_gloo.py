"""CPU, world_size 2 (gloo): the N-sharded multi-GPU path's host logic — column ranges,
chunked compute + async gather, root re-layout, and the lossless 1/1 popcount wire —
with each rank's block computed by the oracle (on the GPU box the block comes from the
sm_100a kernels; bench.py --gpus N exercises that with NCCL)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2306_08960_b200 import data, shard


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        orc = oracle.Oracle()
        rng = np.random.default_rng(case["seed"])
        m, n, k = case["m"], case["n"], case["k"]
        a, wpr = data.random_words(rng, m, k)
        b, _ = data.random_words(rng, n, k)
        t, h, mm, _ = data.random_planes(rng, n, k)

        def compute_1x1(lo, hi, r0, r1, block):
            u, _ = orc.gemm_1x1(a[r0:r1], b[lo:hi], k, wpr)
            block.copy_(torch.from_numpy(u))

        def compute_1x2(lo, hi, r0, r1, block):
            _, o = orc.gemm_1x2(a[r0:r1], 1.0, t[lo:hi], h[lo:hi], mm[lo:hi], k, wpr, 0.5)
            block.copy_(torch.from_numpy(o))

        wire = shard.popcount_wire(k) if case["wire"] else None
        got11 = shard.run_sharded(m, n, torch.int32, compute_1x1, torch.device("cpu"),
                                  chunk_rows=case["chunk"], wire=wire)
        got12 = shard.run_sharded(m, n, torch.float32, compute_1x2, torch.device("cpu"),
                                  chunk_rows=case["chunk"])
        if rank == 0:
            want11 = orc.gemm_1x1(a, b, k, wpr)[0]
            want12 = orc.gemm_1x2(a, 1.0, t, h, mm, k, wpr, 0.5)[1]
            result_q.put((np.array_equal(got11.numpy(), want11),
                          np.array_equal(got12.numpy(), want12)))
        else:
            result_q.put(None if got11 is None and got12 is None else "non-root got data")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [
    dict(m=37, n=101, k=300, chunk=None, wire=False, seed=1),   # odd N: short last shard
    dict(m=64, n=96, k=1000, chunk=16, wire=True, seed=2),      # chunked, popcount wire
    dict(m=5, n=1, k=64, chunk=2, wire=True, seed=3),           # rank 1 owns no columns
])
def test_sharded_gather_world2(case):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    results = [q.get() for _ in range(world)]
    root = [r for r in results if isinstance(r, tuple)]
    assert root == [(True, True)], results
    assert [r for r in results if not isinstance(r, tuple)] == [None]


def test_column_ranges_cover_exactly():
    for n in (1, 7, 4096, 32768, 32769):
        for world in (1, 2, 3, 4, 8):
            spans = [shard.column_range(n, g, world) for g in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (l0, h0), (l1, h1) in zip(spans, spans[1:]):
                assert h0 == l1 and l0 <= h0
            assert max(h - l for l, h in spans) == shard.shard_width(n, world)


def test_popcount_wire_roundtrip():
    k = 32768
    x = torch.randint(0, k + 1, (1000,), dtype=torch.int32)
    u = k - 2 * x
    w = shard.popcount_wire(k)
    enc = w.encode(u)
    assert enc.dtype == torch.int16 and enc.element_size() == 2
    assert torch.equal(w.decode(enc), u)
    with pytest.raises(ValueError):
        shard.popcount_wire(1 << 16)
