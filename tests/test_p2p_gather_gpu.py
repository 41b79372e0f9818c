"""The gather fused into the GEMM epilogue (shard.PeerOutput), on one GPU.

Two processes (gloo for the handle exchange, both on cuda:0): rank 0 owns the M x N output,
rank 1 maps it through CUDA IPC (bitmm_ipc_get_handle / bitmm_ipc_open), and each rank's
1/1 GEMM writes its column block straight into that matrix at column offset lo with ldc = N.
Rank 0 compares the assembled matrix with the oracle. On an 8-GPU box the same calls write
across NVLink (the epilogue switches to st.global for another device's memory); here the
mapping, the offsets and the strided output are what is checked. The ranks' kernels do not
wait on each other.
"""
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, REPO)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from paper_2306_08960_b200 import _lib, data, shard
        m, n, k = 300, 1000, 1500
        rng = np.random.default_rng(9)
        a, wpr = data.random_words(rng, m, k)
        b, _ = data.random_words(rng, n, k)
        lo, hi = shard.column_range(n, rank, world)
        be = bench.GpuC5Backend(torch, torch.device("cuda", 0), _lib.load())
        da, db = be.upload(a), be.upload(b[lo:hi])
        po = shard.PeerOutput(m, n, torch.int32, torch.device("cuda", 0))
        if rank == 0:
            po.tensor.fill_(-7)
        dist.barrier()
        be.gemm_ptr(da, db, k, po.block_ptr(lo), n)
        be.status()
        torch.cuda.synchronize()
        dist.barrier()
        if rank == 0:
            import oracle
            want = oracle.Oracle().gemm_1x1(a, b, k, wpr)[0]
            q.put(bool(np.array_equal(po.tensor.cpu().numpy(), want)))
        dist.barrier()
        po.close()
    finally:
        dist.destroy_process_group()


def test_peer_output_gather_two_ranks():
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok
