"""bench.py's multi-rank orchestration on CPU (gloo, world size 2) with a CPU stub for the GEMM.

The config-5 sweep (bench.c5_sweep) shards N across the ranks, times the per-rank GEMM, runs
the NCCL-path gather (shard.run_sharded with the uint16 popcount wire; gloo here) and checks
sampled rows of the gathered matrix on rank 0. The stub evaluates the blocks with the oracle,
so this pins the orchestration (column ranges, max-over-ranks reductions, the gather and the
row check), not the GPU kernels (tests/test_full_parity_gpu.py does that). Also: `--gpus N`
without torchrun must refuse to run on fewer than N visible GPUs instead of timing one.
"""
import os
import socket
import subprocess
import sys
import time

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class CpuStub:
    """The backend interface bench.c5_sweep uses, on CPU tensors and the oracle."""

    p2p = False  # no CUDA IPC on CPU: the fused-epilogue gather is GPU-only

    def __init__(self):
        import oracle
        self.orc = oracle.Oracle()

    def upload(self, words):
        return torch.from_numpy(np.ascontiguousarray(words).view(np.int64).copy())

    def empty(self, rows, cols):
        return torch.empty((rows, cols), dtype=torch.int32)

    def gemm(self, a, b, k, out):
        wpr = a.shape[1]
        u, _ = self.orc.gemm_1x1(a.contiguous().numpy().view(np.uint64), b.contiguous().numpy().view(np.uint64),
                                 k, wpr)
        out.copy_(torch.from_numpy(u))

    def time(self, fn, reps):
        fn()
        out = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            out.append((time.perf_counter() - t0) * 1e3)
        return out

    def reduce_max(self, dist_, v):
        t = torch.tensor([v], dtype=torch.float64)
        dist_.all_reduce(t, op=dist_.ReduceOp.MAX)
        return float(t.item())

    def status(self):
        pass


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, REPO)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        res = bench.c5_sweep(CpuStub(), dist, world, rank, 96, 200, 300, reps=1, check_rows=5)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_c5_sweep_orchestration_world2():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    root = out[0]
    assert root["n_ranks"] == 2 and root["columns_per_rank"] == 100
    assert root["rows_match"] == {"single_gpu": True, "nccl": True}
    assert root["nccl_bytes_to_root"] == 96 * 100 * 2  # one rank's block as uint16 popcounts
    for key in ("kernel_ms", "nccl_gather_ms", "single_gpu_ms", "nccl_gather_speedup_vs_1gpu"):
        assert root[key] > 0
    assert "p2p_gather_ms" not in root  # no CUDA IPC on CPU
    assert out[1]["kernel_ms"] == root["kernel_ms"]  # max over ranks, the same on every rank


def test_gpus_flag_refuses_missing_gpus():
    import torch as _t
    visible = _t.cuda.device_count()
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", str(max(2, visible + 1)),
                        "--steps", "1", "--warmup", "0"], cwd=REPO, env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode != 0
    assert "refusing" in r.stderr
