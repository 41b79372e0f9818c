"""bench.py's multi-rank path end to end on ONE GPU: two ranks (torchrun) sharing cuda:0, with the
host-side collectives on gloo (BITMM_BENCH_BACKEND=gloo). It runs the weak-scaled step, the
timed gather and the config-5 sweep (kernel-only, the gather fused into the epilogue through
CUDA IPC, the NCCL-path gather) and must print one JSON line for two ranks whose sampled rows of
both gathered 32768 x 32768 matrices match rank 0's own evaluation. Not a scaling measurement;
the ranks' kernels do not wait on each other."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_on_one_gpu():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, BITMM_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(REPO, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--no-e2e", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["gpu_launches"] > 0
    assert line["gather"]["bytes_to_root_per_step"] > 0
    sw = line["c5_sweep"]
    assert sw["n_ranks"] == 2 and sw["columns_per_rank"] == 16384
    assert sw["rows_match"] == {"single_gpu": True, "p2p": True, "nccl": True}
    for key in ("kernel_ms", "p2p_gather_ms", "nccl_gather_ms", "single_gpu_ms"):
        assert sw[key] > 0
