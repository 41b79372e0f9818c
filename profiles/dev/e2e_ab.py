"""e2e pass of bench.py alone (the three host calls on pinned buffers), for A/B of the host
wire's settings in separate processes: BITMM_WIRE_SPIN=1 python profiles/dev/e2e_ab.py [label]"""
import sys
import types

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2306_08960_b200 import _lib  # noqa: E402

lib = _lib.load()
ops = bench.make_operands(np.random.default_rng(bench.SEED))
args = types.SimpleNamespace(steps=10, warmup=3)
vals, seq = [], []
for _ in range(3):
    r = bench.e2e_pass(args, ops, torch, lib)
    vals.append(r["value"])
    seq.append(r["per_call"]["value"])
print(sys.argv[1] if len(sys.argv) > 1 else "", "e2e T-upd/s batch:", " ".join(f"{v:.1f}" for v in vals),
      "| per call:", " ".join(f"{v:.1f}" for v in seq),
      "| ms/call:", {k: round(v, 3) for k, v in r["per_call"]["ms_per_call"].items()},
      "| pageable:", round(r["pageable_host_buffers"]["value"], 1), flush=True)
