"""GPU: the reference's OWN acceptance suite (proj/tests/acceptance.cpp, unmodified) run with
the six GEMM entry points replaced by integration/reference_dropin/kernels_b200.cpp — i.e.
gemm_1x1 / gemm_1x2 / gemm_2x2 / gemm_1x32_ref / spmm_csr / layer_forward executing on the
B200 through the C ABI. Built here by `make -C oracle dropin` (needs /root/reference); the
binary travels to the GPU box prebuilt.

Gates criteria 1-7 (row ops, 220-shape GEMM equality at tolerance 0, plane bijection, 100
APB layers within 1e-4, gradients, memory and throughput models). Criterion 8 checks the
CPU cost ORDER t(1x1) < t(1x2) < t(2x2) of the bit-serial algorithms; on the tensor-core
path all three cost one int8 MAC per update, so it is recorded, not gated."""
import os
import re
import subprocess

import pytest

from conftest import REPO

BIN = os.path.join(REPO, "oracle", "_ref", "acceptance_b200")
pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="acceptance_b200 not built (needs /root/reference)")
def test_reference_acceptance_suite_with_b200_kernels():
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=900).stdout
    verdicts = dict(re.findall(r"^\[(\d+)\] (PASS|FAIL|SKIP)", out, flags=re.M))
    print(out)
    for crit in ("1", "2", "3", "4", "5", "6", "7"):
        assert verdicts.get(crit) == "PASS", f"criterion {crit}: {out}"
    assert "220 shapes" in out and " 0 mismatches" in out
