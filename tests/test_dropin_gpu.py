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


VERIFY_B200 = os.path.join(REPO, "oracle", "_ref", "verify_b200")
VERIFY_ROWOPS = os.path.join(REPO, "oracle", "_ref", "verify_b200_rowops")
VERIFY_REF = os.path.join(REPO, "oracle", "_ref", "verify_ref")


@pytest.mark.skipif(not os.path.exists(VERIFY_B200), reason="verify_b200 not built (needs /root/reference)")
def test_reference_verification_sweep_on_b200():
    """bitmm::run_verification (verify.cpp:352-376, unmodified) with the GEMMs and packers on
    the B200: every suite passes, and the report is identical to the one the reference's own
    CPU library prints for the same options (the sweep is deterministic per seed)."""
    got = subprocess.run([VERIFY_B200], capture_output=True, text=True, timeout=900)
    assert got.returncode == 0, got.stdout + got.stderr
    assert "all suites passed" in got.stdout and "suite gemm-bitwise-vs-oracle" in got.stdout
    want = subprocess.run([VERIFY_REF], capture_output=True, text=True, timeout=900)
    assert want.returncode == 0
    assert got.stdout == want.stdout


@pytest.mark.skipif(not os.path.exists(VERIFY_B200), reason="verify_b200 not built (needs /root/reference)")
def test_reference_verification_fault_injection_on_b200():
    """--inject-fault adds 1.0 to C[0][0] of the first 1/1 case (verify.cpp:257): the sweep must
    fail and name it, as the reference CLI test expects (test_bench_cli.cpp:205-210)."""
    r = subprocess.run([VERIFY_B200, "--gemm-cases", "2", "--max-dim", "12", "--inject-fault"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 1
    for s in ("verification FAILED", "first failure", "routine=1x1", "cell=(0,0)"):
        assert s in r.stdout, r.stdout


@pytest.mark.skipif(not os.path.exists(VERIFY_ROWOPS), reason="verify_b200_rowops not built")
def test_reference_verification_with_row_ops_on_b200():
    """The same sweep with dot_binary / mbm (kernels.cpp:120-140) also routed to the GPU, one
    row pair per call (reduced exhaustive lengths: each call is a launch)."""
    args = ["--dot-n", "6", "--mbm-n", "4", "--rowop-cases", "300", "--gemm-cases", "6", "--max-dim", "40"]
    got = subprocess.run([VERIFY_ROWOPS] + args, capture_output=True, text=True, timeout=900)
    assert got.returncode == 0, got.stdout + got.stderr
    want = subprocess.run([VERIFY_REF] + args, capture_output=True, text=True, timeout=900)
    assert got.stdout == want.stdout
