"""CPU: the C-ABI library builds/loads, exports every symbol include/bitmm_b200.h declares,
and rejects bad arguments with the reference's error classes before touching a device."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from conftest import HAS_GPU, REPO
from paper_2306_08960_b200 import _lib, api


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    declared = _lib.header_symbols()
    assert len(declared) >= 20
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    # and the ctypes signature table covers exactly the declared surface
    assert sorted(_lib.SIGNATURES) == declared


def test_nm_dynamic_symbols_match_header():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(_lib.header_symbols()) <= exported


def test_library_is_sm100a_cubin():
    out = subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True,
                          check=True).stdout
    # UTCOMMA: the kind::mxf4 product path (the default); UTCIMMA / UTCHMMA: the int8 A/B
    # path and the fp16 APB GEMM; UTMALDG / UTMASTG: TMA loads and the epilogue's TMA stores;
    # LDTM / STTM: TMEM reads and the scale-factor fill
    for mnemonic in ("UTCOMMA.2CTA", "UTCIMMA", "UTCHMMA", "UTMALDG", "UTMASTG", "LDTM", "STTM"):
        assert mnemonic in sass, mnemonic


def test_abi_version():
    assert _lib.load().bitmm_abi_version() == 1


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def test_argument_errors_without_device():
    lib = _lib.load()
    a = np.zeros((1, 8), np.uint64)
    out = np.zeros((1, 1), np.float32)
    # dims <= 0, K over the 2^20 cap, words_per_row too small: invalid_argument class
    assert lib.bitmm_gemm_1x1_host(_p(a), 0, _p(a), 1, 3, 8, 1.0, 1.0, None, _p(out), 1) == _lib.ERR_INVALID_ARGUMENT
    assert lib.bitmm_gemm_1x1_host(_p(a), 1, _p(a), 1, (1 << 20) + 1, 8, 1.0, 1.0, None, _p(out), 1) == _lib.ERR_INVALID_ARGUMENT
    assert lib.bitmm_gemm_1x1_host(_p(a), 1, _p(a), 1, 513, 8, 1.0, 1.0, None, _p(out), 1) == _lib.ERR_INVALID_ARGUMENT
    assert "words_per_row" in _lib.last_error()
    # non-positive plane scale: InvalidEncoding class (tensor.cpp:140)
    assert lib.bitmm_gemm_1x2_dev(_p(a), 1, 1.0, _p(a), _p(a), _p(a), 1, 3, 8, 0.0, 0, 1.0, None, None,
                                  None, _p(out), 1, None) == _lib.ERR_INVALID_ENCODING
    assert lib.bitmm_spmm_csr_dev(0, 1, None, None, None, None, 1, 1, None, 1, None) == _lib.ERR_INVALID_ARGUMENT


@pytest.mark.skipif(HAS_GPU, reason="checks the no-device path")
def test_no_device_means_error_not_fallback():
    lib = _lib.load()
    a = np.zeros((1, 8), np.uint64)
    out = np.zeros((1, 1), np.float32)
    rc = lib.bitmm_gemm_1x1_host(_p(a), 1, _p(a), 1, 3, 8, 1.0, 1.0, None, _p(out), 1)
    assert rc == _lib.ERR_NO_DEVICE
    assert lib.bitmm_device_sm_count() == 0
    # the multi-GPU plan too (no plan is created)
    import ctypes as C
    plan = C.c_void_p()
    dv = (C.c_int * 1)(0)
    assert lib.bitmm_shard_plan_create(dv, 1, 64, 256, 512, 8, C.byref(plan)) == _lib.ERR_NO_DEVICE
    assert not plan.value
    with pytest.raises(_lib.BitmmError):
        api.gemm_1x1(api.BitMatrix(1, 3), api.BitMatrix(1, 3))


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(_lib.BitmmError):
        _lib.load()
    monkeypatch.setattr(_lib, "_lib", None)


def test_workspace_bytes_model():
    lib = _lib.load()
    # 1/1 4096^3: two expanded int8 operands of 16 MiB each
    assert lib.bitmm_workspace_bytes(0, 4096, 4096, 4096) >= 2 * 4096 * 4096
    # 1/32 (APB): fp16 signs + two fp16 parts of X^T + per-token scales
    assert lib.bitmm_workspace_bytes(3, 3072, 8192, 768) >= 2 * (3072 * 768 + 8192 * 2 * 768) + 4 * 8192
    assert lib.bitmm_workspace_bytes(0, 0, 1, 1) == 0


def test_header_compiles_as_c():
    hdr = os.path.join(REPO, "include", "bitmm_b200.h")
    src = f'#include "{hdr}"\nint main(void) {{ return bitmm_abi_version(); }}\n'
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-x", "c", "-fsyntax-only", "-"],
                   input=src, text=True, check=True)


def test_gemm_item_struct_layout_matches_c(tmp_path):
    """ctypes GemmItem and the C bitmm_gemm_item agree on size and every field offset."""
    import ctypes as C
    hdr = os.path.join(REPO, "include", "bitmm_b200.h")
    names = [f[0] for f in _lib.GemmItem._fields_]
    body = "".join(f'  printf("%zu\\n", offsetof(bitmm_gemm_item, {n}));\n' for n in names)
    src = (f'#include <stddef.h>\n#include <stdio.h>\n#include "{hdr}"\n'
           f'int main(void) {{\n  printf("%zu\\n", sizeof(bitmm_gemm_item));\n{body}  return 0;\n}}\n')
    exe = str(tmp_path / "layout")
    subprocess.run(["gcc", "-std=c99", "-x", "c", "-", "-o", exe], input=src, text=True, check=True)
    out = [int(x) for x in subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()]
    assert out[0] == C.sizeof(_lib.GemmItem)
    assert out[1:] == [getattr(_lib.GemmItem, n).offset for n in names]


def test_host_out_struct_layout_matches_c(tmp_path):
    """ctypes HostOut and the C bitmm_host_out (late-output callback) agree on the layout."""
    import ctypes as C
    hdr = os.path.join(REPO, "include", "bitmm_b200.h")
    names = [f[0] for f in _lib.HostOut._fields_]
    body = "".join(f'  printf("%zu\\n", offsetof(bitmm_host_out, {n}));\n' for n in names)
    src = (f'#include <stddef.h>\n#include <stdio.h>\n#include "{hdr}"\n'
           f'int main(void) {{\n  printf("%zu\\n", sizeof(bitmm_host_out));\n{body}  return 0;\n}}\n')
    exe = str(tmp_path / "layout")
    subprocess.run(["gcc", "-std=c99", "-x", "c", "-", "-o", exe], input=src, text=True, check=True)
    out = [int(x) for x in subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()]
    assert out[0] == C.sizeof(_lib.HostOut)
    assert out[1:] == [getattr(_lib.HostOut, n).offset for n in names]
    assert (_lib.WANT_UNITS, _lib.WANT_C) == (1, 2)
