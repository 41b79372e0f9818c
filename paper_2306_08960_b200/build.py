"""Build recipe for the sm_100a shared library (in-tree, so it travels to the GPU box).

    python -m paper_2306_08960_b200.build          # builds libbitmm_b200.so next to this file

nvcc cross-compiles here without a GPU. The library links cudart statically so it
does not depend on which libcudart torch happens to have loaded.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG_DIR)
CSRC = os.path.join(PKG_DIR, "csrc")
INCLUDE = os.path.join(REPO, "include")
LIB_NAME = "libbitmm_b200.so"
LIB_PATH = os.path.join(PKG_DIR, LIB_NAME)

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "--expt-relaxed-constexpr",
    "-Xcompiler",
    "-fPIC",
    "-Xcompiler",
    "-Wall",
    "-Xptxas",
    "-v",
]
SOURCES = ["bitmm_capi.cu", "wire_host.cpp"]


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found")
    return cand


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = LIB_PATH,
          extra: tuple = ()) -> str:
    """Build the library into `out` (default: the in-tree libbitmm_b200.so). `extra`: more
    nvcc flags (A/B variants, e.g. ("-DFX_STATS",), built next to the product library)."""
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(INCLUDE, "bitmm_b200.h"),
        os.path.abspath(__file__),
    ]
    if not force and not extra and not _stale(out, deps):
        return out
    tmp = out + ".tmp"
    cmd = (
        [nvcc()]
        + ARCH_FLAGS
        + NVCC_FLAGS
        + os.environ.get("BITMM_NVCC_EXTRA", "").split()  # A/B builds, e.g. -DSPMM_SCRATCH
        + list(extra)
        + ["-I", INCLUDE, "-I", CSRC, "-shared", "-o", tmp]
        + [os.path.join(CSRC, s) for s in SOURCES]
        + ["-cudart", "static", "-Xlinker", "-soname=libbitmm_b200.so"]
    )
    proc = subprocess.run(cmd, capture_output=True, text=True)
    log_path = os.path.join(PKG_DIR, "build.log") if out == LIB_PATH else out + ".log"
    with open(log_path, "w") as f:
        f.write(" ".join(cmd) + "\n" + proc.stdout + proc.stderr)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError(f"nvcc failed (see {log_path})")
    if verbose:
        sys.stdout.write(proc.stdout + proc.stderr)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    # python -m paper_2306_08960_b200.build [--force] [-v] [--out PATH -- NVCC_FLAGS...]
    argv = sys.argv[1:]
    extra = tuple(argv[argv.index("--") + 1:]) if "--" in argv else ()
    out = argv[argv.index("--out") + 1] if "--out" in argv else LIB_PATH
    print(build(force="--force" in argv, verbose="-v" in argv, out=os.path.abspath(out), extra=extra))
