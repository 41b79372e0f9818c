import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def _gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


HAS_GPU = _gpu_available()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.Oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle
    r = oracle.load_ref()
    if r is None:
        pytest.skip("oracle/_ref/libbitmm_ref.so not built (needs /root/reference)")
    return r


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name)))


@pytest.fixture(scope="session")
def gemm_golden():
    return load_golden("gemm_cases.npz")


@pytest.fixture(scope="session")
def apb_golden():
    return load_golden("apb_cases.npz")


@pytest.fixture(scope="session")
def packing_golden():
    return load_golden("packing_cases.npz")


def gemm_case(g, i):
    p = f"g{i:03d}_"
    m, k, n, wpr, lane = (int(x) for x in g[p + "shape"])
    s_w, s_a, g_a, g_b, g_w = (float(x) for x in g[p + "params"])
    return dict(m=m, k=k, n=n, wpr=wpr, lane=lane, s_w=s_w, s_a=s_a, g_a=g_a, g_b=g_b, g_w=g_w,
                a=g[p + "a"], b=g[p + "b"], lw=g[p + "lw"], la=g[p + "la"], c11=g[p + "c11"],
                c12=g[p + "c12"], c22=g[p + "c22"])


def apb_case(g, i):
    p = f"a{i:03d}_"
    d = {k[len(p):]: v for k, v in g.items() if k.startswith(p)}
    m, k, n, wpr = (int(x) for x in d["shape"])
    d.update(m=m, k=k, n=n, wpr=wpr)
    return d
