"""pytest configuration: markers, repo on sys.path, shared helpers."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long CPU test, opt-in with LOKA_SLOW=1")
    config.addinivalue_line("markers", "dist: multi-process torch.distributed test (gloo on CPU)")


def pytest_collection_modifyitems(config, items):
    if os.environ.get("LOKA_SLOW") == "1":
        return
    skip = pytest.mark.skip(reason="slow test; set LOKA_SLOW=1")
    for it in items:
        if "slow" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def fp8_host_cast(tmp_path_factory):
    """Build the test-only cuda_fp8.hpp host-cast helper (tests/helpers/fp8_host_cast.cpp)."""
    out = tmp_path_factory.mktemp("helpers") / "fp8_host_cast"
    src = os.path.join(ROOT, "tests", "helpers", "fp8_host_cast.cpp")
    cuda_inc = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "include")
    r = subprocess.run(["g++", "-O2", "-I", cuda_inc, src, "-o", str(out)], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("cannot build cuda_fp8 host helper: " + r.stderr[-300:])
    return str(out)


@pytest.fixture(autouse=True)
def _gpu_watchdog(request):
    """For GPU tests: fail loudly if a GEMM pipeline wait timed out (libloka's mbarrier watchdog)."""
    yield
    if "gpu" not in request.keywords:
        return
    import torch
    if not torch.cuda.is_available():
        return
    import paper_2605_10886_b200 as lk
    torch.cuda.synchronize()
    n, tag, blk, thr = lk.debug_hang_info(reset=True)
    assert n == 0, f"pipeline watchdog: {n} timed-out waits, tag={tag} block={blk} thread={thr & 0xffffffff} parity={thr >> 32}"


@pytest.fixture(scope="session")
def fp4_host_cast(tmp_path_factory):
    """Build the test-only cuda_fp4.hpp host-cast helper (tests/helpers/fp4_host_cast.cpp)."""
    out = tmp_path_factory.mktemp("helpers4") / "fp4_host_cast"
    src = os.path.join(ROOT, "tests", "helpers", "fp4_host_cast.cpp")
    cuda_inc = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "include")
    r = subprocess.run(["g++", "-O2", "-I", cuda_inc, src, "-o", str(out)], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("cannot build cuda_fp4 host helper: " + r.stderr[-300:])
    return str(out)
