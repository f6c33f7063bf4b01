"""The reference's OWN test suites against the B200 index.

proj/tests/test_ivf_index.cpp, test_rearrange.cpp, test_concurrency.cpp and
test_executor.cpp (the reference Executor driving the GPU index) —
unmodified — compiled by oracle/Makefile (`make -C oracle ref`) with
oracle/gpu_suite_shim.hpp force-included: `ClusterIndex` becomes a class over
the C-ABI (libbivf_gpu.so), so every search, insert, assign, rearrangement,
block header, hop count, snapshot and concurrent-access check of those suites
runs on the GPU index (full-probe exactness test_ivf_index.cpp:142-160,
rearrange-during-search test_concurrency.cpp:142-186, ...).  The binaries are
built here (they need /root/reference) and travel with the repo."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITES = ["ivf_index", "rearrange", "concurrency", "executor"]


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_gpu_index(gpu_ready, suite):
    exe = os.path.join(ROOT, "oracle", "_ref", f"suite_{suite}")
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (make -C oracle ref needs /root/reference)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(r.stdout[-2000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
    assert "0 failed; assertions" in r.stdout
