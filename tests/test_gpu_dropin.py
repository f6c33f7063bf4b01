"""Drop-in proof on the GPU: the reference's own Executor + replay harness
(unmodified src/executor.cpp, src/workload.cpp) drives the B200 index through
include/bivf_vector_index.hpp, and its results equal the reference
ClusterIndex loaded from the same snapshot (oracle/ref_dropin.cpp)."""
import os
import subprocess

import pytest

from helpers import ROOT

BIN = os.path.join(ROOT, "oracle", "_ref", "ref_dropin")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/ref_dropin not built")
def test_reference_executor_drives_gpu_index(gpu_ready, tmp_path):
    r = subprocess.run([BIN, str(tmp_path / "snap.bivf")], capture_output=True, text=True,
                       timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatches=0" in r.stdout
