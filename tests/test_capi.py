"""CPU checks of the C-ABI library: it loads, exports exactly what
include/bivf.h declares, maps errors without a GPU (no silent fallback), and
its host-side helpers reproduce the reference's golden vectors."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from helpers import GOLDEN, ROOT

import paper_2408_02937_b200 as bivf
from paper_2408_02937_b200 import _lib


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "bivf.h")).read()
    decl = r"^(?:bivf_status|const char\*|int|uint64_t|void)\s+(bivf_[a-z0-9_]+)\("
    return sorted(set(re.findall(decl, txt, flags=re.M)))


def test_library_exports_every_header_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (bivf_[a-z0-9_]+)", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing
    # and the ctypes table covers them all
    assert sorted(_lib.SIGNATURES) == header_symbols()


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_fails_loudly_or_runs():
    L = _lib.lib()
    cfg = _lib.Config()
    cfg.dim = 8
    cfg.num_clusters = 4
    h = C.c_void_p()
    rc = L.bivf_create(C.byref(cfg), C.byref(h))
    if L.bivf_device_count() == 0:
        assert rc == _lib.ECUDA
        assert b"no CPU fallback" in L.bivf_last_error()
        with pytest.raises(bivf.CudaError):
            bivf.ClusterIndex(np.zeros((8, 8), np.float32), clusters=4)
    else:
        assert rc == _lib.OK
        L.bivf_destroy(h)


def test_config_validation_maps_to_value_error():
    L = _lib.lib()
    cfg = _lib.Config()  # dim 0
    h = C.c_void_p()
    assert L.bivf_create(C.byref(cfg), C.byref(h)) == _lib.EINVAL
    assert b"dim" in L.bivf_last_error()
    with pytest.raises(ValueError):
        _lib.check(_lib.EINVAL)


def test_synthetic_dataset_matches_reference_golden():
    z = np.load(os.path.join(GOLDEN, "primitives.npz"))
    for key in z.files:
        if not key.startswith("ds_"):
            continue
        n, d, c, s = (int(v) for v in key.split("_")[1:])
        got = bivf.synthetic_dataset(n, d, c, s)
        assert np.array_equal(got.view(np.uint32), z[key].view(np.uint32)), key


def test_pool_sizing_formula_matches_bindings():
    # bindings.cpp:43-45
    from paper_2408_02937_b200.index import build_config
    cfg = build_config(600, 16, 8, 16, 256, 0, 25, 3)
    assert cfg.num_blocks == (2 * 600 + 15) // 16 + 2 * 8 + 64
    assert cfg.nprobe_default == 8


def test_error_types_mirror_reference():
    with pytest.raises(bivf.PoolExhaustedError) as ei:
        _lib.check(_lib.EPOOL, inserted=4)
    assert ei.value.inserted == 4
    with pytest.raises(IndexError):
        _lib.check(_lib.ERANGE)
    with pytest.raises(bivf.CorruptListError):
        _lib.check(_lib.ECORRUPT)
