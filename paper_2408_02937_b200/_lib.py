"""ctypes binding of libbivf_gpu.so (include/bivf.h).

There is no fallback: if the shared library is missing this module raises on
import, and every compute call on a host without a CUDA device returns
BIVF_ECUDA, which surfaces as CudaError.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

# BIVF_LIB: an alternative in-tree build of the same library (kernel variants under test)
LIB_PATH = os.environ.get("BIVF_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libbivf_gpu.so")

OK, EINVAL, EPOOL, ECORRUPT, ERANGE, ELOGIC, EIO, ECUDA, EBUSY, ENOMEM = range(10)
METRIC_L2, METRIC_IP = 0, 1


class BivfError(RuntimeError):
    code = -1


class PoolExhaustedError(BivfError):
    """Mirror of blockivf::PoolExhaustedError (types.hpp:19-30)."""

    code = EPOOL

    def __init__(self, msg, inserted=0, ids=None):
        super().__init__(msg)
        self.inserted = inserted
        self.ids = ids


class CorruptListError(BivfError):
    code = ECORRUPT


class CudaError(BivfError):
    code = ECUDA


class BusyError(BivfError):
    code = EBUSY


class Config(C.Structure):
    _fields_ = [
        ("num_clusters", C.c_uint64),
        ("dim", C.c_uint64),
        ("nprobe_default", C.c_uint64),
        ("rearrange_threshold", C.c_uint64),
        ("kmeans_iters", C.c_uint64),
        ("kmeans_seed", C.c_uint64),
        ("num_blocks", C.c_uint64),
        ("block_capacity", C.c_uint64),
        ("alert_watermark", C.c_double),
        ("metric", C.c_int32),
        ("device", C.c_int32),
        ("num_leases", C.c_uint32),
        ("max_list_blocks", C.c_uint32),
        ("kmeans_seed_set", C.c_uint32),
        ("reserved", C.c_uint32 * 7),
    ]


class ExecutorConfig(C.Structure):
    _fields_ = [
        ("num_lanes", C.c_uint32),
        ("central_grants", C.c_uint32),
        ("lane_cache_bytes", C.c_uint64),
        ("central_grant_bytes", C.c_uint64),
        ("flush_interval_ms", C.c_uint32),
        ("batch_multiple", C.c_uint32),
        ("batch_cap", C.c_uint32),
        ("max_search_batch", C.c_uint32),
        ("serialized", C.c_int32),
        ("reserved", C.c_uint32 * 5),
    ]


class TicketInfo(C.Structure):
    _fields_ = [
        ("status", C.c_int32),
        ("type", C.c_int32),
        ("lane", C.c_int32),
        ("nq", C.c_uint32),
        ("k", C.c_uint32),
        ("n", C.c_uint64),
        ("latency_us", C.c_double),
        ("queue_us", C.c_double),
        ("exec_us", C.c_double),
    ]


class ReplaySpec(C.Structure):
    _fields_ = [
        ("qps_search", C.c_double),
        ("qps_insert", C.c_double),
        ("duration_s", C.c_double),
        ("search_batch", C.c_uint32),
        ("insert_batch", C.c_uint32),
        ("k", C.c_uint32),
        ("nprobe", C.c_uint32),
        ("seed", C.c_uint64),
        ("poisson", C.c_int32),
        ("reserved", C.c_uint32 * 5),
    ]


_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

vp, u64, u32, i32, i64 = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int32, C.c_int64
pu64 = C.POINTER(u64)

# name -> (restype, argtypes); mirrors include/bivf.h one to one
SIGNATURES = {
    "bivf_last_error": (C.c_char_p, []),
    "bivf_version": (C.c_char_p, []),
    "bivf_device_count": (C.c_int, []),
    "bivf_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(vp)]),
    "bivf_host_free": (C.c_int, [vp]),
    "bivf_create": (C.c_int, [C.POINTER(Config), C.POINTER(vp)]),
    "bivf_destroy": (C.c_int, [vp]),
    "bivf_get_config": (C.c_int, [vp, C.POINTER(Config)]),
    "bivf_train": (C.c_int, [vp, _f32p, u64]),
    "bivf_set_centroids": (C.c_int, [vp, _f32p]),
    "bivf_get_centroids": (C.c_int, [vp, _f32p]),
    "bivf_bulk_load": (C.c_int, [vp, vp, u64, vp, vp]),
    "bivf_save_snapshot": (C.c_int, [vp, C.c_char_p]),
    "bivf_load_snapshot": (C.c_int, [C.c_char_p, C.POINTER(Config), C.POINTER(vp)]),
    "bivf_load_snapshot_shard": (C.c_int, [C.c_char_p, u32, u32, C.POINTER(Config), C.POINTER(vp)]),
    "bivf_pool_alert": (C.c_int, [vp, C.POINTER(i32), pu64]),
    "bivf_seed_samples": (C.c_int, [vp, vp, u64, pu64]),
    "bivf_block_set_next": (C.c_int, [vp, i32, i32]),
    "bivf_exact_knn": (C.c_int, [vp, u64, u64, vp, u64, u64, i32, i32, vp, vp, vp]),
    "bivf_add": (C.c_int, [vp, vp, u64, vp, vp, pu64]),
    "bivf_search": (C.c_int, [vp, vp, u64, u64, u64, vp, vp, vp]),
    "bivf_search_device": (C.c_int, [vp, vp, u64, u64, u64, vp, vp, vp, vp]),
    "bivf_assign": (C.c_int, [vp, vp, u64, vp]),
    "bivf_probes": (C.c_int, [vp, vp, u64, u64, vp]),
    "bivf_remove": (C.c_int, [vp, vp, u64, pu64, vp]),
    "bivf_exceed": (C.c_int, [vp, u32, C.POINTER(C.c_int)]),
    "bivf_rearrange": (C.c_int, [vp, u32]),
    "bivf_rearrange_sweep": (C.c_int, [vp]),
    "bivf_take_rearrange_events": (C.c_int, [vp, vp, u64, pu64]),
    "bivf_size": (C.c_int, [vp, pu64]),
    "bivf_scalars_copied": (C.c_int, [vp, pu64]),
    "bivf_reallocations": (C.c_int, [vp, pu64]),
    "bivf_cow_ops": (C.c_int, [vp, pu64]),
    "bivf_quiescent_ops": (C.c_int, [vp, pu64]),
    "bivf_extend_copy": (C.c_int, [vp, vp, u64, vp, vp, pu64]),
    "bivf_list_length": (C.c_int, [vp, u32, pu64]),
    "bivf_offline_count": (C.c_int, [vp, u32, pu64]),
    "bivf_hop_count": (C.c_int, [vp, u32, pu64]),
    "bivf_online_head": (C.c_int, [vp, u32, C.POINTER(i32)]),
    "bivf_allocated_blocks": (C.c_int, [vp, pu64]),
    "bivf_block_header": (C.c_int, [vp, i32, _i32p]),
    "bivf_block_ids": (C.c_int, [vp, i32, _i64p]),
    "bivf_block_payload": (C.c_int, [vp, i32, _f32p]),
    "bivf_cluster_contents": (C.c_int, [vp, u32, vp, vp, pu64]),
    "bivf_dump_pool": (C.c_int, [vp, C.c_char_p, u64, pu64]),
    "bivf_next_id": (C.c_int, [vp, C.POINTER(i64)]),
    "bivf_synthetic_dataset": (C.c_int, [u64, u64, u64, u64, _f32p]),
    "bivf_kmeans": (C.c_int, [_f32p, u64, u64, u64, u64, u64, i32, _f32p, _u32p, pu64]),
    "bivf_merge_topk_device": (C.c_int, [i32, vp, vp, u64, u64, u64, vp, vp, vp, vp]),
    "bivf_nccl_unique_id": (C.c_int, [vp]),
    "bivf_group_create_local": (C.c_int, [C.POINTER(vp), u32, C.POINTER(vp)]),
    "bivf_group_create_nccl": (C.c_int, [vp, vp, i32, i32, u32, C.POINTER(vp)]),
    "bivf_group_destroy": (None, [vp]),
    "bivf_group_size": (C.c_int, [vp, C.POINTER(u32)]),
    "bivf_group_search": (C.c_int, [vp, vp, u64, u64, u64, vp, vp, vp, u32]),
    "bivf_group_search_device": (C.c_int, [vp, vp, u64, u64, u64, vp, vp, vp, vp, u32]),
    "bivf_group_insert": (C.c_int, [vp, vp, u64, vp, vp, pu64]),
    "bivf_group_remove": (C.c_int, [vp, vp, u64, pu64, vp]),
    "bivf_executor_create": (C.c_int, [vp, C.POINTER(ExecutorConfig), C.POINTER(vp)]),
    "bivf_executor_destroy": (C.c_int, [vp]),
    "bivf_executor_submit_search": (C.c_int, [vp, vp, u64, u64, u64, C.POINTER(vp)]),
    "bivf_executor_submit_insert": (C.c_int, [vp, vp, u64, vp, C.POINTER(vp)]),
    "bivf_executor_flush": (C.c_int, [vp]),
    "bivf_executor_set_mode": (C.c_int, [vp, C.c_int]),
    "bivf_executor_shutdown": (C.c_int, [vp]),
    "bivf_executor_stats": (C.c_int, [vp, vp]),
    "bivf_ticket_wait": (C.c_int, [vp, C.POINTER(TicketInfo)]),
    "bivf_ticket_results": (C.c_int, [vp, vp, vp, vp]),
    "bivf_ticket_error": (C.c_int, [vp, C.c_char_p, u64]),
    "bivf_ticket_free": (C.c_int, [vp]),
    "bivf_replay": (C.c_int, [vp, C.POINTER(ReplaySpec), vp, u64, vp, u64, vp, u64, pu64, vp, u64,
                              pu64, pu64, pu64]),
    "bivf_kernel_launches": (u64, []),
    "bivf_set_scan_mode": (C.c_int, [vp, C.c_int]),
    "bivf_prewarm": (C.c_int, [vp, C.c_uint64, C.c_uint64, C.c_uint64]),
    "bivf_set_timing": (C.c_int, [vp, C.c_int]),
    "bivf_last_timings": (C.c_int, [vp, C.POINTER(C.c_float)]),
}

_lib = None


def lib():
    """Load libbivf_gpu.so (fail loudly: there is no CPU implementation)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2408_02937_b200.build` "
                "(the B200 path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc, inserted=None, ids=None):
    if rc == OK:
        return
    msg = lib().bivf_last_error().decode(errors="replace")
    if rc == EINVAL:
        raise ValueError(msg)
    if rc == EPOOL:
        raise PoolExhaustedError(msg, inserted or 0, ids)
    if rc == ERANGE:
        raise IndexError(msg)
    if rc == ECORRUPT:
        raise CorruptListError(msg)
    if rc == ECUDA:
        raise CudaError(msg)
    if rc == EBUSY:
        raise BusyError(msg)
    if rc == ENOMEM:
        raise MemoryError(msg)
    err = BivfError(msg)
    err.code = rc
    raise err


def ptr(a):
    return None if a is None else a.ctypes.data
