"""B200-native online IVF-Flat path (RTAMS-GANNS, arXiv 2408.02937).

The product is libbivf_gpu.so (hand-written sm_100a kernels + C++ runtime
behind the C-ABI in include/bivf.h).  This package is the thin Python host
mirror of the reference's binding surface (blockivf._core) over that ABI.
"""
from ._lib import (BivfError, BusyError, CorruptListError, CudaError, METRIC_IP, METRIC_L2,
                   PoolExhaustedError)
from .index import (BaselineIndex, ClusterIndex, device_count, exact_knn, kernel_launches, kmeans, pinned_empty,
                    synthetic_dataset)

__all__ = [
    "ClusterIndex",
    "BaselineIndex",
    "pinned_empty",
    "PoolExhaustedError",
    "CorruptListError",
    "CudaError",
    "BusyError",
    "BivfError",
    "synthetic_dataset",
    "kmeans",
    "exact_knn",
    "device_count",
    "kernel_launches",
    "METRIC_L2",
    "METRIC_IP",
]

__version__ = "0.1.0"
