// Count of kernel launches issued by libbivf_gpu.so (bench.py's
// gpu_launches, read through bivf_kernel_launches()).
#pragma once
#include <atomic>
#include <cstdint>

namespace bivf {
extern std::atomic<uint64_t> g_launches;
// per-thread count too: a CUDA-graph capture measures the launches it records
inline thread_local uint64_t t_launches = 0;
inline void count_launch(uint64_t n = 1) {
    g_launches.fetch_add(n, std::memory_order_relaxed);
    t_launches += n;
}
}  // namespace bivf
