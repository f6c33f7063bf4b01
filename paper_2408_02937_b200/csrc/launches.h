// Count of kernel launches issued by libbivf_gpu.so (bench.py's
// gpu_launches, read through bivf_kernel_launches()).
#pragma once
#include <atomic>
#include <cstdint>

namespace bivf {
extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }
}  // namespace bivf
