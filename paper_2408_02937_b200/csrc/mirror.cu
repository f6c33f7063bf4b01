// Tensor-core scan mirror maintenance (see mirror.cuh).  sm_100a.
#include <algorithm>

#include "launches.h"
#include "maint.cuh"
#include "mirror.cuh"

namespace bivf {

namespace {

__device__ __forceinline__ float tf32_trunc_m(float x) {
    return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

// one vector -> its mirror column `lane` of group `g`.  x[d * xs] is dim d.
__device__ __forceinline__ void mirror_column(float* g, uint32_t lane, const float* x, uint32_t xs,
                                              const float* c, uint32_t D) {
    float n2 = 0.f;
    for (uint32_t d = 0; d < D; ++d) {
        const float s = __fsub_rn(x[(uint64_t)d * xs], c[d]);
        const float h = tf32_trunc_m(s);
        g[(uint64_t)d * 32u + lane] = h;
        g[(uint64_t)(D + 1 + d) * 32u + lane] = __fsub_rn(s, h);
        n2 = __fadd_rn(n2, __fmul_rn(s, s));
    }
    g[(uint64_t)D * 32u + lane] = n2;
    g[(uint64_t)(2 * D + 1) * 32u + lane] = sqrtf(n2);
}

__device__ __forceinline__ float* mirror_slot(const MirrorView& M, uint64_t a, uint32_t& lane) {
    if (a >> 63) {
        const uint64_t gs = a & ~(1ull << 63);
        const uint64_t blk = gs / M.T, slot = gs - blk * M.T;
        lane = (uint32_t)(slot & 31u);
        return M.arena_mir + blk * M.MPS + (slot >> 5) * M.GF;
    }
    lane = (uint32_t)(a & 31u);
    return M.off_mir + (a >> 5) * M.GF;
}

__global__ void mirror_insert_kernel(MirrorView M, uint32_t n, const float* x, const uint32_t* asg,
                                     const int32_t* out_blk, const uint32_t* out_did) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t b = out_blk[i];
    if (b < 0) return;
    const uint32_t slot = out_did[i] % M.T;
    float* g = M.arena_mir + (uint64_t)b * M.MPS + (uint64_t)(slot >> 5) * M.GF;
    mirror_column(g, slot & 31u, x + (uint64_t)i * M.D, 1, M.cent + (uint64_t)asg[i] * M.D, M.D);
}

__global__ void mirror_offline_kernel(MirrorView M, uint32_t n, const float* x,
                                      const uint64_t* dest, const uint32_t* asg) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t s = dest[i];
    mirror_column(M.off_mir + (s >> 5) * M.GF, (uint32_t)(s & 31u), x + (uint64_t)i * M.D, 1,
                  M.cent + (uint64_t)asg[i] * M.D, M.D);
}

// warp per group, lane = slot: payload group rows are coalesced
__global__ void mirror_groups_kernel(MirrorView M, const float* payload, int arena, uint64_t PS,
                                     const uint64_t* groups, const uint32_t* cl, uint32_t n) {
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31u;
    if (w >= n) return;
    const uint64_t gi = groups[w];
    const float* src;
    float* dst;
    if (arena) {
        const uint64_t blk = gi / M.gpb, j = gi - blk * M.gpb;
        src = payload + blk * PS + j * 32ull * M.D;
        dst = M.arena_mir + blk * M.MPS + j * M.GF;
    } else {
        src = payload + gi * 32ull * M.D;
        dst = M.off_mir + gi * M.GF;
    }
    mirror_column(dst, lane, src + lane, 32, M.cent + (uint64_t)cl[w] * M.D, M.D);
}

__global__ void mirror_slot_move_kernel(MirrorView M, const uint64_t* id_addr, uint32_t n,
                                        float* scr, int phase) {
    const uint32_t R = 2 * M.D + 2;
    const uint64_t total = (uint64_t)n * R;
    for (uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total;
         o += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t m = (uint32_t)(o / R), r = (uint32_t)(o - (uint64_t)m * R);
        uint32_t lane;
        if (phase == 0) {
            const float* g = mirror_slot(M, id_addr[m], lane);
            scr[o] = g[(uint64_t)r * 32u + lane];
        } else {
            float* g = mirror_slot(M, id_addr[n + m], lane);
            g[(uint64_t)r * 32u + lane] = scr[o];
        }
    }
}

}  // namespace

cudaError_t launch_mirror_insert(const MirrorView& M, uint32_t n, const float* x,
                                 const uint32_t* asg, const int32_t* out_blk,
                                 const uint32_t* out_did, cudaStream_t s) {
    if (!n || !M.arena_mir) return cudaSuccess;
    mirror_insert_kernel<<<(n + 127) / 128, 128, 0, s>>>(M, n, x, asg, out_blk, out_did);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_mirror_offline(const MirrorView& M, uint32_t n, const float* x,
                                  const uint64_t* dest, const uint32_t* asg, cudaStream_t s) {
    if (!n || !M.off_mir) return cudaSuccess;
    mirror_offline_kernel<<<(n + 127) / 128, 128, 0, s>>>(M, n, x, dest, asg);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_mirror_groups(const MirrorView& M, const float* payload, bool arena,
                                 uint64_t PS, const uint64_t* groups, const uint32_t* cl,
                                 uint32_t n, cudaStream_t s) {
    if (!n || !(arena ? M.arena_mir : M.off_mir)) return cudaSuccess;
    mirror_groups_kernel<<<(n + 3) / 4, 128, 0, s>>>(M, payload, arena ? 1 : 0, PS, groups, cl, n);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_mirror_slot_moves(const MirrorView& M, const uint64_t* id_addr, uint32_t n,
                                     float* scratch, cudaStream_t s) {
    if (!n || !M.off_mir) return cudaSuccess;
    const uint64_t total = (uint64_t)n * (2 * M.D + 2);
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((total + 255) / 256, 148 * 16));
    for (int phase = 0; phase < 2; ++phase) {
        mirror_slot_move_kernel<<<g, 256, 0, s>>>(M, id_addr, n, scratch, phase);
        count_launch();
    }
    return cudaGetLastError();
}

}  // namespace bivf
