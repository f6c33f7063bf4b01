// Tensor-core scan mirror maintenance (see mirror.cuh).  sm_100a.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>

#include "launches.h"
#include "maint.cuh"
#include "mirror.cuh"

namespace bivf {

namespace {

// one vector -> its mirror column `lane` of group `g` (+ the group's norm block
// `nrm`).  x[d * xs] is dim d.  Planes are bf16 (mirror.cuh): s_hi = bf16_rn(s),
// s_lo = bf16_rn(s - s_hi).
__device__ __forceinline__ void mirror_column(float* gf, float* nrm, float* row, uint32_t lane,
                                              const float* x, uint32_t xs, const float* c,
                                              uint32_t D, uint32_t K, uint32_t wide) {
    uint16_t* g = reinterpret_cast<uint16_t*>(gf);
    float n2 = 0.f;
    if (wide) {  // inner product: uncentred fp16 plane scaled by 2^ev, norms [2^-ev][|x|]
        float mx = 0.f;
        for (uint32_t d = 0; d < D; ++d) mx = fmaxf(mx, fabsf(x[(uint64_t)d * xs]));
        const int ev = wide_scale_exp(mx);
        for (uint32_t d = 0; d < D; ++d) {
            const float xd = x[(uint64_t)d * xs];
            if (row) row[d] = xd;
            g[(uint64_t)d * 32u + lane] = __half_as_ushort(__float2half_rn(ldexpf(xd, ev)));
            n2 = __fadd_rn(n2, __fmul_rn(xd, xd));
        }
        nrm[lane] = ldexpf(1.f, -ev);
        nrm[32 + lane] = sqrtf(n2);
        return;
    }
    for (uint32_t d = 0; d < D; ++d) {
        const float xd = x[(uint64_t)d * xs];
        if (row) row[d] = xd;
        const float s = __fsub_rn(xd, c[d]);
        const __nv_bfloat16 h = __float2bfloat16_rn(s);
        g[(uint64_t)d * 32u + lane] = __bfloat16_as_ushort(h);
        g[(uint64_t)(K + d) * 32u + lane] =
            __bfloat16_as_ushort(__float2bfloat16_rn(__fsub_rn(s, __bfloat162float(h))));
        n2 = __fadd_rn(n2, __fmul_rn(s, s));
    }
    nrm[lane] = n2;
    nrm[32 + lane] = n2 * kVScale;
}

// group base (mirror planes) and norm block of a slot address
__device__ __forceinline__ float* mirror_slot(const MirrorView& M, uint64_t a, uint32_t& lane,
                                              float*& nrm, float*& row) {
    if (a >> 63) {
        const uint64_t gs = a & ~(1ull << 63);
        const uint64_t blk = gs / M.T, slot = gs - blk * M.T;
        lane = (uint32_t)(slot & 31u);
        const uint64_t g = blk * M.gpb + (slot >> 5);
        nrm = M.arena_nrm + g * kNormFloats;
        row = M.arena_rows ? M.arena_rows + (g * 32u + lane) * M.D : nullptr;
        return M.arena_mir + g * M.GF;
    }
    lane = (uint32_t)(a & 31u);
    nrm = M.off_nrm + (a >> 5) * kNormFloats;
    row = M.off_rows ? M.off_rows + (a >> 5 << 5 | lane) * (uint64_t)M.D : nullptr;
    return M.off_mir + (a >> 5) * M.GF;
}

__global__ void mirror_insert_kernel(MirrorView M, uint32_t n, const float* x, const uint32_t* asg,
                                     const int32_t* out_blk, const uint32_t* out_did) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t b = out_blk[i];
    if (b < 0) return;
    const uint32_t slot = out_did[i] % M.T;
    const uint64_t g = (uint64_t)b * M.gpb + (slot >> 5);
    float* row = M.arena_rows ? M.arena_rows + (g * 32u + (slot & 31u)) * M.D : nullptr;
    mirror_column(M.arena_mir + g * M.GF, M.arena_nrm + g * kNormFloats, row, slot & 31u,
                  x + (uint64_t)i * M.D, 1, M.cent + (uint64_t)asg[i] * M.D, M.D, M.K, M.wide);
}

__global__ void mirror_offline_kernel(MirrorView M, uint32_t n, const float* x,
                                      const uint64_t* dest, const uint32_t* asg) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t s = dest[i];
    float* row = M.off_rows ? M.off_rows + s * M.D : nullptr;
    mirror_column(M.off_mir + (s >> 5) * M.GF, M.off_nrm + (s >> 5) * kNormFloats, row,
                  (uint32_t)(s & 31u), x + (uint64_t)i * M.D, 1, M.cent + (uint64_t)asg[i] * M.D,
                  M.D, M.K, M.wide);
}

// warp per group, lane = slot: payload group rows are coalesced
__global__ void mirror_groups_kernel(MirrorView M, const float* payload, int arena, uint64_t PS,
                                     const uint64_t* groups, const uint32_t* cl, uint32_t n) {
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31u;
    if (w >= n) return;
    const uint64_t gi = groups[w];
    const float* src;
    float *dst, *nrm, *rows;
    if (arena) {
        const uint64_t blk = gi / M.gpb, j = gi - blk * M.gpb;
        src = payload + blk * PS + j * 32ull * M.D;
        dst = M.arena_mir + gi * M.GF;
        nrm = M.arena_nrm + gi * kNormFloats;
        rows = M.arena_rows;
    } else {
        src = payload + gi * 32ull * M.D;
        dst = M.off_mir + gi * M.GF;
        nrm = M.off_nrm + gi * kNormFloats;
        rows = M.off_rows;
    }
    float* row = rows ? rows + (gi * 32u + lane) * M.D : nullptr;
    mirror_column(dst, nrm, row, lane, src + lane, 32, M.cent + (uint64_t)cl[w] * M.D, M.D, M.K, M.wide);
}

__global__ void mirror_slot_move_kernel(MirrorView M, const uint64_t* id_addr, uint32_t n,
                                        float* scr, int phase) {
    // per slot: 2K plane rows (K in wide mode) + 2 norm entries + D row entries
    const uint32_t PR = M.wide ? M.K : 2 * M.K;
    const uint32_t R = PR + 2 + M.D;
    const uint64_t total = (uint64_t)n * R;
    for (uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total;
         o += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t m = (uint32_t)(o / R), r = (uint32_t)(o - (uint64_t)m * R);
        uint32_t lane;
        float *nrm, *row;
        float* g = mirror_slot(M, id_addr[phase == 0 ? m : n + m], lane, nrm, row);
        if (r < PR) {  // bf16 plane element (carried in a float scratch slot)
            uint16_t* e16 = reinterpret_cast<uint16_t*>(g) + (uint64_t)r * 32u + lane;
            if (phase == 0) scr[o] = __uint_as_float(*e16);
            else *e16 = (uint16_t)__float_as_uint(scr[o]);
            continue;
        }
        float* e;
        if (r < PR + 2) e = nrm + (r - PR) * 32u + lane;
        else if (row) e = row + (r - PR - 2);
        else continue;
        if (phase == 0) scr[o] = *e;
        else *e = scr[o];
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
    const uint64_t total = (uint64_t)n * ((M.wide ? M.K : 2 * M.K) + 2 + M.D);
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((total + 255) / 256, 148 * 16));
    for (int phase = 0; phase < 2; ++phase) {
        mirror_slot_move_kernel<<<g, 256, 0, s>>>(M, id_addr, n, scratch, phase);
        count_launch();
    }
    return cudaGetLastError();
}

}  // namespace bivf
