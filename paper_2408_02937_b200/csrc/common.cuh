// Device-side building blocks shared by every kernel of the online IVF-Flat
// path: exact (reference-bit-identical) distance steps, the warp-wide sorted
// top-k, and the PTX wrappers for mbarriers + bulk async copies (TMA 1D).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace bivf {

constexpr int kGroup = 32;  // interleave group (block_store.hpp:20)

// ---------------------------------------------------------------- distance
// The reference accumulates sum_d (a_d - b_d)^2 in ascending d with one fp32
// accumulator and no FMA (distance.hpp:11-30, compiled without contraction).
// __fsub_rn/__fmul_rn/__fadd_rn are never contracted by nvcc, so each step
// below rounds exactly like the reference's `t = a-b; acc += t*t`.
__device__ __forceinline__ float l2_step(float acc, float q, float x) {
    const float t = __fsub_rn(q, x);
    return __fadd_rn(acc, __fmul_rn(t, t));
}
// Inner product (extension): s += q*x, no FMA.  The
// ranking key is -s, applied once at the end (negation is exact).
__device__ __forceinline__ float ip_step(float acc, float q, float x) {
    return __fadd_rn(acc, __fmul_rn(q, x));
}

enum Metric : int { kL2 = 0, kIP = 1 };

template <int M>
__device__ __forceinline__ float dstep(float acc, float q, float x) {
    if constexpr (M == kL2) return l2_step(acc, q, x);
    else return ip_step(acc, q, x);
}
template <int M>
__device__ __forceinline__ float dfinal(float acc) {
    if constexpr (M == kL2) return acc;
    else return -acc;
}

// (dist, id) lexicographic order: TopK keeps the k smallest, equal distances
// resolve by ascending id (topk.hpp:14-28).
__device__ __forceinline__ bool pair_less(float da, long long ia, float db, long long ib) {
    return da < db || (da == db && ia < ib);
}

// ---------------------------------------------------------------- warp top-k
// A warp holds one sorted list of up to K = 32*KPL (dist,id) entries; entry
// e = r*32 + lane lives in register r of `lane`.  Insert is warp-cooperative
// (ballot for the position, one shuffle-shift), so k=100 needs no per-lane
// heaps.  `thr_d/thr_i` cache entry k-1 (the admission threshold).
template <int KPL>
struct WarpTopK {
    float d[KPL];
    long long id[KPL];
    float thr_d;
    long long thr_i;

    __device__ __forceinline__ void init() {
#pragma unroll
        for (int r = 0; r < KPL; ++r) {
            d[r] = __int_as_float(0x7f800000);  // +inf
            id[r] = -1;
        }
        thr_d = __int_as_float(0x7f800000);
        thr_i = 0x7fffffffffffffffLL;
    }

    // true if (cd, ci) would enter a full list (strictly smaller than entry k-1)
    __device__ __forceinline__ bool admits(float cd, long long ci) const {
        return pair_less(cd, ci, thr_d, thr_i);
    }

    // warp-uniform candidate; all 32 lanes must call.
    __device__ __forceinline__ void insert(float cd, long long ci, int k, int lane) {
        int pos = 0;
#pragma unroll
        for (int r = 0; r < KPL; ++r) {
            const int e = r * 32 + lane;
            const bool lt = (e < k) && pair_less(d[r], id[r], cd, ci);
            pos += __popc(__ballot_sync(0xffffffffu, lt));
        }
        if (pos >= k) return;
        // shift entries >= pos up by one (entry e takes e-1), then place.
        float carry_d = 0.f;
        long long carry_i = 0;
#pragma unroll
        for (int r = 0; r < KPL; ++r) {
            const float up_d = __shfl_up_sync(0xffffffffu, d[r], 1);
            const long long up_i = __shfl_up_sync(0xffffffffu, id[r], 1);
            const float top_d = __shfl_sync(0xffffffffu, d[r], 31);
            const long long top_i = __shfl_sync(0xffffffffu, id[r], 31);
            const int e = r * 32 + lane;
            const float prev_d = lane == 0 ? carry_d : up_d;
            const long long prev_i = lane == 0 ? carry_i : up_i;
            if (e == pos) {
                d[r] = cd;
                id[r] = ci;
            } else if (e > pos) {
                d[r] = prev_d;
                id[r] = prev_i;
            }
            carry_d = top_d;
            carry_i = top_i;
        }
        const int rk = (k - 1) >> 5, lk = (k - 1) & 31;
        float td = d[0];
        long long ti = id[0];
#pragma unroll
        for (int r = 1; r < KPL; ++r)
            if (r == rk) {
                td = d[r];
                ti = id[r];
            }
        thr_d = __shfl_sync(0xffffffffu, td, lk);
        thr_i = __shfl_sync(0xffffffffu, ti, lk);
    }
};

// The k smallest VALUES (no ids) across a warp, ascending, lane-strided like
// WarpTopK: enough for a threshold (the k-th smallest value does not depend on
// how ties are ordered), at half WarpTopK's shuffle traffic per insert.
template <int KPL>
struct WarpTopVal {
    float d[KPL];
    float thr;  // the k-th smallest so far (+inf until k were inserted)

    __device__ __forceinline__ void init() {
#pragma unroll
        for (int r = 0; r < KPL; ++r) d[r] = __int_as_float(0x7f800000);
        thr = __int_as_float(0x7f800000);
    }
    __device__ __forceinline__ bool admits(float x) const { return x < thr; }
    // warp-uniform x; all 32 lanes must call
    __device__ __forceinline__ void insert(float x, int k, int lane) {
        int pos = 0;
#pragma unroll
        for (int r = 0; r < KPL; ++r) pos += __popc(__ballot_sync(0xffffffffu, (r * 32 + lane < k) && d[r] <= x));
        if (pos >= k) return;
        float carry = 0.f;
#pragma unroll
        for (int r = 0; r < KPL; ++r) {
            const float up = __shfl_up_sync(0xffffffffu, d[r], 1);
            const float top = __shfl_sync(0xffffffffu, d[r], 31);
            const int e = r * 32 + lane;
            const float prev = lane == 0 ? carry : up;
            if (e == pos)
                d[r] = x;
            else if (e > pos)
                d[r] = prev;
            carry = top;
        }
        const int rk = (k - 1) >> 5;
        float td = d[0];
#pragma unroll
        for (int r = 1; r < KPL; ++r)
            if (r == rk) td = d[r];
        thr = __shfl_sync(0xffffffffu, td, (k - 1) & 31);
    }
};

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1-D bulk async copy global -> shared (TMA engine, SASS UBLKCP), completion
// counted on `bar` in bytes.  dst/src 16-byte aligned, bytes % 16 == 0.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace bivf
