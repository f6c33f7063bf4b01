// Tensor-core filtered list scan (K3 on tcgen05) + exact refine, sm_100a.
//
// Reference semantics (paths under /root/reference/proj): the scan returns
// exactly ClusterIndex::search's top-k (src/ivf_index.cpp:262-298) — ids and
// bit-identical l2_sqr_strided distances (include/blockivf/distance.hpp:22-30)
// under TopK's (dist, id) order (include/blockivf/topk.hpp:14-28).
//
// Design.  Exact distances are sequential fp32 sums, so
// tensor cores can only FILTER: per work item (list c, tile of <=128 queries,
// chunk of groups) a persistent CTA
//   producer warp : TMA (cp.async.bulk.tensor.2d, SWIZZLE_128B) of each
//                   32-vector group, dims as rows -> an MN-major SW128 B tile
//   math warps    : centre the tile in place (x - c_list), per-slot residual
//                   norms, and build A = centred queries (K-major SW128)
//   MMA warp      : tcgen05.mma.kind::tf32 128x32xD into TMEM (4 buffers)
//   math warps    : tcgen05.ld the 32 dot products of their query, form the
//                   approximate distance a = |r|^2 + |s|^2 - 2 r.s and a
//                   PROVEN bound eps (TF32 + fp32 rounding, see err_bound),
//                   keep the k smallest upper bounds (a+eps) and every vector
//                   whose lower bound (a-eps) can still enter the top-k.
// A refine kernel (one warp per query) takes the k-th smallest upper bound
// over all of the query's items as threshold, recomputes the EXACT distance
// (sequential fp32, the reference's bits) of every surviving candidate and
// builds the exact top-k; an item whose candidate buffer overflowed is
// rescanned exactly.  Pruned vectors provably cannot be in the top-k.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "launches.h"
#include "scan.cuh"
#include "scan_common.cuh"
#include "scan_tc.cuh"

namespace bivf {

namespace {

constexpr int kTcThreads = 192;     // warp0 TMA, warp1 MMA, warps 2-5 math
constexpr int kM = 128;             // queries per tile (MMA M, TMEM lanes)
constexpr int kNS = 4;              // smem stages (one group each)
constexpr int kNB = 4;              // TMEM accumulator buffers (32 columns each)
constexpr int kMaxD = 128;
constexpr int kStageBytes = kMaxD * 128;       // 128 rows (dims) x 128 B
constexpr int kABytes = kMaxD * kM * 4;        // 4 K-blocks x 128 rows x 128 B

struct TcParams {
    DevLists L;
    uint32_t D, Dk, Dp, k, P, maxch;
    const float* centroids;      // [C][D] row-major
    const float* queries;        // [nq][Dp]
    const uint32_t* snap_off;
    const uint32_t* snap_len;
    const uint32_t* gc;
    const uint32_t* nch;
    const uint32_t* qoff;
    const uint32_t* item_off;
    const uint32_t* n_items_ptr;
    const uint32_t* plist;
    uint32_t* item_ctr;
    // per (pair, chunk) outputs
    float* ub;          // [runs][k]
    uint32_t* ccount;   // [runs]   (kKC+1 = overflow)
    float* clb;         // [runs][kKC]
    uint32_t* cloc;     // [runs][kKC]   (group << 5 | slot)
};

// ----------------------------------------------------------------- PTX
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void named_bar(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// SW128 smem matrix descriptor (version 1, layout type 2 = SWIZZLE_128B)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;
    d |= 2ull << 61;
    return d;
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Bound on |a - e| where a = approximate (TF32 MMA on centred residuals) and
// e = the reference's sequential fp32 l2_sqr.  With r = q-c, s = x-c rounded to
// fp32 and TF32 operands (<= 2^-10 relative each, truncation), fp32 tensor
// accumulation over K <= 128 terms and fp32 norms:
//   |P - r.s| <= (2^-9 + 2^-16) |r||s|,   |nq - |r|^2| <= 2^-17 |r|^2 (same for s),
//   |e - |q-x|^2| <= (D+2) 2^-24 |q-x|^2,  | |r-s| - |q-x| | <= 2^-23 (|r|+|s|).
// Constants below carry a 2x margin (DESIGN.md §Scan-TC error bound).
__device__ __forceinline__ float err_bound(float nq, float ns, float a) {
    const float rs = sqrtf(nq * ns);
    return 0.0078125f * rs + 6.2e-5f * (nq + ns) + 6.2e-5f * fabsf(a) + 1e-30f;
}

struct TcItem {
    uint32_t c, npairs, g0, g1, chunk, off, len;
    const uint32_t* pairs;
};

__device__ __forceinline__ TcItem tc_decode(const TcParams& p, uint32_t it) {
    uint32_t lo = 0, hi = p.L.C;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (p.item_off[mid] <= it) lo = mid;
        else hi = mid;
    }
    TcItem d;
    d.c = lo;
    const uint32_t local = it - p.item_off[lo];
    const uint32_t nch = p.nch[lo];
    const uint32_t tile = local / nch, h = local - tile * nch;
    const uint32_t q0 = p.qoff[lo] + tile * kM;
    d.pairs = p.plist + q0;
    d.npairs = min((uint32_t)kM, p.qoff[lo + 1] - q0);
    d.off = p.snap_off[lo];
    d.len = p.snap_len[lo];
    const uint32_t ng = ivf_ngroups(p.L, d.off, d.len);
    d.g0 = h * p.gc[lo];
    d.g1 = min(ng, d.g0 + p.gc[lo]);
    d.chunk = h;
    return d;
}

// TMA row coordinate of group j (rows of 32 floats = one dim of one group)
__device__ __forceinline__ void group_row(const DevLists& L, uint32_t c, uint32_t off,
                                          uint32_t j, bool& arena, int& row) {
    const uint32_t og = (off + 31u) >> 5;
    if (j < og) {
        arena = false;
        row = (int)((L.off_start[c] / 32u + j) * L.D);
    } else {
        const uint32_t jj = j - og;
        const uint32_t mid = jj / L.gpb, gi = jj - mid * L.gpb;
        const int32_t blk = L.table[(uint64_t)c * L.MLB + mid];
        arena = true;
        row = (int)(((uint64_t)blk * L.gpb + gi) * L.D);
    }
}

template <int KT>
__global__ void __launch_bounds__(kTcThreads, 1)
    scan_tc_kernel(const TcParams p, const __grid_constant__ CUtensorMap map_off,
                   const __grid_constant__ CUtensorMap map_arena) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-align the dynamic smem base (SWIZZLE_128B atoms)
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* sA = smem;                                  // kABytes
    unsigned char* sB = sA + kABytes;                          // kNS * kStageBytes
    float* cent_s = reinterpret_cast<float*>(sB + kNS * kStageBytes);       // kMaxD
    float* npart = cent_s + kMaxD;                             // [kNB][4][32]
    float* nsum = npart + kNB * 4 * 32;                        // [kNB][32]
    float* cand_lb = nsum + kNB * 32;                          // [128][kKC]
    uint32_t* cand_loc = reinterpret_cast<uint32_t*>(cand_lb + kM * kKC);
    uint64_t* bars = reinterpret_cast<uint64_t*>(cand_loc + kM * kKC);
    uint64_t* full = bars;                // kNS
    uint64_t* empty = full + kNS;         // kNS
    uint64_t* cent_full = empty + kNS;    // kNS
    uint64_t* acc_full = cent_full + kNS; // kNB
    uint64_t* acc_empty = acc_full + kNB; // kNB
    uint64_t* a_full = acc_empty + kNB;   // 1
    uint64_t* it_full = a_full + 1;       // 2
    uint64_t* it_empty = it_full + 2;     // 2
    int* ring = reinterpret_cast<int*>(it_empty + 2);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t D = p.D;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kNS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
            mbar_init(&cent_full[s], 1);
        }
        for (int b = 0; b < kNB; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 4);
        }
        mbar_init(a_full, 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&it_full[s], 1);
            mbar_init(&it_empty[s], 5);
        }
        fence_mbar_init();
    }
    // zero the K-padding rows (D..Dk) of A and of every stage once: TMA never writes them
    if (p.Dk != D) {
        for (uint32_t i = threadIdx.x; i < kNS * (p.Dk - D) * 32; i += blockDim.x) {
            const uint32_t s = i / ((p.Dk - D) * 32), r = i % ((p.Dk - D) * 32);
            reinterpret_cast<float*>(sB + s * kStageBytes + D * 128)[r] = 0.f;
        }
    }
    fence_proxy_async();  // the zeroed padding rows are read by the async proxy
    if (warp == 1) {  // TMEM: kNB accumulators x 32 fp32 columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(kNB * 32)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t n_items = *p.n_items_ptr;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            uint32_t unit = 0;
            for (uint32_t seq = 0;; ++seq) {
                const uint32_t rs = seq & 1;
                mbar_wait(&it_empty[rs], ((seq >> 1) & 1) ^ 1);
                const uint32_t it = atomicAdd(p.item_ctr, 1u);
                const int v = it < n_items ? (int)it : -1;
                ring[rs] = v;
                mbar_arrive(&it_full[rs]);
                if (v < 0) break;
                const TcItem d = tc_decode(p, it);
                for (uint32_t j = d.g0; j < d.g1; ++j, ++unit) {
                    const uint32_t st = unit % kNS;
                    mbar_wait(&empty[st], ((unit / kNS) & 1) ^ 1);
                    bool ar;
                    int row;
                    group_row(p.L, d.c, d.off, j, ar, row);
                    mbar_arrive_expect_tx(&full[st], D * 128u);
                    tma_load_2d(sB + st * kStageBytes, ar ? &map_arena : &map_off, 0, row, &full[st]);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) |
                               ((32u >> 3) << 17) | ((uint32_t)(kM >> 4) << 24);
        uint32_t unit = 0, aphase = 0;
        for (uint32_t seq = 0;; ++seq) {
            const uint32_t rs = seq & 1;
            mbar_wait(&it_full[rs], (seq >> 1) & 1);
            const int v = ring[rs];
            __syncwarp();
            if (lane == 0) mbar_arrive(&it_empty[rs]);
            if (v < 0) break;
            const TcItem d = tc_decode(p, (uint32_t)v);
            if (d.g1 <= d.g0) continue;
            mbar_wait(a_full, aphase & 1);
            ++aphase;
            for (uint32_t j = d.g0; j < d.g1; ++j, ++unit) {
                const uint32_t st = unit % kNS, b = unit % kNB;
                mbar_wait(&cent_full[st], (unit / kNS) & 1);
                mbar_wait(&acc_empty[b], ((unit / kNB) & 1) ^ 1);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB + st * kStageBytes);
                    for (uint32_t ks = 0; ks < p.Dk / 8; ++ks) {
                        const uint32_t kb = ks >> 2, kin = ks & 3;
                        const uint64_t ad = sw128_desc(a0 + kb * (kM * 128) + kin * 32, 16, 1024);
                        const uint64_t bd = sw128_desc(b0 + ks * 1024, 4096, 1024);
                        mma_tf32(tmem_base + b * 32, ad, bd, idesc, ks > 0 ? 1u : 0u);
                    }
                    mma_commit(&acc_full[b]);
                    mma_commit(&empty[st]);
                }
                __syncwarp();
            }
        }
    } else {
        // ------------------------------------------------ math warps (128 threads)
        const int mt = threadIdx.x - 64;             // 0..127
        const int m = 32 * (warp & 3) + lane;        // TMEM lane / query row of the tile
        const uint32_t taddr_lane = (uint32_t)(32 * (warp & 3)) << 16;
        float* my_lb = cand_lb + m * kKC;
        uint32_t* my_loc = cand_loc + m * kKC;
        uint32_t unit = 0;
        for (uint32_t seq = 0;; ++seq) {
            const uint32_t rs = seq & 1;
            mbar_wait(&it_full[rs], (seq >> 1) & 1);
            const int v = ring[rs];
            __syncwarp();
            if (lane == 0) mbar_arrive(&it_empty[rs]);
            if (v < 0) break;
            const TcItem d = tc_decode(p, (uint32_t)v);
            // centroid of the list
            for (uint32_t i = mt; i < D; i += 128) cent_s[i] = p.centroids[(uint64_t)d.c * D + i];
            named_bar(1, 128);
            // A = centred queries, K-major SW128: row m, K-block kb at kb*16KB + m*128,
            // 16-byte chunk (k%32)/4 swizzled by m%8.
            const bool active = (uint32_t)m < d.npairs;
            uint32_t pair = 0;
            float nq = 0.f;
            if (active) {
                pair = d.pairs[m];
                const float* q = p.queries + (uint64_t)(pair / p.P) * p.Dp;
                for (uint32_t k0 = 0; k0 < p.Dk; k0 += 4) {
                    float4 r;
                    r.x = k0 + 0 < D ? __fsub_rn(q[k0 + 0], cent_s[k0 + 0]) : 0.f;
                    r.y = k0 + 1 < D ? __fsub_rn(q[k0 + 1], cent_s[k0 + 1]) : 0.f;
                    r.z = k0 + 2 < D ? __fsub_rn(q[k0 + 2], cent_s[k0 + 2]) : 0.f;
                    r.w = k0 + 3 < D ? __fsub_rn(q[k0 + 3], cent_s[k0 + 3]) : 0.f;
                    nq = __fadd_rn(nq, __fmul_rn(r.x, r.x));
                    nq = __fadd_rn(nq, __fmul_rn(r.y, r.y));
                    nq = __fadd_rn(nq, __fmul_rn(r.z, r.z));
                    nq = __fadd_rn(nq, __fmul_rn(r.w, r.w));
                    const uint32_t kb = k0 >> 5, ch = (k0 & 31) >> 2;
                    *reinterpret_cast<float4*>(sA + kb * (kM * 128) + m * 128 +
                                               ((ch ^ (m & 7)) << 4)) = r;
                }
            } else {
                for (uint32_t k0 = 0; k0 < p.Dk; k0 += 4) {
                    const uint32_t kb = k0 >> 5, ch = (k0 & 31) >> 2;
                    *reinterpret_cast<float4*>(sA + kb * (kM * 128) + m * 128 +
                                               ((ch ^ (m & 7)) << 4)) = make_float4(0, 0, 0, 0);
                }
            }
            fence_proxy_async();
            named_bar(1, 128);
            if (mt == 0 && d.g1 > d.g0) mbar_arrive(a_full);

            // per-query running state
            float ubl[KT];
#pragma unroll
            for (int i = 0; i < KT; ++i) ubl[i] = __int_as_float(0x7f800000);
            float ubk = __int_as_float(0x7f800000);
            uint32_t ncand = 0;
            bool overflow = false;

            auto epilogue = [&](uint32_t eunit, uint32_t j) {
                const uint32_t b = eunit % kNB;
                mbar_wait(&acc_full[b], (eunit / kNB) & 1);
                tc_fence_after();
                float dot[32];
                tmem_ld32(tmem_base + taddr_lane + b * 32, dot);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_empty[b]);
                if (!active) return;
                const GroupRef g = ivf_group(p.L, d.c, d.off, d.len, j);
                const float* ns = nsum + b * 32;
                const uint32_t jl = j << 5;
#pragma unroll 4
                for (uint32_t n = 0; n < 32; ++n) {
                    if (n >= g.nvalid) break;
                    const float nx = ns[n];
                    const float a = nq + nx - 2.f * dot[n];
                    const float e = err_bound(nq, nx, a);
                    const float hi = a + e, lo = a - e;
                    if (hi < ubk) {  // keep the KT smallest upper bounds, sorted
                        float x = hi;
#pragma unroll
                        for (int i = 0; i < KT; ++i) {
                            if (i < (int)p.k && x < ubl[i]) {
                                const float t = ubl[i];
                                ubl[i] = x;
                                x = t;
                            }
                        }
                        float kk = ubl[0];
#pragma unroll
                        for (int i = 1; i < KT; ++i)
                            if (i == (int)p.k - 1) kk = ubl[i];
                        ubk = kk;
                    }
                    if (lo <= ubk && !overflow) {
                        if (ncand == kKC) {  // compact against the tighter threshold
                            uint32_t w = 0;
                            for (uint32_t i = 0; i < kKC; ++i)
                                if (my_lb[i] <= ubk) {
                                    my_lb[w] = my_lb[i];
                                    my_loc[w] = my_loc[i];
                                    ++w;
                                }
                            ncand = w;
                        }
                        if (ncand < kKC) {
                            my_lb[ncand] = lo;
                            my_loc[ncand] = jl | n;
                            ++ncand;
                        } else {
                            overflow = true;
                        }
                    }
                }
            };

            uint32_t first_unit = unit;
            for (uint32_t j = d.g0; j < d.g1; ++j, ++unit) {
                const uint32_t st = unit % kNS, b = unit % kNB;
                mbar_wait(&full[st], (unit / kNS) & 1);
                // centre in place: thread -> slot (mt & 31), rows (mt >> 5) + 4i
                {
                    const uint32_t slot = mt & 31, r0 = mt >> 5;
                    unsigned char* base = sB + st * kStageBytes;
                    float part = 0.f;
                    for (uint32_t k = r0; k < D; k += 4) {
                        float* px = reinterpret_cast<float*>(
                            base + k * 128 + ((((slot >> 2) ^ (k & 7))) << 4) + (slot & 3) * 4);
                        const float sv = __fsub_rn(*px, cent_s[k]);
                        *px = sv;
                        part = __fadd_rn(part, __fmul_rn(sv, sv));
                    }
                    npart[(b * 4 + r0) * 32 + slot] = part;
                }
                fence_proxy_async();
                named_bar(1, 128);
                if (mt < 32) {
                    const float* pp = npart + b * 128;
                    nsum[b * 32 + mt] = pp[mt] + pp[32 + mt] + pp[64 + mt] + pp[96 + mt];
                }
                if (mt == 0) mbar_arrive(&cent_full[st]);
                named_bar(1, 128);
                if (j > d.g0) epilogue(unit - 1, j - 1);
            }
            if (d.g1 > d.g0) epilogue(unit - 1, d.g1 - 1);
            (void)first_unit;

            // item output: k upper bounds + surviving candidates
            if (active) {
                const uint64_t run = (uint64_t)pair * p.maxch + d.chunk;
#pragma unroll
                for (int i = 0; i < KT; ++i)
                    if (i < (int)p.k) p.ub[run * p.k + i] = ubl[i];
                uint32_t w = 0;
                if (!overflow) {
                    for (uint32_t i = 0; i < ncand; ++i)
                        if (my_lb[i] <= ubk) {
                            p.clb[run * kKC + w] = my_lb[i];
                            p.cloc[run * kKC + w] = my_loc[i];
                            ++w;
                        }
                }
                p.ccount[run] = overflow ? kKC + 1 : w;
            }
            named_bar(1, 128);
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(kNB * 32)
                     : "memory");
    }
}

// ------------------------------------------------------------------ refine
// One warp per query: threshold = k-th smallest upper bound over all of the
// query's (probe, chunk) runs; exact fp32 distance of every surviving
// candidate; exact top-k.  Overflowed runs are rescanned exactly.
template <int KPL>
__global__ void refine_kernel(TcParams p, const long long* probes, float* out_d, long long* out_i,
                              uint32_t* out_cnt, uint32_t nq) {
    extern __shared__ float qsm[];  // [warps][Dp]
    const uint32_t wq = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t q = blockIdx.x * (blockDim.x >> 5) + wq;
    if (q >= nq) return;
    float* qs = qsm + wq * p.Dp;
    for (uint32_t i = lane; i < p.D; i += 32) qs[i] = p.queries[(uint64_t)q * p.Dp + i];
    __syncwarp();
    // 1. threshold
    WarpTopK<KPL> th;
    th.init();
    for (uint32_t pi = 0; pi < p.P; ++pi) {
        const uint32_t c = (uint32_t)probes[(uint64_t)q * p.P + pi];
        const uint32_t n = p.nch[c];
        for (uint32_t h = 0; h < n; ++h) {
            const uint64_t run = ((uint64_t)q * p.P + pi) * p.maxch + h;
            for (uint32_t e0 = 0; e0 < p.k; e0 += 32) {
                const uint32_t e = e0 + lane;
                const float v = e < p.k ? p.ub[run * p.k + e] : 0.f;
                const long long id = (long long)(run * p.k + e);
                const bool pass = e < p.k && th.admits(v, id);
                unsigned msk = __ballot_sync(0xffffffffu, pass);
                if (!msk) break;
                while (msk) {
                    const int src = __ffs(msk) - 1;
                    msk &= msk - 1;
                    const float bv = __shfl_sync(0xffffffffu, v, src);
                    const long long bi = __shfl_sync(0xffffffffu, id, src);
                    if (th.admits(bv, bi)) th.insert(bv, bi, (int)p.k, lane);
                }
            }
        }
    }
    const float theta = th.thr_d;  // +inf if fewer than k vectors were scanned
    // 2. exact top-k over surviving candidates
    WarpTopK<KPL> tk;
    tk.init();
    auto offer = [&](float dist, long long id, bool valid) {
        const bool pass = valid && tk.admits(dist, id);
        unsigned msk = __ballot_sync(0xffffffffu, pass);
        while (msk) {
            const int src = __ffs(msk) - 1;
            msk &= msk - 1;
            const float bd = __shfl_sync(0xffffffffu, dist, src);
            const long long bi = __shfl_sync(0xffffffffu, id, src);
            if (tk.admits(bd, bi)) tk.insert(bd, bi, (int)p.k, lane);
        }
    };
    for (uint32_t pi = 0; pi < p.P; ++pi) {
        const uint32_t c = (uint32_t)probes[(uint64_t)q * p.P + pi];
        const uint32_t n = p.nch[c];
        const uint32_t off = p.snap_off[c], len = p.snap_len[c];
        for (uint32_t h = 0; h < n; ++h) {
            const uint64_t run = ((uint64_t)q * p.P + pi) * p.maxch + h;
            const uint32_t cnt = p.ccount[run];
            if (cnt <= kKC) {
                for (uint32_t e0 = 0; e0 < cnt; e0 += 32) {
                    const uint32_t e = e0 + lane;
                    bool ok = e < cnt && p.clb[run * kKC + e] <= theta;
                    float dist = 0.f;
                    long long id = -1;
                    if (ok) {
                        const uint32_t loc = p.cloc[run * kKC + e];
                        const GroupRef g = ivf_group(p.L, c, off, len, loc >> 5);
                        const uint32_t sl = loc & 31;
                        const float* x = g.base + sl;
                        float acc = 0.f;
                        for (uint32_t dd = 0; dd < p.D; ++dd) acc = l2_step(acc, qs[dd], x[dd * 32]);
                        dist = acc;
                        id = g.ids[sl];
                    }
                    offer(dist, id, ok);
                }
            } else {  // overflow: exact rescan of the chunk
                const uint32_t ng = ivf_ngroups(p.L, off, len);
                const uint32_t g0 = h * p.gc[c], g1 = min(ng, g0 + p.gc[c]);
                for (uint32_t j = g0; j < g1; ++j) {
                    const GroupRef g = ivf_group(p.L, c, off, len, j);
                    const bool ok = lane < g.nvalid;
                    float acc = 0.f;
                    for (uint32_t dd = 0; dd < p.D; ++dd) acc = l2_step(acc, qs[dd], g.base[dd * 32 + lane]);
                    offer(acc, ok ? g.ids[lane] : -1, ok);
                }
            }
        }
    }
    uint32_t cntq = 0;
#pragma unroll
    for (int r = 0; r < KPL; ++r) {
        const uint32_t e = r * 32 + lane;
        cntq += __popc(__ballot_sync(0xffffffffu, e < p.k && tk.id[r] >= 0));
        if (e < p.k) {
            out_d[(uint64_t)q * p.k + e] = tk.d[r];
            out_i[(uint64_t)q * p.k + e] = tk.id[r];
        }
    }
    if (lane == 0 && out_cnt) out_cnt[q] = cntq;
}

size_t tc_smem_bytes() {
    return 1024 + kABytes + kNS * kStageBytes + kMaxD * 4 + kNB * 4 * 32 * 4 + kNB * 32 * 4 +
           kM * kKC * 8 + 32 * 8 + 64;
}

}  // namespace

// ------------------------------------------------------------------ host side
namespace {
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}
}  // namespace

bool tc_supported(uint32_t D, uint32_t k, int metric) {
    return metric == kL2 && D >= 8 && D <= (uint32_t)kMaxD && k <= 32;
}

cudaError_t make_group_map(const float* base, uint64_t rows, uint32_t D, CUtensorMap* out) {
    auto enc = get_encode();
    if (!enc) return cudaErrorNotSupported;
    cuuint64_t dims[2] = {32, std::max<cuuint64_t>(rows, 1)};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {32, D};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_ivf_search_tc(const DevLists& L, const PlanBufs& B, const long long* probes,
                                 const float* queries, const float* centroids,
                                 const SearchShape& sh, const CUtensorMap& map_off,
                                 const CUtensorMap& map_arena, const TcBufs& T, float* out_d,
                                 long long* out_i, uint32_t* out_cnt, int num_sms,
                                 cudaStream_t s, cudaEvent_t ev0, cudaEvent_t ev1) {
    if (sh.nq == 0) return cudaSuccess;
    SearchShape s2 = sh;
    s2.QT = kM;
    cudaError_t e = launch_plan(L, B, probes, s2, s);
    if (e != cudaSuccess) return e;
    TcParams p{};
    p.L = L;
    p.D = L.D;
    p.Dk = (L.D + 7) & ~7u;
    p.Dp = pad4(L.D);
    p.k = sh.k;
    p.P = sh.P;
    p.maxch = sh.maxch;
    p.centroids = centroids;
    p.queries = queries;
    p.snap_off = B.snap_off;
    p.snap_len = B.snap_len;
    p.gc = B.gc;
    p.nch = B.nch;
    p.qoff = B.qoff;
    p.item_off = B.item_off;
    p.n_items_ptr = B.n_items;
    p.plist = B.plist;
    p.item_ctr = B.item_ctr;
    p.ub = T.ub;
    p.ccount = T.ccount;
    p.clb = T.clb;
    p.cloc = T.cloc;
    const size_t sm = tc_smem_bytes();
    static bool attr = false;
    if (!attr) {
        e = cudaFuncSetAttribute(scan_tc_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sm);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(scan_tc_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sm);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    if (ev0) cudaEventRecord(ev0, s);
    if (sh.k <= 16) scan_tc_kernel<16><<<num_sms, kTcThreads, sm, s>>>(p, map_off, map_arena);
    else scan_tc_kernel<32><<<num_sms, kTcThreads, sm, s>>>(p, map_off, map_arena);
    count_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (ev1) cudaEventRecord(ev1, s);
    const uint32_t wpb = 4;
    refine_kernel<1><<<(sh.nq + wpb - 1) / wpb, wpb * 32, wpb * p.Dp * 4, s>>>(p, probes, out_d,
                                                                              out_i, out_cnt, sh.nq);
    count_launch();
    return cudaGetLastError();
}

}  // namespace bivf
