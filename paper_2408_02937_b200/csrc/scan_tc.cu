// Tensor-core filtered list scan (K3 on tcgen05) + exact refine, sm_100a.
//
// Reference semantics (paths under /root/reference/proj): the scan returns
// exactly ClusterIndex::search's top-k (src/ivf_index.cpp:262-298) — ids and
// bit-identical l2_sqr_strided distances (include/blockivf/distance.hpp:22-30)
// under TopK's (dist, id) order (include/blockivf/topk.hpp:14-28).
//
// Design.  Exact distances are sequential fp32 sums, so
// tensor cores can only FILTER.  Per work item (list c, tile of <=128 queries,
// chunk of groups) a persistent CTA (one per SM) runs
//   producer warp : one TMA box per 32-vector group from the scan mirror
//                   (mirror.cuh: list-centred residual s = x - c pre-split into
//                   bf16 hi/lo planes + |s|^2) -> MN-major B tiles (SWIZZLE_64B)
//   MMA warp      : 3xBF16 tcgen05.mma kind::f16 128x64x16 per K-step (A =
//                   centred queries, bf16 hi/lo pairs in TMEM; B hi/lo from smem)
//                   into one of 4 TMEM accumulators (fp32)
//   2 math warpgroups (alternate groups): build A once per item, then per
//                   group tcgen05.ld the 32 dot products of their query, form
//                   a = |r|^2 + |s|^2 - 2 r.s and a PROVEN bound eps (bf16 split +
//                   fp32 rounding, mirror.cuh), keep the k smallest upper
//                   bounds (a+eps) and every vector whose lower bound (a-eps)
//                   can still enter the top-k (one run per warpgroup).
// A refine kernel (one warp per query) takes the k-th smallest upper bound
// over all of the query's runs as threshold, recomputes the EXACT distance
// (sequential fp32 over the reference-layout payload, the reference's bits) of
// every surviving candidate and builds the exact top-k; a chunk whose candidate
// buffer overflowed is rescanned exactly.  Pruned vectors provably cannot be in
// the top-k.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "maint.cuh"
#include "mirror.cuh"
#include "launches.h"
#include "scan.cuh"
#include "scan_common.cuh"
#include "scan_tc.cuh"

namespace bivf {

namespace {

constexpr int kWG = 2;                     // math warpgroups
constexpr int kTcThreads = 64 + 128 * kWG;  // warp0 TMA, warp1 MMA, warps 2.. math
constexpr int kM = 128;                    // queries per tile (MMA M, TMEM lanes)
constexpr int kGU = 2;                     // groups per unit (MMA N = 32 * kGU)
// smem stages (one group each; kNS / kGU unit slots) and smem candidate slots
// per thread, by top-k width: k <= 16 -> 6 stages, 40 slots; k <= 32 -> 4, 56.
// Wide mode stages hold one 128-row fp16 chunk (8 KB instead of 16 KB); the
// smem freed goes to 10 stages (k <= 16) and candidate slots (48 / 72: the looser
// inner-product bound keeps more candidates).  An overflowed run is rescanned
// exactly by the refine.
#ifndef BIVF_TC_NS16
#define BIVF_TC_NS16 6
#endif
#ifndef BIVF_TC_KC16
#define BIVF_TC_KC16 40
#endif
#ifndef BIVF_TCW_NS16
#define BIVF_TCW_NS16 10  // wide mode: deeper B prefetch (cfg5 scan 14.9 -> 13.0 ms)
#endif
#ifndef BIVF_TCW_KC16
#define BIVF_TCW_KC16 48  // (32 slots overflow: rescans)
#endif
template <int KT, bool W = false>
struct TcCfg {
    static constexpr int NS = W ? (KT <= 16 ? BIVF_TCW_NS16 : 4) : (KT <= 16 ? BIVF_TC_NS16 : 4);
    static constexpr int KC = W ? (KT <= 16 ? BIVF_TCW_KC16 : 72) : (KT <= 16 ? BIVF_TC_KC16 : 56);
    static constexpr int NU = NS / 2;
    static constexpr int STAGE = W ? 128 * 64 : 2 * 128 * 64;  // bytes per stage
};
// Measured and dropped: releasing a unit's accumulator before filtering (no gain,
// more registers), both warpgroups on every unit (twice the per-unit fixed cost).
constexpr int kNB = 4;                     // TMEM accumulators (32 * kGU columns each; even)
constexpr uint32_t kUnitArrivals = 4;      // warps releasing a unit's accumulator (its warpgroup)
// Wide mode W (inner product, D <= 768): 1xFP16 over 2^e-scaled operands (mirror.cuh),
// queries uncentred, the B mirror streamed in 128-row K-chunks, A = the query rows'
// fp16 plane (<= 384 TMEM columns, one buffer), 2 accumulators.  Otherwise 3xBF16 L2 (D <= 128): two A
// buffers (hi + lo, 128 columns each), 4 accumulators.
template <bool W>
struct TcMode {
    static constexpr int NB = W ? 2 : 4;
    static constexpr uint32_t ColAcc = W ? 384 : 256;
};
constexpr int kRing = 4;                   // decoded work items in flight (producer lookahead)
constexpr int kNR = 8;                     // norm slots (ring, one unit each; decoupled from kNB)

// Per-role cycle accounting of the scan kernel (build with -DBIVF_TC_PROF=1; CTA 0
// prints its producer / MMA / math-warp counters).  A no-op otherwise.
#ifndef BIVF_TC_PROF
#define BIVF_TC_PROF 0
#endif
struct TcProf {
#if BIVF_TC_PROF
    uint32_t t0 = 0, t00 = 0, acc[12] = {};
    __device__ __forceinline__ void start() { t00 = t0 = (uint32_t)clock(); }
    __device__ __forceinline__ void mark(int i) {
        const uint32_t n = (uint32_t)clock();
        acc[i] += n - t0;
        t0 = n;
    }
    __device__ void report(const char* role, int warp) {
        acc[11] = (uint32_t)clock() - t00;
        if (blockIdx.x == 0 && (threadIdx.x & 31) == 0)
            printf("[tc-prof] %s w%d: %u %u %u %u %u %u %u %u %u %u %u total %u\n", role, warp, acc[0],
                   acc[1], acc[2], acc[3], acc[4], acc[5], acc[6], acc[7], acc[8], acc[9], acc[10],
                   acc[11]);
    }
#else
    __device__ __forceinline__ void start() {}
    __device__ __forceinline__ void mark(int) {}
    __device__ __forceinline__ void report(const char*, int) {}
#endif
};
constexpr int kMaxD = 128;
// a stage = one group's mirror planes: 2K rows of 64 bytes (32 bf16: [s_hi], [s_lo]);
// wide mode: one 128-row K-chunk of the fp16 plane (TcCfg::STAGE)
// TMEM columns (a column holds two bf16 of a row): two A buffers (items alternate,
// so the next item's A is written while the MMAs of the current one run), each
// A_hi [0,64) + A_lo [64,128); accumulators [256, 256 + 64*kNB)
constexpr uint32_t kColAlo = 64, kColA2 = 128, kColAcc = 256, kTmemCols = 512;
static_assert(kColAcc + 32 * kGU * kNB <= kTmemCols, "TMEM budget");

struct TcParams {
    DevLists L;
    uint32_t D, Dk, Dp, k, P, maxch;
    uint32_t brow, gstride, nkc;  // TMA box rows, map rows per group, K-chunks per group (wide: Dk / brow)
    uint32_t seed_groups;        // seeding pass: scan only the first seed_groups groups, no run output
    uint32_t qt;                 // plan tile: pairs per work item (kM, or kVmQ for scan_vm_kernel;
                                 // kVmQ also marks runs whose upper bounds only warpgroup 0 writes)
    const float* samp_rows;      // seed samples (maint.cuh kSampS per list, [list][d][slot]) or null
    const long long* samp_ids;   // their ids (-1: empty / deleted)
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
    float* qthr;                // [nq] per-query threshold shared by all its runs (f2ord bits, atomicMin)
    // dense mode (the coarse quantizer): approximate distances a = |r|^2 + |s|^2 - 2 r.s of
    // every (query, slot of the single list) -> dense_out[query * dense_ld + slot], |r|^2 ->
    // dense_nq[query]; no filtering (dense_select_kernel does the selection)
    float* dense_out;
    float* dense_nq;
    uint32_t dense_ld;
    // IVF dense mode (k > 32): list c's tiles start at dense_list_base[c]; tile t of a
    // list with ng groups holds [ng][128 tile rows][32 slots] (a row's group is one 128 B line)
    const uint64_t* dense_list_base;
    const uint32_t* dense_ppos;      // the plan's per-pair position in its list
    float2* dense_gsum;              // IVF dense mode: per (pair, group) (min upper, min lower bound)
    const float* off_rows;      // mirror rows (mirror.cuh): slot-major exact payload copy
    const float* arena_rows;
    const float* off_nrm;       // mirror norms (mirror.cuh), 64 floats per group
    const float* arena_nrm;
    // per run outputs; run = ((pair * maxch + chunk) << 1) | warpgroup
    float* ub;          // [runs][k]
    uint32_t* ccount;   // [runs]   (kOverflow = overflow)
    float* clb;         // [runs][kKC]
    uint32_t* cloc;     // [runs][kKC]   (group << 5 | slot)
};

// the vector-major scan's tensor maps: [offline, arena][one group's hi plane,
// four groups' hi planes, four groups' norm rows] (make_vm_maps)
struct VmMaps {
    CUtensorMap m[2][3];
};

// order-preserving float -> uint32 (negative values included)
__device__ __forceinline__ uint32_t f2ord(float x) {
    const uint32_t b = __float_as_uint(x);
    return b ^ ((b >> 31) ? 0xffffffffu : 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t u) {
    return __uint_as_float(u ^ ((u >> 31) ? 0x80000000u : 0xffffffffu));
}

// The shared per-query thresholds (TcParams::qthr) hold f2ord-encoded keys so
// atomicMin orders negative (inner-product) keys too; 0xffffffff (the memset
// pattern) is "no threshold yet".
__device__ __forceinline__ float qthr_dec(uint32_t u) {
    return u == 0xffffffffu ? __int_as_float(0x7f800000) : ord2f(u);
}

// ----------------------------------------------------------------- PTX
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
// L2 prefetch of a 2-D tensor-map box (no shared memory, no completion)
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void named_bar(int id, int n) {
    asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(n) : "memory");  // non-.aligned: tolerates divergence
}
// UMMA smem matrix descriptor (version 1).  layout 4 = SWIZZLE_64B, MN-major
// 16-bit B: atoms of 32 slots (64 B) x 8 K-rows = 512 B (SBO = 512 between K
// atoms, LBO = the stride to the next 32 slots = the next stage), which is what
// TMA CU_TENSOR_MAP_SWIZZLE_64B writes for a {32, 2K} bf16 box.  Verified on
// B200 by tools/tc_probe_bf16.cu (exact small-integer products, N = 64 across
// two stages, A bf16 pairs in TMEM).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;
    d |= (uint64_t)layout << 61;
    return d;
}
#define BIVF_TMEM_ST32(addr, v)                                                                  \
    asm volatile(                                                                                \
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12," \
        "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::     \
            "r"(addr),                                                                           \
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),  \
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),        \
        "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),      \
        "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),      \
        "r"(v[29]), "r"(v[30]), "r"(v[31])                                                       \
        : "memory")
// bf16 RN split of a pair of fp32 values into (hi pair, lo pair), each packed
// low half = first element (the K order of A in TMEM, tools/tc_probe_bf16.cu)
__device__ __forceinline__ void bf16_split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);  // one packed convert (low = x0)
    const float2 hf = __bfloat1622float2(h);
    const __nv_bfloat162 l = __floats2bfloat162_rn(__fsub_rn(x0, hf.x), __fsub_rn(x1, hf.y));
    hi = *reinterpret_cast<const uint32_t*>(&h);
    lo = *reinterpret_cast<const uint32_t*>(&l);
}
// Warp-collective issue of one 3xBF16 K-step (A_hi*B_hi, A_hi*B_lo, A_lo*B_hi):
// the whole (converged) warp executes it, elect.sync picks the issuing lane
// inside the asm, so no per-MMA elect loop is generated around it.
__device__ __forceinline__ void mma3_bf16_elect(uint32_t dcol, uint32_t ah, uint32_t al, uint64_t bh,
                                                uint64_t bl, uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred e, p, t;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "setp.eq.b32 t, 0, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %3, %5, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %4, %5, t;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %3, %5, t;\n\t}" ::"r"(dcol),
        "r"(ah), "r"(al), "l"(bh), "l"(bl), "r"(idesc), "r"(accum)
        : "memory");
}
// one 1xBF16 K-step (wide mode: A_hi * B_hi)
__device__ __forceinline__ void mma1_bf16_elect(uint32_t dcol, uint32_t ah, uint64_t bh, uint32_t idesc,
                                                uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %3, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %4, p;\n\t}" ::"r"(dcol),
        "r"(ah), "l"(bh), "r"(accum), "r"(idesc)
        : "memory");
}
__device__ __forceinline__ void mma_commit_elect(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
            smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    // the load and its wait in ONE asm statement: the destination registers are
    // undefined until tcgen05.wait::ld, and with two statements the compiler may
    // schedule their consumers between the two
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr)
        : "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Bound on |a - e| where a = nq + ns - 2P is the tensor-core approximation and e
// the reference's sequential fp32 l2_sqr (DESIGN.md §Scan-TC error bound).
// r = fl(q-c), s = fl(x-c); 3xBF16: r = r0 + r1 + rho with r0 = bf16_rn(r),
// r1 = bf16_rn(r - r0) (r - r0 exact), |r1| <= 2^-8|r|, |rho| <= 2^-16|r| (same for s);
// bf16 products are exact in fp32, and P = r0.s0 + r0.s1 + r1.s0 drops r1.s1, rho.s
// and r.sigma: <= 3.01*2^-16 sum|r_d s_d|; fp32 accumulation of 3*K/16 MMA steps adds
// <= 24*2^-24 sum|r_d s_d| (K=128): |P - r.s| <= 2^-14.3 |r||s| (measured worst
// 2^-19.0 on B200, tools/tc_probe_bf16.cu).  Norms: sequential fp32,
// |nq - |r|^2| <= (D+1) 2^-24 |r|^2; exact value: |e - |q-x|^2| <= (D+2) 2^-24 |q-x|^2;
// centring: | |r-s|^2 - |q-x|^2 | <= 2^-22 (|r|^2 + |s|^2).  Constants (mirror.cuh)
// carry >= 2x margin; |r||s| is bounded by (|r|^2+|s|^2)/2 so every term is a
// function of (nq + ns) and |a|:  eps' = kEpsT*(nq+ns) + kEpsRel*|a| + 1e-30.
struct TcItem {
    uint32_t c, npairs, g0, g1, chunk, off, len, valid;
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
    d.valid = 1;
    d.c = lo;
    const uint32_t local = it - p.item_off[lo];
    const uint32_t nch = p.nch[lo];
    const uint32_t tile = local / nch, h = local - tile * nch;
    const uint32_t q0 = p.qoff[lo] + tile * p.qt;
    d.pairs = p.plist + q0;
    d.npairs = min(p.qt, p.qoff[lo + 1] - q0);
    d.off = p.snap_off[lo];
    d.len = p.snap_len[lo];
    const uint32_t ng = ivf_ngroups(p.L, d.off, d.len);
    d.g0 = h * p.gc[lo];
    d.g1 = min(ng, d.g0 + p.gc[lo]);
    if (p.seed_groups) d.g1 = min(d.g1, d.g0 + p.seed_groups);
    d.chunk = h;
    return d;
}

// bounds + filtering of one group for this thread's query (see tc_unit)
template <int KT, bool W>
__device__ __forceinline__ void tc_filter(const TcParams& p, const TcItem& d, uint32_t j,
                                          const float* wn, bool active, float nq, float sq,
                                          const float (&dot)[32], float (&ubl)[KT], float& ubk,
                                          uint32_t& ncand, bool& overflow, float* clb,
                                          uint32_t* cloc, float* scr, TcProf& pf) {
    if (!active) return;
    // W (inner product): key a = -q.x, the MMA value P' = 2^(eq+ev_n) q.x (+ error
    // <= kEpsIP |q||x| unscaled); `nq` holds kEpsIP |q| 2^eq, `sq` 2^eq, wn[n] 2^-ev_n,
    // wn[32 + n] |x_n|.  Scaled by 2^eq: slot n can enter iff
    // P'_n 2^-ev_n + nq |x_n| >= -ubk 2^eq.
    const float Wt = W ? -ubk * sq : 0.f;
    // pass 1 (L2): slot n can still enter the top-k only if its lower bound a - eps' <= ubk,
    // i.e. dot >= V[n] + W (V = kVScale*ns from the mirror norms; a < 0 passes too,
    // since ubk > 0).  Most groups have no such slot: test max_n (dot - V) >= W first
    // (an FADD per slot, 3-input max, two independent chains), build the mask only
    // when the group has a survivor.
    const float Wl = W ? 0.f : fmaf(kVScale, nq, -ubk * (0.5f / (1.0f - kEpsRel)));
    {
        float m0 = -__int_as_float(0x7f800000), m1 = m0;
#pragma unroll
        for (uint32_t n = 0; n < 32; n += 4) {
            const float4 v = reinterpret_cast<const float4*>(wn + 32)[n / 4];
            if constexpr (W) {
                const float4 s4 = reinterpret_cast<const float4*>(wn)[n / 4];
                m0 = fmaxf(m0, fmaxf(fmaf(dot[n], s4.x, nq * v.x), fmaf(dot[n + 1], s4.y, nq * v.y)));
                m1 = fmaxf(m1, fmaxf(fmaf(dot[n + 2], s4.z, nq * v.z), fmaf(dot[n + 3], s4.w, nq * v.w)));
            } else {
                m0 = fmaxf(m0, fmaxf(dot[n] - v.x, dot[n + 1] - v.y));  // FMNMX3
                m1 = fmaxf(m1, fmaxf(dot[n + 2] - v.z, dot[n + 3] - v.w));
            }
        }
        if (!(fmaxf(m0, m1) >= (W ? Wt : Wl))) return;
    }

    // valid slots of group j, from the snapshot (no table lookups)
    uint32_t nvalid;
    {
        const uint32_t og = (d.off + 31u) >> 5;
        if (j < og) {
            nvalid = min(32u, d.off - 32u * j);
        } else {
            const uint32_t jj = j - og, mid = jj / p.L.gpb, gi = jj - mid * p.L.gpb;
            nvalid = min(32u, min(p.L.T, d.len - mid * p.L.T) - 32u * gi);
        }
    }
    const uint32_t vmask = nvalid >= 32 ? 0xffffffffu : ((1u << nvalid) - 1u);
    uint32_t need = 0;
#pragma unroll
    for (uint32_t n = 0; n < 32; n += 4) {
        const float4 v = reinterpret_cast<const float4*>(wn + 32)[n / 4];
        if constexpr (W) {
            const float4 s4 = reinterpret_cast<const float4*>(wn)[n / 4];
            need |= (fmaf(dot[n], s4.x, nq * v.x) >= Wt) ? (1u << n) : 0u;
            need |= (fmaf(dot[n + 1], s4.y, nq * v.y) >= Wt) ? (2u << n) : 0u;
            need |= (fmaf(dot[n + 2], s4.z, nq * v.z) >= Wt) ? (4u << n) : 0u;
            need |= (fmaf(dot[n + 3], s4.w, nq * v.w) >= Wt) ? (8u << n) : 0u;
        } else {
            need |= (dot[n] >= v.x + Wl) ? (1u << n) : 0u;
            need |= (dot[n + 1] >= v.y + Wl) ? (2u << n) : 0u;
            need |= (dot[n + 2] >= v.z + Wl) ? (4u << n) : 0u;
            need |= (dot[n + 3] >= v.w + Wl) ? (8u << n) : 0u;
        }
    }
    need &= vmask;
    if (!need) return;
    // pass 2 (a few slots per group): park the dot products in this thread's
    // scratch column and walk the surviving slots in order
#pragma unroll
    for (uint32_t n = 0; n < 32; ++n) scr[n * kM] = dot[n];
    const uint32_t jl = j << 5;
    while (need) {
        const uint32_t n = __ffs(need) - 1;
        need &= need - 1;
        float h, l;
        if constexpr (W) {
            const float isq = 1.0f / sq;  // exact: a power of 2
            const float a = -(scr[n * kM] * wn[n]) * isq;
            const float e = fmaf(nq * isq, wn[32 + n], 1e-30f);
            h = a + e;
            l = a - e;
        } else {
            const float t = nq + wn[n];
            const float a = fmaf(-2.f, scr[n * kM], t);
            const float e = fmaf(kEpsRel, fabsf(a), fmaf(kEpsT, t, 1e-30f));
            h = a + e;
            l = a - e;
        }
        if (h < ubk) {  // keep the k smallest upper bounds, sorted
            // ubl: ascending; entries [0, KT-k) are -inf sentinels, [KT-k, KT) the
            // k smallest upper bounds, so the k-th is always ubl[KT-1] (static
            // register indices only; a min/max bubble drops the largest)
            float x = h;
#pragma unroll
            for (int i = 0; i < KT; ++i) {
                const float lo = fminf(x, ubl[i]);
                x = fmaxf(x, ubl[i]);
                ubl[i] = lo;
            }
            ubk = fminf(ubk, ubl[KT - 1]);  // ubk = min(own k-th UB, the query's shared one)
        }
        if (l <= ubk && !overflow) {
            if (ncand == (uint32_t)TcCfg<KT, W>::KC) {  // compact against the tighter threshold
                uint32_t w = 0;
                for (uint32_t i = 0; i < (uint32_t)TcCfg<KT, W>::KC; ++i) {
                    const float li = clb[i * kM];
                    if (li <= ubk) {
                        const uint32_t ci = cloc[i * kM];
                        clb[w * kM] = li;
                        cloc[w * kM] = ci;
                        ++w;
                    }
                }
                ncand = w;
            }
            if (ncand < (uint32_t)TcCfg<KT, W>::KC) {
                clb[ncand * kM] = l;
                cloc[ncand * kM] = jl | n;
                ++ncand;
            } else {
                overflow = true;
            }
        }
    }
}

// One unit (kGU consecutive groups j0.. of the item, accumulator u % kNB, norm
// slot u % kNR), filtered by the warpgroup (u & 1); accumulator and norm slot
// are released when the filter is done.
template <int KT, bool W>
__device__ __forceinline__ void tc_unit(const TcParams& p, const TcItem& d, uint32_t u, uint32_t j0,
                                        uint64_t* acc_full, uint64_t* acc_empty, uint32_t tmem_base,
                                        uint32_t taddr_lane, int lane, bool active, float nq, float sq,
                                        float (&ubl)[KT], float& ubk, uint32_t& ncand,
                                        bool& overflow, float* clb, uint32_t* cloc,
                                        float* scr, float* nslots, uint64_t* nfull,
                                        uint64_t* nempty, float* qt, uint32_t qshared, uint64_t qrow,
                                        uint32_t m, TcProf& pf) {
    constexpr int NB = TcMode<W>::NB;
    const uint32_t b = u % NB, ns = u % kNR;
    // qshared: the query's shared threshold (the smallest k-th upper bound any of
    // its runs has published, a valid filter bound for every run of the query),
    // loaded by the caller one unit ahead
    const uint32_t ng = min((uint32_t)kGU, d.g1 - j0);
    pf.mark(8);
    mbar_wait(&acc_full[b], (u / NB) & 1);
    __syncwarp();  // tcgen05.ld is .sync.aligned: reconverge after the per-thread spin
    pf.mark(4);
    tc_fence_after();
    const uint32_t acol = tmem_base + taddr_lane + TcMode<W>::ColAcc + b * 32 * kGU;
    float dot[32];
    pf.mark(5);
    mbar_wait(&nfull[ns], (u / kNR) & 1);
    pf.mark(6);
    const float* wslot = nslots + ns * kGU * kNormFloats;
    if (p.dense_out) {  // dense mode: write the approximate keys, no filtering
        // this warp's 32 x 32 staging tile in the (otherwise unused) pass-2 scratch,
        // 16 B chunks XOR-swizzled by row: each thread parks its row, then every
        // store instruction writes four whole 128 B row segments
        float4* sw = reinterpret_cast<float4*>(scr - m + (m & ~31u) * 32u);
        const unsigned act = __ballot_sync(0xffffffffu, active);
        // IVF: this warp's first row of the tile (the tile base from an active row)
        float* wtile = nullptr;
        if (p.dense_list_base && act)
            wtile = p.dense_out +
                    __shfl_sync(0xffffffffu, (unsigned long long)(qrow - m), __ffs(act) - 1) + (m & ~31u) * 32u;
#pragma unroll
        for (int h = 0; h < kGU; ++h) {
            if ((uint32_t)h >= ng) break;
            const float* wn = wslot + h * kNormFloats;
            tmem_ld32(acol + 32 * h, dot);
            float av[32];
            if constexpr (W) {
                // inner product (tc_filter's W key): a = -(P' 2^-ev) 2^-eq, exact scalings
                const float isq = 1.0f / sq;
#pragma unroll
                for (int i = 0; i < 32; ++i) av[i] = -(dot[i] * wn[i]) * isq;
            } else {
#pragma unroll
                for (int i = 0; i < 32; i += 4) {
                    const float4 v = reinterpret_cast<const float4*>(wn)[i / 4];
                    av[i] = fmaf(-2.f, dot[i], nq + v.x);
                    av[i + 1] = fmaf(-2.f, dot[i + 1], nq + v.y);
                    av[i + 2] = fmaf(-2.f, dot[i + 2], nq + v.z);
                    av[i + 3] = fmaf(-2.f, dot[i + 3], nq + v.w);
                }
            }
            if (act) {
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    sw[lane * 8 + (c ^ (lane & 7))] = make_float4(av[4 * c], av[4 * c + 1], av[4 * c + 2], av[4 * c + 3]);
                __syncwarp();
                if (p.dense_list_base) {
                    // IVF: element (j, m, n) at tile + (j * 128 + m) * 32 + n, so the warp's
                    // 32 rows are one contiguous 4 KB run (rows past the tile's pairs
                    // are written too: the tile is allocated whole and never read there)
                    float4* dst = reinterpret_cast<float4*>(wtile + (uint64_t)(j0 + h) * kM * 32u);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int r = i * 4 + (lane >> 3), ch = lane & 7;
                        dst[i * 32 + lane] = sw[r * 8 + (ch ^ (r & 7))];
                    }
                } else {  // quantizer: one contiguous row per query
                    float* rowp = p.dense_out + qrow + 32u * (j0 + h);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int r = i * 4 + (lane >> 3), ch = lane & 7;
                        float4* dst = reinterpret_cast<float4*>(
                            __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(rowp), r));
                        if ((act >> r) & 1u) dst[ch] = sw[r * 8 + (ch ^ (r & 7))];
                    }
                }
                __syncwarp();
            }
            if (active) {
                if (p.dense_gsum) {  // group summary: smallest upper / lower bound of its valid slots
                    const uint32_t j = j0 + h, og = (d.off + 31u) >> 5;
                    uint32_t nvalid;
                    if (j < og) {
                        nvalid = min(32u, d.off - 32u * j);
                    } else {
                        const uint32_t jj = j - og, mid = jj / p.L.gpb, gi = jj - mid * p.L.gpb;
                        nvalid = min(32u, min(p.L.T, d.len - mid * p.L.T) - 32u * gi);
                    }
                    float mh = __int_as_float(0x7f800000), ml = mh;
#pragma unroll
                    for (uint32_t n = 0; n < 32; ++n) {
                        const float e = W ? fmaf(nq * (1.0f / sq), wn[32 + n], 1e-30f)
                                          : fmaf(kEpsRel, fabsf(av[n]), fmaf(kEpsT, nq + wn[n], 1e-30f));
                        if (n < nvalid) {
                            mh = fminf(mh, av[n] + e);
                            ml = fminf(ml, av[n] - e);
                        }
                    }
                    // summaries [tile][row m][group j] (IVF) / [query][group j] (quantizer):
                    // the selection reads a row's groups contiguously
                    const uint32_t ngl = ivf_ngroups(p.L, d.off, d.len);
                    if (p.dense_list_base)
                        p.dense_gsum[(qrow - m) / 32u + (uint64_t)m * ngl + j] = make_float2(mh, ml);
                    else
                        p.dense_gsum[(qrow / p.dense_ld) * ngl + j] = make_float2(mh, ml);
                }
            }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&acc_empty[b]);
            mbar_arrive(&nempty[ns]);
        }
        return;
    }
    ubk = fminf(ubk, qthr_dec(qshared));
    const float ubk0 = ubk;
#pragma unroll
    for (int h = 0; h < kGU; ++h) {
        if ((uint32_t)h >= ng) break;
        pf.mark(7);
        tmem_ld32(acol + 32 * h, dot);
        pf.mark(10);
        tc_filter<KT, W>(p, d, j0 + h, wslot + h * kNormFloats, active, nq, sq, dot, ubl, ubk, ncand,
                         overflow, clb, cloc, scr, pf);
    }
    tc_fence_before();
    __syncwarp();
    pf.mark(7);
    if (lane == 0) {
        mbar_arrive(&acc_empty[b]);
        mbar_arrive(&nempty[ns]);
    }
    // publish an improved threshold
    if (active && ubk < ubk0) atomicMin(reinterpret_cast<uint32_t*>(qt), f2ord(ubk));
}

template <int KT, bool W>
__global__ void __launch_bounds__(kTcThreads, 1)
    scan_tc_kernel(const TcParams p, const __grid_constant__ CUtensorMap map_off,
                   const __grid_constant__ CUtensorMap map_arena) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-align the dynamic smem base (swizzle atoms)
    const uint32_t raw_s = smem_u32(smem_raw);
    const uint32_t pad = ((raw_s + 1023u) & ~1023u) - raw_s;
    constexpr int kNS = TcCfg<KT, W>::NS, kNU = TcCfg<KT, W>::NU, kKCs = TcCfg<KT, W>::KC;
    constexpr int kStage = TcCfg<KT, W>::STAGE;
    unsigned char* sB = smem_raw + pad;                        // kNS * kStage
    float* scratch = reinterpret_cast<float*>(sB + kNS * kStage);  // [kWG][32][kM] pass-2 dots
    float* cand_lb = scratch + kWG * 32 * kM;                        // [kWG][kKCs][kM]
    uint32_t* cand_loc = reinterpret_cast<uint32_t*>(cand_lb + kWG * kKCs * kM);
    float* nslots = reinterpret_cast<float*>(cand_loc + kWG * kKCs * kM);  // [kNR][kGU][64] norms
    uint64_t* bars = reinterpret_cast<uint64_t*>(nslots + kNR * kGU * kNormFloats);
    uint64_t* full = bars;                 // kNU
    uint64_t* empty = full + kNU;          // kNU
    uint64_t* acc_full = empty + kNU;      // kNB
    uint64_t* acc_empty = acc_full + kNB;  // kNB
    uint64_t* a_full = acc_empty + kNB;    // 2 (A buffers)
    uint64_t* a_free = a_full + 2;         // 2
    uint64_t* it_full = a_free + 2;        // kRing
    uint64_t* it_empty = it_full + kRing;  // kRing
    uint64_t* nfull = it_empty + kRing;    // kNR
    uint64_t* nempty = nfull + kNR;        // kNR
    TcItem* ring = reinterpret_cast<TcItem*>(nempty + kNR);  // kRing decoded items
    float* cent_s = reinterpret_cast<float*>(ring + kRing);  // [kWG][kMaxD] the item's centroid
    float* nqx = cent_s + kWG * kMaxD;  // [2][kWG][kM] partial |r|^2, then (wide) [2][kWG][kM] maxima
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(nqx + 4 * kWG * kM);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t D = p.D;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kNU; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);  // MMA commit
        }
        for (int b = 0; b < kNB; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], kUnitArrivals);
        }
        for (int r = 0; r < kNR; ++r) {
            mbar_init(&nfull[r], 1);
            mbar_init(&nempty[r], kUnitArrivals);  // the warps that filtered the unit
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&a_full[a], kWG);
            mbar_init(&a_free[a], 1);
        }
        for (int s = 0; s < kRing; ++s) {
            mbar_init(&it_full[s], 1);
            mbar_init(&it_empty[s], 1 + 4 * kWG);
        }
        fence_mbar_init();
    }
    if (warp == 1) {  // TMEM: 2 A buffers + kNB accumulators
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t n_items = *p.n_items_ptr;
    const uint32_t stages = smem_u32(sB);

    // Work items flow through a ring of kRing DECODED items: the producer claims
    // and decodes item seq + 1 before it issues item seq's loads, so the math
    // warpgroups can build item seq + 1's A operand (into the other TMEM A buffer)
    // before they filter item seq — the MMAs never wait for an A build.
    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            TcProf pf;
            pf.start();
            auto fetch = [&](uint32_t seq) -> bool {
                const uint32_t rs = seq % kRing;
                mbar_wait(&it_empty[rs], ((seq / kRing) & 1) ^ 1);
                const uint32_t it = atomicAdd(p.item_ctr, 1u);
                TcItem d{};
                if (it < n_items) d = tc_decode(p, it);
                ring[rs] = d;
                mbar_arrive(&it_full[rs]);  // release: the item is visible to the consumers
                return d.valid != 0;
            };
            uint32_t unit = 0, step = 0;
            bool have = fetch(0);
            pf.mark(1);
            for (uint32_t seq = 0; have; ++seq) {
                const TcItem d = ring[seq % kRing];
                have = fetch(seq + 1);
                pf.mark(1);
                // hoisted per-item lookups: the offline segment's first group, the
                // list's block-table row (one entry per gpb groups, cached)
                const uint32_t og = (d.off + 31u) >> 5;
                const uint64_t offg0 = og ? p.L.off_start[d.c] / 32u : 0ull;
                const int32_t* trow = p.L.rowptr[d.c];
                uint32_t cmid = 0xffffffffu;
                uint64_t cblk = 0;
                for (uint32_t j0 = d.g0; j0 < d.g1; j0 += kGU, ++unit) {
                    const uint32_t ng = min((uint32_t)kGU, d.g1 - j0);
                    const uint32_t nsl = unit % kNR;
                    uint64_t gidx[kGU];
                    bool gar[kGU];
#pragma unroll
                    for (int h = 0; h < kGU; ++h) {
                        if ((uint32_t)h >= ng) break;
                        const uint32_t j = j0 + h;
                        if (j < og) {
                            gar[h] = false;
                            gidx[h] = offg0 + j;
                        } else {
                            const uint32_t jj = j - og, mid = jj / p.L.gpb, gi = jj - mid * p.L.gpb;
                            if (mid != cmid) {
                                cmid = mid;
                                cblk = (uint64_t)trow[mid];
                            }
                            gar[h] = true;
                            gidx[h] = cblk * p.L.gpb + gi;
                        }
                    }
                    // one stage pair per K-chunk (a single chunk unless wide): box
                    // {32, brow} rows from row gidx * gstride + kc * brow
                    for (uint32_t kc = 0; kc < p.nkc; ++kc, ++step) {
                        const uint32_t us = step % kNU;
                        mbar_wait(&empty[us], ((step / kNU) & 1) ^ 1);
                        pf.mark(2);
                        mbar_arrive_expect_tx(&full[us], ng * p.brow * 64u);
#pragma unroll
                        for (int h = 0; h < kGU; ++h) {
                            if ((uint32_t)h >= ng) break;
                            tma_load_2d(sB + (us * kGU + h) * kStage, gar[h] ? &map_arena : &map_off, 0,
                                        (int)(gidx[h] * p.gstride + kc * p.brow), &full[us]);
                        }
                    }
                    pf.mark(3);
                    // the unit's group norms -> norm slot nsl, once unit - kNR released it
                    mbar_wait(&nempty[nsl], ((unit / kNR) & 1) ^ 1);
                    pf.mark(4);
                    mbar_arrive_expect_tx(&nfull[nsl], ng * kNormFloats * 4u);
                    if (ng == 2 && gar[0] == gar[1] && gidx[1] == gidx[0] + 1) {  // adjacent: one copy
                        bulk_g2s(nslots + nsl * kGU * kNormFloats,
                                 (gar[0] ? p.arena_nrm : p.off_nrm) + gidx[0] * kNormFloats,
                                 2 * kNormFloats * 4u, &nfull[nsl]);
                    } else {
                        for (uint32_t h = 0; h < ng; ++h)
                            bulk_g2s(nslots + (nsl * kGU + h) * kNormFloats,
                                     (gar[h] ? p.arena_nrm : p.off_nrm) + gidx[h] * kNormFloats,
                                     kNormFloats * 4u, &nfull[nsl]);
                    }
                    pf.mark(3);
                }
            }
            pf.report("producer", warp);
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        // N = 32*kGU: the unit's groups sit in consecutive stages, kStage apart (LBO)
        // D fp32, A/B bf16, A K-major (TMEM), B MN-major, N = 32*kGU, M = 128
        // (wide: A/B fp16, format code 0)
        const uint32_t idesc = (1u << 4) | (W ? 0u : (1u << 7) | (1u << 10)) | (1u << 16) |
                               (((32u * kGU) >> 3) << 17) | ((uint32_t)(kM >> 4) << 24);
        uint32_t unit = 0, step = 0;
        TcProf pf;
        pf.start();
        for (uint32_t seq = 0;; ++seq) {
            const uint32_t rs = seq % kRing;
            mbar_wait(&it_full[rs], (seq / kRing) & 1);
            pf.mark(0);
            const TcItem d = ring[rs];
            __syncwarp();
            if (lane == 0) mbar_arrive(&it_empty[rs]);
            if (!d.valid) break;
            const uint32_t ab = W ? 0u : (seq & 1);  // this item's A buffer
            mbar_wait(&a_full[ab], W ? (seq & 1) : ((seq >> 1) & 1));
            pf.mark(2);
            const uint32_t abase = tmem_base + ab * kColA2;
            constexpr int NB = TcMode<W>::NB;
            for (uint32_t j0 = d.g0; j0 < d.g1; j0 += kGU, ++unit) {
                const uint32_t b = unit % NB;
                const uint32_t dcol = tmem_base + TcMode<W>::ColAcc + b * 32 * kGU;
                mbar_wait(&acc_empty[b], ((unit / NB) & 1) ^ 1);
                pf.mark(4);
                for (uint32_t kc = 0; kc < p.nkc; ++kc, ++step) {
                    const uint32_t us = step % kNU;
                    mbar_wait(&full[us], (step / kNU) & 1);
                    pf.mark(3);
                    __syncwarp();
                    tc_fence_after();
                    // a K-step is 16 rows of 64 B: descriptors advance 1024 B (64 in the
                    // >>4 address field), A 8 TMEM columns (16 bf16)
                    const uint32_t bh0 = stages + us * kGU * (uint32_t)kStage;
                    const uint64_t bh = umma_desc(bh0, kStage, 512, 4);
                    if constexpr (W) {
                        // 1xBF16: A_hi * B_hi over this 128-row K-chunk
                        const uint32_t nks = p.brow / 16, a0 = abase + kc * (p.brow / 2);
                        for (uint32_t ks = 0; ks < nks; ++ks)
                            mma1_bf16_elect(dcol, a0 + ks * 8, bh + ks * 64ull, idesc, kc | ks);
                    } else {
                        // 3xBF16: A_hi*B_hi + A_hi*B_lo + A_lo*B_hi (A from TMEM, B from smem)
                        const uint64_t bl = umma_desc(bh0 + p.Dk * 64u, kStage, 512, 4);
                        const uint32_t nks = p.Dk / 16;
                        for (uint32_t ks = 0; ks < nks; ++ks)
                            mma3_bf16_elect(dcol, abase + ks * 8, abase + kColAlo + ks * 8,
                                            bh + ks * 64ull, bl + ks * 64ull, idesc, ks);
                    }
                    mma_commit_elect(&empty[us]);
                    __syncwarp();
                }
                mma_commit_elect(&acc_full[b]);
                __syncwarp();
                pf.mark(5);
            }
            mma_commit_elect(&a_free[ab]);  // the A buffer may be rewritten once these retire
            __syncwarp();
        }
        pf.report("mma", warp);
    } else {
        // ------------------------------------------------ math warpgroups
        const int wg = (warp - 2) >> 2;               // 0: builds A_hi, 1: builds A_lo
        const int q4 = warp & 3;                      // TMEM lane quarter of this warp
        const int m = 32 * q4 + lane;                 // query row of the tile
        const int wt = threadIdx.x - 64 - 128 * wg;   // 0..127 within the warpgroup
        const uint32_t taddr_lane = (uint32_t)(32 * q4) << 16;
        TcProf pf;
        pf.start();
        // read item seq from the ring and write its A operand (centred queries
        // r = q - c of the tile, split r_hi = bf16_rn(r), r_lo = bf16_rn(r - r_hi);
        // lane m = query row, column = a pair of dims) into A buffer seq & 1
        auto build = [&](uint32_t seq, TcItem& d, float& nq, float& sq) -> bool {
            const uint32_t rs = seq % kRing;
            mbar_wait(&it_full[rs], (seq / kRing) & 1);
            d = ring[rs];
            __syncwarp();
            if (lane == 0) mbar_arrive(&it_empty[rs]);
            if (!d.valid) return false;
            pf.mark(0);
            const uint32_t ab = W ? 0u : (seq & 1);
            if (W && seq >= 1) mbar_wait(&a_free[0], (seq - 1) & 1);
            if (!W && seq >= 2) mbar_wait(&a_free[ab], ((seq - 2) >> 1) & 1);
            pf.mark(2);
            const bool active = (uint32_t)m < d.npairs;
            const uint32_t pair = active ? d.pairs[m] : 0u;
            const float* q = p.queries + (uint64_t)(pair / p.P) * p.Dp;
            if constexpr (W) {
                // inner product: A = the query rows (uncentred) scaled by 2^eq (max
                // |q_d| 2^eq in [2^13, 2^14), mirror.cuh) as one fp16 plane; 64-dim
                // chunks alternate between the warpgroups.  Pass 1: max |q_d| and
                // |q|^2 (halves exchanged in smem); pass 2: scale, convert, store.
                float mxh = 0.f, nqh = 0.f;
                for (uint32_t c = wg; 64 * c < p.Dk; c += 2) {
                    float4 qv[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        qv[i] = (active && 64 * c + 4 * i < p.Dp)
                                    ? __ldg(reinterpret_cast<const float4*>(q + 64 * c) + i)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        mxh = fmaxf(mxh, fmaxf(fmaxf(fabsf(qv[i].x), fabsf(qv[i].y)),
                                               fmaxf(fabsf(qv[i].z), fabsf(qv[i].w))));
                        nqh = __fadd_rn(nqh, __fmul_rn(qv[i].x, qv[i].x));
                        nqh = __fadd_rn(nqh, __fmul_rn(qv[i].y, qv[i].y));
                        nqh = __fadd_rn(nqh, __fmul_rn(qv[i].z, qv[i].z));
                        nqh = __fadd_rn(nqh, __fmul_rn(qv[i].w, qv[i].w));
                    }
                }
                float* nqb = nqx + (seq & 1) * kWG * kM;                 // partial |q|^2
                float* mxs = nqx + 2 * kWG * kM + (seq & 1) * kWG * kM;  // partial max |q_d|
                nqb[wg * kM + m] = nqh;
                mxs[wg * kM + m] = mxh;
                named_bar(3, 256);
                const float mx = fmaxf(mxs[m], mxs[kM + m]);
                const int eq = wide_scale_exp(mx);
                sq = ldexpf(1.f, eq);
                nq = kEpsIP * sqrtf(__fadd_rn(nqb[m], nqb[kM + m])) * sq;
                if (p.dense_out && wg == 0 && active && d.chunk == 0)
                    p.dense_nq[pair / p.P] = nq / sq;  // kEpsIP |q| (dense_select's IP bound)
                __syncwarp();
                tc_fence_after();
                for (uint32_t c = wg; 64 * c < p.Dk; c += 2) {
                    float4 qv[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        qv[i] = (active && 64 * c + 4 * i < p.Dp)
                                    ? __ldg(reinterpret_cast<const float4*>(q + 64 * c) + i)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
                    uint32_t vh[32];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        // x 2^eq is exact (a power of 2, scaling toward [2^13, 2^14))
                        const __half2 h0 = __floats2half2_rn(qv[i].x * sq, qv[i].y * sq);
                        const __half2 h1 = __floats2half2_rn(qv[i].z * sq, qv[i].w * sq);
                        vh[2 * i] = *reinterpret_cast<const uint32_t*>(&h0);
                        vh[2 * i + 1] = *reinterpret_cast<const uint32_t*>(&h1);
                    }
                    __syncwarp();
                    BIVF_TMEM_ST32(tmem_base + taddr_lane + 32 * c, vh);
                }
                __syncwarp();
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                tc_fence_before();
                named_bar(3, 256);
                if (wt == 0) mbar_arrive(&a_full[0]);
                pf.mark(3);
                return true;
            }
            // warpgroup g writes dims [64g, 64g + 64) of both planes (A_hi and A_lo):
            // its half of the thread's query row (registers, all loads in flight at
            // once) minus its half of the list centroid (the warpgroup's smem row)
            const int g0 = 64 * wg;
            const bool mine = (uint32_t)g0 < p.Dk;
            float4 qv[16];
#pragma unroll
            for (int i = 0; i < 16; ++i)
                qv[i] = (active && mine && (uint32_t)(g0 + 4 * i) < p.Dp)
                            ? __ldg(reinterpret_cast<const float4*>(q + g0) + i)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
            float* cs = cent_s + wg * kMaxD;
            if (wt < 64) cs[wt] = (uint32_t)(g0 + wt) < D ? __ldg(p.centroids + (uint64_t)d.c * D + g0 + wt) : 0.f;
            named_bar(1 + wg, 128);
            pf.mark(9);
            float nqh = 0.f;  // |r|^2 over this warpgroup's dims
            __syncwarp();
            tc_fence_after();
            if (mine) {
                uint32_t vh[32], vl[32];
#pragma unroll
                for (int i = 0; i < 64; i += 4) {
                    const float4 c4 = *reinterpret_cast<const float4*>(cs + i);
                    const float qa[4] = {qv[i / 4].x, qv[i / 4].y, qv[i / 4].z, qv[i / 4].w};
                    const float ca[4] = {c4.x, c4.y, c4.z, c4.w};
                    float ra[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        // padded dims: q and the centroid row are zero there
                        const float r = __fsub_rn(qa[e], ca[e]);
                        nqh = __fadd_rn(nqh, __fmul_rn(r, r));
                        ra[e] = r;
                    }
                    bf16_split2(ra[0], ra[1], vh[i / 2], vl[i / 2]);
                    bf16_split2(ra[2], ra[3], vh[i / 2 + 1], vl[i / 2 + 1]);
                }
                __syncwarp();
                const uint32_t ta = tmem_base + ab * kColA2 + taddr_lane + (uint32_t)g0 / 2;
                BIVF_TMEM_ST32(ta, vh);
                BIVF_TMEM_ST32(ta + kColAlo, vl);
            }
            // |r|^2 = the two halves' sums, added in a fixed order by both warpgroups
            // (any summation order meets the (D+1) 2^-24 bound of mirror.cuh)
            float* nqb = nqx + (seq & 1) * kWG * kM;  // double-buffered across builds
            nqb[wg * kM + m] = nqh;
            __syncwarp();
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_fence_before();
            named_bar(3, 256);  // both warpgroups: A complete, partial norms visible
            nq = __fadd_rn(nqb[m], nqb[kM + m]);
            if (wt == 0) mbar_arrive(&a_full[ab]);
            if (p.dense_out && wg == 0 && active && d.chunk == 0)
                p.dense_nq[p.dense_list_base ? pair : pair / p.P] = nq;
            pf.mark(3);
            return true;
        };
        uint32_t unit = 0;
        TcItem d;
        float nq = 0.f, sq = 1.f;
        bool have = build(0, d, nq, sq);
        for (uint32_t seq = 0; have; ++seq) {
            TcItem dn;
            float nqn = 0.f, sqn = 1.f;
            bool hn = false;
            // the next item's A while this one's MMAs run (two A buffers); wide mode
            // has one A buffer: it is rewritten after this item's units
            if constexpr (!W) hn = build(seq + 1, dn, nqn, sqn);
            const bool active = (uint32_t)m < d.npairs;
            const uint32_t pair = active ? d.pairs[m] : 0u;
            const uint64_t run = ((((uint64_t)pair * p.maxch + d.chunk) << 1) | (uint32_t)wg);
            float* clb = cand_lb + wg * kKCs * kM + m;      // this thread's candidate column
            uint32_t* cloc = cand_loc + wg * kKCs * kM + m;
            float ubl[KT];
#pragma unroll
            for (int i = 0; i < KT; ++i)
                ubl[i] = i < KT - (int)p.k ? -__int_as_float(0x7f800000) : __int_as_float(0x7f800000);
            float ubk = __int_as_float(0x7f800000);
            uint32_t ncand = 0;
            bool overflow = false;
            uint64_t dbase = 0;  // dense mode: this thread's base element
            if (p.dense_out) {
                if (p.dense_list_base) {
                    const uint32_t tile = (uint32_t)((d.pairs - p.plist) - p.qoff[d.c]) / kM;
                    const uint32_t ngl = ivf_ngroups(p.L, d.off, d.len);
                    dbase = p.dense_list_base[d.c] + (uint64_t)tile * ngl * 32u * kM + m;
                } else {
                    dbase = (uint64_t)(pair / p.P) * p.dense_ld;
                }
            }
            pf.mark(1);
            float* qt = p.qthr + (active ? pair / p.P : 0u);
            // raw f2ord bits, decoded at use: the load stays in flight during a unit
            uint32_t qsh = active ? __ldcg(reinterpret_cast<const uint32_t*>(qt)) : 0xffffffffu;
            for (uint32_t j0 = d.g0; j0 < d.g1; j0 += kGU, ++unit) {
                if ((unit & 1u) != (uint32_t)wg) continue;
                const uint32_t qcur = qsh;
                if (active) qsh = __ldcg(reinterpret_cast<const uint32_t*>(qt));  // in flight during this unit, used by the next
                tc_unit<KT, W>(p, d, unit, j0, acc_full, acc_empty, tmem_base, taddr_lane, lane,
                            active, nq, sq, ubl, ubk, ncand, overflow, clb, cloc,
                            scratch + wg * 32 * kM + m, nslots, nfull, nempty, qt, qcur,
                            dbase, (uint32_t)m, pf);
            }
            pf.mark(8);
            // run output: k upper bounds + surviving candidates (compacted in place)
            if (active && !p.dense_out && !p.seed_groups) {
#pragma unroll
                for (int i = 0; i < KT; ++i)
                    if (i >= KT - (int)p.k) p.ub[run * p.k + (i - (KT - (int)p.k))] = ubl[i];
                uint32_t w = 0;
                if (!overflow) {
                    for (uint32_t i = 0; i < ncand; ++i) {
                        const float li = clb[i * kM];
                        if (li <= ubk) {
                            p.clb[run * kKC + w] = li;
                            p.cloc[run * kKC + w] = cloc[i * kM];
                            ++w;
                        }
                    }
                }
                p.ccount[run] = overflow ? kOverflow : w;
            }
            pf.mark(8);
            if constexpr (W) hn = build(seq + 1, dn, nqn, sqn);
            d = dn;
            nq = nqn;
            sq = sqn;
            have = hn;
        }
        pf.report("math", warp);
    }
    __syncthreads();
    if (warp == 1) {
        __syncwarp();
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(kTmemCols)
                     : "memory");
    }
}

// ------------------------------------------------------------------ vector-major scan
// scan_vm_kernel (L2, D <= 128, k <= 32): the list scan with the roles of the
// MMA operands swapped.  A work item's queries (<= kVmQ centred residuals,
// split into bf16 hi + lo planes) are the B operand (N <= 32 columns, written
// once per item into shared memory); the list's stored vectors are the A
// operand, 128 per MMA (M = a "unit" of four 32-slot groups), streamed from
// the scan mirror's bf16 hi plane only (K rows x 64 B per group: half the bytes
// of the 3xBF16 scan).  Every TMEM lane holds one vector against every query of
// the tile, so a thread filters (vector, query) pairs with no idle rows when a
// list has few queries (north-star: ~29 queries per list).
// Bound (mirror.cuh): s_hi = bf16_rn(s) (unit roundoff 2^-8), |s_d - s_hi_d| <=
// 2^-8 |s_d|; the query r = r_hi + r_lo + rho, |rho_d| <= 2^-16 |r_d|; bf16
// products are exact in fp32: |P - r.s| <= ((1 + 2^-16) 2^-8 + 2^-16) sum|r_d s_d|
// + fp32 accumulation (2K/16 MMA steps, <= 2^-17) <= 2^-7.98 |r||s|, so
// a = nr + ns - 2P is off by <= 2^-6.98 |r||s| from |r-s|^2, plus the norm /
// centring / exact-rounding terms of the 3xBF16 bound (kEpsRel).  kVmCross = 2^-6
// carries a ~2x margin on the cross term.
//   eps = kVmCross |r||s| + kEpsRel (nr + ns) + kEpsRel |a|
// Pass 1 (every pair, superset of lb <= theta; |r||s| <= (nr+ns)/2):
//   P >= U_n + V_s,  U_n = (c1 nr_n - c2 theta_n) / 2,  V_s = c1 ns / 2
// Filtering: each math warp of the unit's warpgroup reads its TMEM lane
// quarter (one 32-vector group x the item's queries) and transposes it through
// a shared-memory tile (XOR-swizzled, conflict-free both ways), so lane n holds
// query n's 32 values; it filters them like the query-major kernel's math
// threads: pass 1 = one FFMA + max per slot against W = (c1 nr - c2 theta) / 2
// (a superset of lb <= theta, |r||s| <= (nr+ns)/2), pass 2 over the few
// surviving slots = the exact bound, the upper bound offered to the query's
// shared k-best set, the candidate (lb, slot) appended to the lane's shared
// column (compacted against theta when full).  The k-best set is per (item,
// query) in shared memory: k slots of f2ord upper bounds, a new value replaces
// the current maximum by compare-and-swap, so its maximum is always the k-th
// smallest upper bound of k distinct vectors seen by ANY of the query's 8 lanes
// (4 warps x 2 warpgroups); theta = min(that maximum, the global per-query
// threshold qthr, which every run of the query tightens).  At the end of an
// item each warpgroup gathers its 4 lanes' candidates of a query into one run
// of refine_kernel's format (warpgroup 0's run carries the k-best set).
constexpr int kVmQ = 32;       // query columns per work item (MMA N <= 32)
#ifndef BIVF_VM_WG
#define BIVF_VM_WG 2  // math warpgroups (units go round-robin; warpgroups >= 1 share run slot 1)
#endif
#ifndef BIVF_VM_NS
#define BIVF_VM_NS 3
#endif
#ifndef BIVF_VM_KC
#define BIVF_VM_KC 24
#endif
constexpr int kVmWG = BIVF_VM_WG;
constexpr int kVmMath = 128 * kVmWG;             // math threads
constexpr int kVmThreads = 64 + kVmMath;         // + producer and MMA warps
constexpr int kVmNS = BIVF_VM_NS;  // A stage slots (one unit of 4 groups each)
#ifndef BIVF_VM_PF
#define BIVF_VM_PF 0
#endif
#ifndef BIVF_VM_SEED_LISTS
#define BIVF_VM_SEED_LISTS 1  // nearest lists whose samples seed a query's threshold (power of 2; 1 measured fastest: 2 -> 1.03 ms, 4 -> 1.04, 8 -> 1.09 vs 1.00)
#endif
constexpr int kVmPF = BIVF_VM_PF;  // units prefetched into L2 ahead of the shared-memory ring
constexpr int kVmNR = 8;       // norm ring slots (a unit's 4 x 32 |s|^2)
#ifndef BIVF_VM_NB
#define BIVF_VM_NB 4  // 8 measured equal (1.004 vs 1.005 ms): the math warps, not buffering, limit
#endif
constexpr int kVmNB = BIVF_VM_NB;  // TMEM accumulators (32 columns each; power of 2)
constexpr int kVmKC = BIVF_VM_KC;  // candidate slots per (warp, query lane)
constexpr uint32_t kVmSlot = 4u * kMaxD * 64u;  // bytes per A slot (4 groups x K rows x 64 B, K <= 128)
constexpr uint32_t kVmPlane = kMaxD * 64u;      // bytes per B plane (K rows x 32 queries bf16)
constexpr float kVmCross = 1.0f / 64.0f;
constexpr float kVmKappa = 0.5f * kVmCross + kEpsRel;
constexpr float kVmC2 = 1.0f / (1.0f - kEpsRel);
constexpr float kVmC1 = 1.0f - kVmKappa * kVmC2 - 1.0f / 262144.0f;  // 2^-18 slack for the test's roundings

// byte offset of element (row k, query column n < 32) of a B plane: MN-major
// SWIZZLE_64B (64-byte rows of 32 bf16, the 16-byte chunk index XOR (k >> 1) & 3),
// the layout TMA writes for the A stages (tools/tc_probe_swap.cu checks both)
__device__ __forceinline__ uint32_t vm_boff(uint32_t k, uint32_t n) {
    return k * 64u + ((((n >> 3) ^ (k >> 1)) & 3u) << 4) + (n & 7u) * 2u;
}

// one K-step of the vector-major MMA: D += A * B_hi + A * B_lo (A, B from smem)
__device__ __forceinline__ void mma_vm_elect(uint32_t dcol, uint64_t ad, uint64_t bh, uint64_t bl,
                                             uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred e, p, t;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %5, 0;\n\t"
        "setp.eq.b32 t, 0, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %4, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %3, %4, t;\n\t}" ::"r"(dcol),
        "l"(ad), "l"(bh), "l"(bl), "r"(idesc), "r"(accum)
        : "memory");
}

// the math warps' 32 x 32 transpose tile: element (vector row s, query column n)
// lives in 16 B chunk (n / 4) ^ (s & 7) of row s -- rows are written as 8 float4
// chunks, columns read as 32 scalars, both without bank conflicts
__device__ __forceinline__ uint32_t vm_tsw(uint32_t s, uint32_t n) {
    return s * 32u + ((((n >> 2) ^ (s & 7u)) << 2) | (n & 3u));
}
__device__ __forceinline__ uint32_t vm_nvalid(const TcParams& p, const TcItem& d, uint32_t j) {
    const uint32_t og = (d.off + 31u) >> 5;
    if (j < og) return min(32u, d.off - 32u * j);
    const uint32_t jj = j - og, mid = jj / p.L.gpb, gi = jj - mid * p.L.gpb;
    return min(32u, min(p.L.T, d.len - mid * p.L.T) - 32u * gi);
}

template <int KT>
__global__ void __launch_bounds__(kVmThreads, 1)
    scan_vm_kernel(const TcParams p, const __grid_constant__ VmMaps maps) {
    const CUtensorMap* map_g1[2] = {&maps.m[0][0], &maps.m[1][0]};  // one group's hi plane
    const CUtensorMap* map_g4[2] = {&maps.m[0][1], &maps.m[1][1]};  // four consecutive groups' hi planes
    const CUtensorMap* map_n4[2] = {&maps.m[0][2], &maps.m[1][2]};  // their |s|^2 rows
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t raw_s = smem_u32(smem_raw);
    const uint32_t pad = ((raw_s + 1023u) & ~1023u) - raw_s;
    unsigned char* sA = smem_raw + pad;                                  // kVmNS * kVmSlot
    unsigned char* sB = sA + kVmNS * kVmSlot;                             // [2 items][hi, lo] planes
    float* tiles = reinterpret_cast<float*>(sB + 4 * kVmPlane);           // [math warps][32][32] transposes
    float* cand_lb = tiles + 4 * kVmWG * 1024;                            // [math warps][kVmKC][32]
    uint32_t* cand_loc = reinterpret_cast<uint32_t*>(cand_lb + 4 * kVmWG * kVmKC * 32);
    float* nslots = reinterpret_cast<float*>(cand_loc + 4 * kVmWG * kVmKC * 32);  // [kVmNR][4 groups][32] |s|^2
    uint32_t* q_thr = reinterpret_cast<uint32_t*>(nslots + kVmNR * 4 * 32);  // [2 items][kVmQ] f2ord theta
    float* q_nr = reinterpret_cast<float*>(q_thr + 2 * kVmQ);             // [2][kVmQ] |r|^2
    float* q_rn = q_nr + 2 * kVmQ;                                        // [2][kVmQ] |r|
    float* cent_s = q_rn + 2 * kVmQ;                                      // [kMaxD] the item's centroid
    float* nrp = cent_s + kMaxD;                                          // [16][kVmQ] partial |r|^2
    uint32_t* q_id = reinterpret_cast<uint32_t*>(nrp + 16 * kVmQ);        // [2][kVmQ] query index
    uint32_t* o_cnt = q_id + 2 * kVmQ;                                    // [2 wg][kVmQ] run fill
    uint32_t* o_ovf = o_cnt + 2 * kVmQ;                                   // [2 wg][kVmQ]
    uint32_t* kbest = o_ovf + 2 * kVmQ;                                   // [2 items][32 slots][kVmQ] f2ord
    uint64_t* bars = reinterpret_cast<uint64_t*>(kbest + 2 * 32 * kVmQ);
    uint64_t* full = bars;                     // kVmNS
    uint64_t* empty = full + kVmNS;            // kVmNS
    uint64_t* acc_full = empty + kVmNS;        // kVmNB
    uint64_t* acc_empty = acc_full + kVmNB;    // kVmNB
    uint64_t* b_full = acc_empty + kVmNB;      // 2
    uint64_t* b_free = b_full + 2;             // 2
    uint64_t* it_full = b_free + 2;            // kRing
    uint64_t* it_empty = it_full + kRing;      // kRing
    uint64_t* nfull = it_empty + kRing;        // kVmNR
    uint64_t* nempty = nfull + kVmNR;          // kVmNR
    TcItem* ring = reinterpret_cast<TcItem*>(nempty + kVmNR);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + kRing);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t K = p.Dk;  // mirror rows per plane (D rounded up to 16)
#if BIVF_TC_PROF
    __shared__ uint32_t prof_ev[8];  // pass-1 survivors, k-best offers, CAS attempts, appends, compactions
    if (threadIdx.x < 8) prof_ev[threadIdx.x] = 0;
#endif
    if (threadIdx.x == 0) {
        for (int s = 0; s < kVmNS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < kVmNB; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 4);  // the 4 warps of the unit's warpgroup
        }
        for (int r = 0; r < kVmNR; ++r) {
            mbar_init(&nfull[r], 1);
            mbar_init(&nempty[r], 4);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&b_full[a], 1);
            mbar_init(&b_free[a], 1);
        }
        for (int s = 0; s < kRing; ++s) {
            mbar_init(&it_full[s], 1);
            mbar_init(&it_empty[s], 1 + 4 * kVmWG);
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(32 * kVmNB)
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
            TcProf pf;
            pf.start();
            auto fetch = [&](uint32_t seq) -> bool {
                const uint32_t rs = seq % kRing;
                mbar_wait(&it_empty[rs], ((seq / kRing) & 1) ^ 1);
                const uint32_t it = atomicAdd(p.item_ctr, 1u);
                TcItem d{};
                if (it < n_items) d = tc_decode(p, it);
                ring[rs] = d;
                mbar_arrive(&it_full[rs]);
                return d.valid != 0;
            };
            uint32_t unit = 0;
            bool have = fetch(0);
            for (uint32_t seq = 0; have; ++seq) {
                const TcItem d = ring[seq % kRing];
                have = fetch(seq + 1);
                const uint32_t og = (d.off + 31u) >> 5;
                const uint64_t offg0 = og ? p.L.off_start[d.c] / 32u : 0ull;
                const int32_t* trow = p.L.rowptr[d.c];
                uint32_t cmid = 0xffffffffu;
                uint64_t cblk = 0;
                // L2 prefetch of the groups kVmPF units ahead (the shared-memory ring
                // holds only kVmNS units; the prefetched loads then hit L2)
                uint32_t pmid = 0xffffffffu;
                uint64_t pblk = 0;
                auto prefetch_unit = [&](uint32_t pj0) {
                    const uint32_t png = min(4u, d.g1 - pj0);
                    for (uint32_t h = 0; h < png; ++h) {
                        const uint32_t j = pj0 + h;
                        uint64_t gi;
                        bool ar;
                        if (j < og) {
                            ar = false;
                            gi = offg0 + j;
                        } else {
                            const uint32_t jj = j - og, mid = jj / p.L.gpb, gq = jj - mid * p.L.gpb;
                            if (mid != pmid) {
                                pmid = mid;
                                pblk = (uint64_t)trow[mid];
                            }
                            ar = true;
                            gi = pblk * p.L.gpb + gq;
                        }
                        if (h == 0 && png == 4 && (j + 3 < og || j >= og) &&
                            (j < og || (j - og) / p.L.gpb == (j + 3 - og) / p.L.gpb)) {
                            // four consecutive groups (one list part, one block): one box each
                            tma_prefetch_3d(map_g4[ar], 0, 0, (int)gi);
                            tma_prefetch_2d(map_n4[ar], 0, (int)gi);
                            break;
                        }
                        tma_prefetch_2d(map_g1[ar], 0, (int)(gi * p.gstride));
                        bulk_prefetch_l2((ar ? p.arena_nrm : p.off_nrm) + gi * kNormFloats, 128u);
                    }
                };
                for (uint32_t u = 0; u < (uint32_t)kVmPF && d.g0 + 4 * u < d.g1; ++u) prefetch_unit(d.g0 + 4 * u);
                for (uint32_t j0 = d.g0; j0 < d.g1; j0 += 4, ++unit) {
                    const uint32_t ng = min(4u, d.g1 - j0);
                    if (kVmPF > 0 && j0 + 4u * kVmPF < d.g1) prefetch_unit(j0 + 4u * kVmPF);
                    uint64_t gidx[4];
                    bool gar[4];
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        if ((uint32_t)h >= ng) break;
                        const uint32_t j = j0 + h;
                        if (j < og) {
                            gar[h] = false;
                            gidx[h] = offg0 + j;
                        } else {
                            const uint32_t jj = j - og, mid = jj / p.L.gpb, gi = jj - mid * p.L.gpb;
                            if (mid != cmid) {
                                cmid = mid;
                                cblk = (uint64_t)trow[mid];
                            }
                            gar[h] = true;
                            gidx[h] = cblk * p.L.gpb + gi;
                        }
                    }
                    // the unit's groups consecutive in one array: one 3-D box of hi planes
                    // and one box of norm rows (groups past the list are loaded and ignored)
                    bool con = true;
#pragma unroll
                    for (int h = 1; h < 4; ++h)
                        if ((uint32_t)h < ng) con = con && gar[h] == gar[0] && gidx[h] == gidx[0] + (uint64_t)h;
                    const uint32_t slot = unit % kVmNS;
                    pf.mark(0);
                    mbar_wait(&empty[slot], ((unit / kVmNS) & 1) ^ 1);
                    pf.mark(1);
                    if (con) {
                        mbar_arrive_expect_tx(&full[slot], 4u * K * 64u);
                        tma_load_3d(sA + slot * kVmSlot, map_g4[gar[0]], 0, 0, (int)gidx[0], &full[slot]);
                    } else {
                        mbar_arrive_expect_tx(&full[slot], ng * K * 64u);
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            if ((uint32_t)h >= ng) break;
                            // the group's hi plane: rows [0, K) of its 2K mirror rows
                            tma_load_2d(sA + slot * kVmSlot + h * K * 64u, map_g1[gar[h]], 0,
                                        (int)(gidx[h] * p.gstride), &full[slot]);
                        }
                    }
                    const uint32_t nsl = unit % kVmNR;
                    pf.mark(2);
                    mbar_wait(&nempty[nsl], ((unit / kVmNR) & 1) ^ 1);
                    pf.mark(3);
                    if (con) {
                        mbar_arrive_expect_tx(&nfull[nsl], 512u);
                        tma_load_2d(nslots + nsl * 4 * 32, map_n4[gar[0]], 0, (int)gidx[0], &nfull[nsl]);
                    } else {
                        mbar_arrive_expect_tx(&nfull[nsl], ng * 128u);
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            if ((uint32_t)h >= ng) break;
                            bulk_g2s(nslots + (nsl * 4 + h) * 32,
                                     (gar[h] ? p.arena_nrm : p.off_nrm) + gidx[h] * kNormFloats, 128u, &nfull[nsl]);
                        }
                    }
                    pf.mark(4);
                }
            }
            pf.report("vm-producer", warp);
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        // D f32, A bf16 MN-major (the stage's 4 groups, LBO = K*64), B bf16 MN-major
        // (the item's query planes), M = 128, N = the item's columns rounded to 16
        const uint32_t idesc0 = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | (8u << 24);
        const uint32_t sa0 = smem_u32(sA), sb0 = smem_u32(sB);
        uint32_t unit = 0;
        TcProf pf;
        pf.start();
        for (uint32_t seq = 0;; ++seq) {
            const uint32_t rs = seq % kRing;
            mbar_wait(&it_full[rs], (seq / kRing) & 1);
            const TcItem d = ring[rs];
            __syncwarp();
            if (lane == 0) mbar_arrive(&it_empty[rs]);
            if (!d.valid) break;
            const uint32_t ib = seq & 1;
            pf.mark(0);
            mbar_wait(&b_full[ib], (seq >> 1) & 1);
            pf.mark(1);
            const uint32_t N = max(16u, (d.npairs + 15u) & ~15u);
            const uint32_t idesc = idesc0 | ((N >> 3) << 17);
            const uint32_t bh0 = sb0 + ib * 2 * kVmPlane, bl0 = bh0 + kVmPlane;
            for (uint32_t j0 = d.g0; j0 < d.g1; j0 += 4, ++unit) {
                const uint32_t b = unit % kVmNB, slot = unit % kVmNS;
                pf.mark(2);
                mbar_wait(&acc_empty[b], ((unit / kVmNB) & 1) ^ 1);
                pf.mark(3);
                mbar_wait(&full[slot], (unit / kVmNS) & 1);
                pf.mark(4);
                __syncwarp();
                tc_fence_after();
                const uint32_t dcol = tmem_base + b * 32u;
                const uint32_t a0 = sa0 + slot * kVmSlot;
                for (uint32_t ks = 0; ks < K / 16; ++ks)
                    mma_vm_elect(dcol, umma_desc(a0 + ks * 1024u, K * 64u, 512, 4),
                                 umma_desc(bh0 + ks * 1024u, kVmPlane, 512, 4),
                                 umma_desc(bl0 + ks * 1024u, kVmPlane, 512, 4), idesc, ks);
                mma_commit_elect(&empty[slot]);
                __syncwarp();
                mma_commit_elect(&acc_full[b]);
                __syncwarp();
            }
            mma_commit_elect(&b_free[ib]);
            __syncwarp();
        }
        pf.report("vm-mma", warp);
    } else {
        // ------------------------------------------------ math warpgroups
        const int wg = (warp - 2) >> 2;
        const uint32_t rs = wg ? 1u : 0u;                 // run slot: warpgroup 0, or the others together
        const int q4 = warp & 3;                          // TMEM lane quarter = group of the unit
        const int wl = (warp - 2) & 3;                    // warp index within the warpgroup (0: filter lanes)
        const int t256 = threadIdx.x - 64;                // 0..255 over both warpgroups
        float* tp = tiles + (warp - 2) * 1024;            // this warp's transpose tile
        float* clb = cand_lb + (warp - 2) * kVmKC * 32 + lane;   // this lane's candidate column
        uint32_t* cloc = cand_loc + (warp - 2) * kVmKC * 32 + lane;
        // item seq's B planes + per-query state (buffer seq & 1), both warpgroups
        auto build = [&](uint32_t seq, TcItem& d) -> bool {
            const uint32_t rs = seq % kRing;
            mbar_wait(&it_full[rs], (seq / kRing) & 1);
            d = ring[rs];
            __syncwarp();
            if (lane == 0) mbar_arrive(&it_empty[rs]);
            // this thread's query values and centroid value: global loads issued
            // before the barrier (they write no shared state)
            // columns n0, n0 + 1 (a bf16 pair: one 4 B store per plane row), dims [8h, 8h + 8)
            const uint32_t n0 = 2u * (t256 & 15), h = t256 >> 4;
            const bool act0 = d.valid && n0 < d.npairs, act1 = d.valid && n0 + 1 < d.npairs;
            float4 qv4[4];  // [query 0: dims 0-3, 4-7][query 1: ...]
            {
                const float* q0 = p.queries + (uint64_t)((act0 ? d.pairs[n0] : 0u) / p.P) * p.Dp;
                const float* q1 = p.queries + (uint64_t)((act1 ? d.pairs[n0 + 1] : 0u) / p.P) * p.Dp;
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const uint32_t k0 = 8 * h + 4 * i;
                    qv4[i] = (act0 && k0 < p.Dp) ? __ldg(reinterpret_cast<const float4*>(q0 + k0))
                                                : make_float4(0.f, 0.f, 0.f, 0.f);
                    qv4[2 + i] = (act1 && k0 < p.Dp) ? __ldg(reinterpret_cast<const float4*>(q1 + k0))
                                                    : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
            const float cv = (d.valid && (uint32_t)t256 < p.D) ? __ldg(p.centroids + (uint64_t)d.c * p.D + t256) : 0.f;
            // both warpgroups are done with item seq - 2's state: taken for the
            // end marker too (no warp may run ahead of another's run output)
            named_bar(3, kVmMath);
            if (t256 < 2 * kVmQ) {  // the run-output gather counters of item seq - 1 (output after this build)
                o_cnt[t256] = 0;
                o_ovf[t256] = 0;
            }
            if (!d.valid) {
                // end marker: the reset above must still be ordered before the last
                // item's run output (every math thread takes this same branch)
                named_bar(3, kVmMath);
                return false;
            }
            const uint32_t ib = seq & 1;
            if (seq >= 2) mbar_wait(&b_free[ib], ((seq - 2) >> 1) & 1);
            if (t256 < (int)K) cent_s[t256] = cv;
            named_bar(3, kVmMath);
            {
                float nh0 = 0.f, nh1 = 0.f;
                if (8 * h < K) {
                    unsigned char* bh = sB + ib * 2 * kVmPlane;
                    unsigned char* bl = bh + kVmPlane;
                    const float qa0[8] = {qv4[0].x, qv4[0].y, qv4[0].z, qv4[0].w, qv4[1].x, qv4[1].y, qv4[1].z, qv4[1].w};
                    const float qa1[8] = {qv4[2].x, qv4[2].y, qv4[2].z, qv4[2].w, qv4[3].x, qv4[3].y, qv4[3].z, qv4[3].w};
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const uint32_t k = 8 * h + e;
                        const float c = cent_s[k];
                        const float r0 = __fsub_rn(qa0[e], act0 ? c : 0.f);
                        const float r1 = __fsub_rn(qa1[e], act1 ? c : 0.f);
                        nh0 = __fadd_rn(nh0, __fmul_rn(r0, r0));
                        nh1 = __fadd_rn(nh1, __fmul_rn(r1, r1));
                        // the same hi / lo split as element-wise bf16_rn (one packed convert each)
                        const __nv_bfloat162 hi = __floats2bfloat162_rn(r0, r1);
                        const __nv_bfloat162 lo = __floats2bfloat162_rn(__fsub_rn(r0, __low2float(hi)),
                                                                        __fsub_rn(r1, __high2float(hi)));
                        *reinterpret_cast<__nv_bfloat162*>(bh + vm_boff(k, n0)) = hi;
                        *reinterpret_cast<__nv_bfloat162*>(bl + vm_boff(k, n0)) = lo;
                    }
                }
                if (h < 16) {
                    nrp[h * kVmQ + n0] = nh0;
                    nrp[h * kVmQ + n0 + 1] = nh1;
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // planes -> the MMA's async proxy
            named_bar(3, kVmMath);
            if (t256 == 0) mbar_arrive(&b_full[ib]);
            if (t256 < kVmQ) {
                const uint32_t n = t256;
                const bool act = n < d.npairs;
                float nr = 0.f;
#pragma unroll
                for (int h = 0; h < 16; ++h) nr = __fadd_rn(nr, nrp[h * kVmQ + n]);  // fixed order
                const uint32_t qi = act ? d.pairs[n] / p.P : 0u;
                q_id[ib * kVmQ + n] = qi;
                q_nr[ib * kVmQ + n] = nr;
                q_rn[ib * kVmQ + n] = sqrtf(nr);
                q_thr[ib * kVmQ + n] = act ? __ldcg(reinterpret_cast<const uint32_t*>(p.qthr) + qi) : 0u;
            }
            if (t256 < 256)
                reinterpret_cast<uint4*>(kbest + ib * 32 * kVmQ)[t256] = make_uint4(~0u, ~0u, ~0u, ~0u);  // 32 x kVmQ slots
            named_bar(3, kVmMath);
            return true;
        };
        uint32_t unit = 0;
        TcItem d;
        TcProf pf;
        pf.start();
        bool have = build(0, d);
        for (uint32_t seq = 0; have; ++seq) {
            TcItem dn;
            pf.mark(0);
            const bool hn = build(seq + 1, dn);
            pf.mark(1);
            const uint32_t ib = seq & 1;
            const int n = lane;                      // this lane's query column
            const bool active = (uint32_t)n < d.npairs;
            const uint32_t qi = q_id[ib * kVmQ + n];
            const float nr = q_nr[ib * kVmQ + n], rn = q_rn[ib * kVmQ + n];
            uint32_t* qts = q_thr + ib * kVmQ + n;   // theta of the query (f2ord, atomicMin)
            uint32_t* kb0 = kbest + ib * 32 * kVmQ;  // k-best sets: query q's slot i at kb0[i * kVmQ + q]
            uint32_t* kb = kb0 + n;                  // this lane's query
            uint32_t ncand = 0;
            bool overflow = false;
            // the global threshold, loaded a unit ahead (its latency stays hidden)
            uint32_t qg = active ? __ldcg(reinterpret_cast<const uint32_t*>(p.qthr) + qi) : 0xffffffffu;
            for (uint32_t j0 = d.g0; j0 < d.g1; j0 += 4, ++unit) {
                if (unit % (uint32_t)kVmWG != (uint32_t)wg) continue;
                const uint32_t b = unit % kVmNB, nsl = unit % kVmNR;
                const uint32_t qcur = qg;
                if (active) qg = __ldcg(reinterpret_cast<const uint32_t*>(p.qthr) + qi);
                pf.mark(2);
                mbar_wait(&acc_full[b], (unit / kVmNB) & 1);
                pf.mark(3);
                __syncwarp();
                tc_fence_after();
                float dot[32];
                tmem_ld32(tmem_base + ((uint32_t)(32 * q4) << 16) + b * 32u, dot);
                // transpose: lane s writes vector s's 32 query values, lane n reads
                // query n's 32 vector values
#pragma unroll
                for (int c = 0; c < 8; ++c)  // 16 B chunks, XOR-swizzled by row (conflict-free)
                    *reinterpret_cast<float4*>(tp + lane * 32 + ((c ^ (lane & 7)) << 2)) =
                        make_float4(dot[4 * c], dot[4 * c + 1], dot[4 * c + 2], dot[4 * c + 3]);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_empty[b]);
#pragma unroll
                for (int s = 0; s < 32; ++s) dot[s] = tp[vm_tsw(s, n)];
                pf.mark(4);
                mbar_wait(&nfull[nsl], (unit / kVmNR) & 1);
                pf.mark(5);
                const float* wn = nslots + (nsl * 4 + q4) * 32;  // |s|^2 of the group's 32 slots
                const uint32_t j = j0 + (uint32_t)q4;
                if (active && j < d.g1) {
                    if (qcur < *reinterpret_cast<volatile uint32_t*>(qts)) atomicMin(qts, qcur);
                    float th = qthr_dec(*reinterpret_cast<volatile uint32_t*>(qts));
                    // pass 1: some slot s can enter iff dot_s - c1 ns_s / 2 >= W
                    const float W = 0.5f * fmaf(kVmC1, nr, -kVmC2 * th);
                    // (the survivor mask directly: one FFMA + compare per slot, the norm
                    // row read once as 8 vector loads)
                    uint32_t need = 0;
#pragma unroll
                    for (int s = 0; s < 32; s += 4) {
                        const float4 v = *reinterpret_cast<const float4*>(wn + s);
                        need |= (fmaf(-0.5f * kVmC1, v.x, dot[s]) >= W) ? (1u << s) : 0u;
                        need |= (fmaf(-0.5f * kVmC1, v.y, dot[s + 1]) >= W) ? (2u << s) : 0u;
                        need |= (fmaf(-0.5f * kVmC1, v.z, dot[s + 2]) >= W) ? (4u << s) : 0u;
                        need |= (fmaf(-0.5f * kVmC1, v.w, dot[s + 3]) >= W) ? (8u << s) : 0u;
                    }
                    pf.mark(6);
                    if (need) {
                        const uint32_t nv = vm_nvalid(p, d, j);
                        need &= nv >= 32 ? 0xffffffffu : ((1u << nv) - 1u);
                        // pass 2 (the tile column still holds this lane's values)
#if BIVF_TC_PROF
                        atomicAdd(&prof_ev[0], (uint32_t)__popc(need));
#endif
                        while (need) {
                            const uint32_t s = __ffs(need) - 1;
                            need &= need - 1;
                            const float ns = wn[s];
                            const float a = fmaf(-2.f, tp[vm_tsw(s, n)], nr + ns);
                            // |s| from the hardware reciprocal square root (rel. error <= 2^-22),
                            // rounded up by 2^-19: e only needs an upper bound
                            const float sn = ns > 0.f ? ns * rsqrtf(ns) * (1.0f + 0x1p-19f) : 0.f;
                            const float e = fmaf(kVmCross, rn * sn,
                                                 fmaf(kEpsRel, nr + ns, fmaf(kEpsRel, fabsf(a), 1e-30f)));
                            const float h = a + e, l = a - e;
                            if (h < th) {
                                // offer h to the query's k-best set: replace its maximum (CAS,
                                // retried when another lane got there first)
                                const uint32_t u = f2ord(h);
#if BIVF_TC_PROF
                                atomicAdd(&prof_ev[1], 1u);
#endif
                                for (;;) {
#if BIVF_TC_PROF
                                    atomicAdd(&prof_ev[2], 1u);
#endif
                                    // all k slots loaded first (independent loads in flight together),
                                    // then the maximum; values only ever decrease, so a stale read
                                    // can only over-estimate the set's maximum (a valid threshold)
                                    uint32_t kv[KT];
#pragma unroll
                                    for (int r = 0; r < KT; ++r)
                                        kv[r] = (uint32_t)r < p.k ? *reinterpret_cast<volatile uint32_t*>(kb + r * kVmQ) : 0u;
                                    uint32_t mx = 0, mi = 0;
#pragma unroll
                                    for (int r = 0; r < KT; ++r)
                                        if (kv[r] >= mx) {
                                            mx = kv[r];
                                            mi = (uint32_t)r;
                                        }
                                    if (u >= mx) break;
                                    if (atomicCAS(kb + mi * kVmQ, mx, u) == mx) {
                                        uint32_t nm = u;
#pragma unroll
                                        for (int r = 0; r < KT; ++r)
                                            if ((uint32_t)r != mi) nm = max(nm, kv[r]);
                                        if (nm < 0xffffffffu) {  // k values: a threshold for the query's runs
                                            atomicMin(qts, nm);
                                            atomicMin(reinterpret_cast<uint32_t*>(p.qthr) + qi, nm);
                                        }
                                        break;
                                    }
                                }
                                th = qthr_dec(*reinterpret_cast<volatile uint32_t*>(qts));
                            }
                            if (l <= th && !overflow) {
#if BIVF_TC_PROF
                                atomicAdd(&prof_ev[3], 1u);
#endif
                                if (ncand == (uint32_t)kVmKC) {  // compact against the tighter threshold
#if BIVF_TC_PROF
                                    atomicAdd(&prof_ev[4], 1u);
#endif
                                    uint32_t w = 0;
                                    for (uint32_t r = 0; r < (uint32_t)kVmKC; ++r) {
                                        const float li = clb[r * 32];
                                        if (li <= th) {
                                            const uint32_t ci = cloc[r * 32];
                                            clb[w * 32] = li;
                                            cloc[w * 32] = ci;
                                            ++w;
                                        }
                                    }
                                    ncand = w;
                                }
                                if (ncand < (uint32_t)kVmKC) {
                                    clb[ncand * 32] = l;
                                    cloc[ncand * 32] = (j << 5) | s;
                                    ++ncand;
                                } else {
                                    overflow = true;
                                }
                            }
                        }
                    }
                }
                pf.mark(9);
                __syncwarp();  // the tile is rewritten by this warp's next unit; norm slot released
                if (lane == 0) mbar_arrive(&nempty[nsl]);
                pf.mark(10);
            }
            pf.mark(7);
            // run output: the warpgroup's 4 lanes of a query -> one run (refine_kernel's
            // format); warpgroup 0's run carries the k-best set, warpgroup 1's +inf.
            // (The gather counters were reset by build(seq + 1) above.)
            if (active) {
                const uint32_t pair = d.pairs[n];
                const uint64_t run = (((uint64_t)pair * p.maxch + d.chunk) << 1) | rs;
                const float th = qthr_dec(*reinterpret_cast<volatile uint32_t*>(qts));
                uint32_t w = 0;
                for (uint32_t i = 0; i < ncand; ++i) w += clb[i * 32] <= th;
                const uint32_t at = overflow ? 0u : atomicAdd(&o_cnt[rs * kVmQ + n], w);
                if (overflow || at + w > kKC) {
                    o_ovf[rs * kVmQ + n] = 1;
                } else {
                    uint32_t o = at;
                    for (uint32_t i = 0; i < ncand; ++i) {
                        const float li = clb[i * 32];
                        if (li <= th) {
                            p.clb[run * kKC + o] = li;
                            p.cloc[run * kKC + o] = cloc[i * 32];
                            ++o;
                        }
                    }
                }
                if (wl == 0 && wg <= 1)  // (run slot 1's +inf values are skipped by the refine)
                    for (uint32_t i = 0; i < p.k; ++i)
                        p.ub[run * p.k + i] =
                            wg == 0 ? qthr_dec(*reinterpret_cast<volatile uint32_t*>(kb0 + i * kVmQ + n))
                                    : __int_as_float(0x7f800000);
            }
            named_bar(1 + rs, rs ? 128 * (kVmWG - 1) : 128);  // the run slot's warpgroups
            if (wl == 0 && wg <= 1 && active) {
                const uint32_t pair = d.pairs[n];
                const uint64_t run = (((uint64_t)pair * p.maxch + d.chunk) << 1) | rs;
                p.ccount[run] = o_ovf[rs * kVmQ + n] ? kOverflow : o_cnt[rs * kVmQ + n];
            }
            pf.mark(8);
            d = dn;
            have = hn;
        }
        pf.report("vm-math", warp);
    }
    __syncthreads();
#if BIVF_TC_PROF
    if (blockIdx.x == 0 && threadIdx.x == 0)
        printf("[tc-prof] vm-events survivors %u offers %u cas %u appends %u compactions %u units %u\n", prof_ev[0],
               prof_ev[1], prof_ev[2], prof_ev[3], prof_ev[4], 0u);
#endif
    if (warp == 1) {
        __syncwarp();
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(32 * kVmNB)
                     : "memory");
    }
}

// ------------------------------------------------------------------ refine
// One warp per query: threshold = k-th smallest upper bound over all of the
// query's (probe, chunk) runs; the surviving candidates (lower bound <=
// threshold) are compacted into a per-warp queue and recomputed EXACTLY
// (sequential fp32, the reference's bits), 32 at a time, loads batched for
// memory-level parallelism; exact top-k.  Overflowed runs are rescanned.
__device__ __forceinline__ float exact_l2(const float* qs, const float* x, uint32_t D) {
    float acc = 0.f;
    uint32_t d0 = 0;
    for (; d0 + 16 <= D; d0 += 16) {
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = x[(d0 + i) * 32];
#pragma unroll
        for (int i = 0; i < 16; ++i) acc = l2_step(acc, qs[d0 + i], v[i]);
    }
    for (; d0 < D; ++d0) acc = l2_step(acc, qs[d0], x[d0 * 32]);
    return acc;
}

// exact distance over a contiguous row (the mirror's slot-major copy): same
// ascending-d sequential fp32 sum, so the same bits as over the interleaved payload
__device__ __forceinline__ float exact_l2_row(const float* qs, const float* x, uint32_t D) {
    float acc = 0.f;
    uint32_t d0 = 0;
    if ((D & 3u) == 0) {
        for (; d0 + 16 <= D; d0 += 16) {
            float4 v[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) v[i] = __ldg(reinterpret_cast<const float4*>(x + d0) + i);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                acc = l2_step(acc, qs[d0 + 4 * i + 0], v[i].x);
                acc = l2_step(acc, qs[d0 + 4 * i + 1], v[i].y);
                acc = l2_step(acc, qs[d0 + 4 * i + 2], v[i].z);
                acc = l2_step(acc, qs[d0 + 4 * i + 3], v[i].w);
            }
        }
    }
    for (; d0 < D; ++d0) acc = l2_step(acc, qs[d0], __ldg(x + d0));
    return acc;
}

// the exact key of either metric: L2 = the sequential l2 sum; IP = -(sequential
// q.x), ip_step (common.cuh), the CUDA-core scan's bits
template <int MET>
__device__ __forceinline__ float exact_key_row(const float* qs, const float* x, uint32_t D) {
    if constexpr (MET == kL2) {
        return exact_l2_row(qs, x, D);
    } else {
        float acc = 0.f;
        uint32_t d0 = 0;
        if ((D & 3u) == 0) {
            for (; d0 + 16 <= D; d0 += 16) {
                float4 v[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) v[i] = __ldg(reinterpret_cast<const float4*>(x + d0) + i);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    acc = ip_step(acc, qs[d0 + 4 * i + 0], v[i].x);
                    acc = ip_step(acc, qs[d0 + 4 * i + 1], v[i].y);
                    acc = ip_step(acc, qs[d0 + 4 * i + 2], v[i].z);
                    acc = ip_step(acc, qs[d0 + 4 * i + 3], v[i].w);
                }
            }
        }
        for (; d0 < D; ++d0) acc = ip_step(acc, qs[d0], __ldg(x + d0));
        return -acc;
    }
}
template <int MET>
__device__ __forceinline__ float exact_key(const float* qs, const float* x, uint32_t D) {
    if constexpr (MET == kL2) {
        return exact_l2(qs, x, D);
    } else {
        // interleaved slot (stride 32 floats): 32 loads in flight per batch, then
        // the sequential chain over them
        float acc = 0.f;
        uint32_t d0 = 0;
        for (; d0 + 32 <= D; d0 += 32) {
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = x[(uint64_t)(d0 + i) * 32];
#pragma unroll
            for (int i = 0; i < 32; ++i) acc = ip_step(acc, qs[d0 + i], v[i]);
        }
        for (; d0 < D; ++d0) acc = ip_step(acc, qs[d0], x[(uint64_t)d0 * 32]);
        return -acc;
    }
}

// row of slot (group j of list c, slot s) in the mirror's row copy
__device__ __forceinline__ const float* cand_row(const TcParams& p, uint32_t c, uint32_t off,
                                                 uint32_t j, uint32_t s) {
    const uint32_t og = (off + 31u) >> 5;
    if (j < og) return p.off_rows + (p.L.off_start[c] + 32ull * j + s) * p.D;
    const uint32_t jj = j - og, mid = jj / p.L.gpb, gi = jj - mid * p.L.gpb;
    const uint64_t g = (uint64_t)p.L.rowptr[c][mid] * p.L.gpb + gi;
    return p.arena_rows + (g * 32u + s) * p.D;
}

// WPQ warps per query (small batches: the latency path has only a few queries,
// one warp each would leave the GPU idle): the warps split the query's runs,
// then merge their thresholds / top-k lists through shared memory.
template <int KPL, int MET, int WPQ>
__global__ void refine_kernel(TcParams p, const long long* probes, float* out_d, long long* out_i,
                              uint32_t* out_cnt, uint32_t nq) {
    extern __shared__ float qsm[];  // [warps][Dp] queries, then [warps][32] x 2 queue, then (WPQ > 1) merge area
    const uint32_t nw = blockDim.x >> 5;
    const uint32_t wq = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t q = blockIdx.x * (nw / WPQ) + wq / WPQ;
    const uint32_t ws = wq % WPQ;  // this warp's share of the query's runs
    if (q >= nq) return;
    float* qs = qsm + wq * p.Dp;
    uint32_t* qc = reinterpret_cast<uint32_t*>(qsm + nw * p.Dp) + wq * 64;  // list
    uint32_t* ql = qc + 32;                                                  // loc
    for (uint32_t i = lane; i < p.D; i += 32) qs[i] = p.queries[(uint64_t)q * p.Dp + i];
    __syncwarp();
    // 1. threshold: the k-th smallest upper bound over every run of the query.
    // All of the query's run slots are one contiguous block [P][maxch][2][k];
    // lanes sweep it flat (slots of chunks h >= nch[c] were never written).
    // Only values <= the scan's shared threshold (itself one run's k-th upper
    // bound, so >= theta) can matter.
    const float pre = qthr_dec(__ldcg(reinterpret_cast<const uint32_t*>(p.qthr) + q));
    WarpTopK<KPL> th;
    th.init();
    {
        const uint32_t per_probe = p.maxch * 2u * p.k;
        const uint32_t total = p.P * per_probe;
        const uint64_t base = (uint64_t)q * total;
        // scan_vm_kernel: only warpgroup 0's runs (the first k of every 2k) hold
        // values; the sweep visits those only
        const uint32_t wsh = p.qt == (uint32_t)kVmQ ? 1u : 0u;
        const uint32_t vis = total >> wsh;
        for (uint32_t f0 = 32 * ws; f0 < vis; f0 += 32 * WPQ) {
            const uint32_t g = f0 + lane;
            bool pass = false;
            float v = 0.f;
            uint32_t f = 0;
            if (g < vis) {
                // g -> f: with wsh, g = (probe, chunk) * k + i maps to (probe, chunk) * 2k + i
                f = wsh ? (g / p.k) * 2u * p.k + g % p.k : g;
                const uint32_t pi = f / per_probe, rem = f - pi * per_probe;
                const uint32_t h = rem / (2u * p.k);
                const uint32_t c = (uint32_t)probes[(uint64_t)q * p.P + pi];
                if (h < p.nch[c]) {
                    v = p.ub[base + f];
                    pass = v <= pre && th.admits(v, (long long)(base + f));
                }
            }
            unsigned msk = __ballot_sync(0xffffffffu, pass);
            while (msk) {
                const int src = __ffs(msk) - 1;
                msk &= msk - 1;
                const float bv = __shfl_sync(0xffffffffu, v, src);
                const long long bi = (long long)(base + __shfl_sync(0xffffffffu, f, src));
                if (th.admits(bv, bi)) th.insert(bv, bi, (int)p.k, lane);
            }
        }
    }
    float theta = fminf(th.thr_d, pre);  // +inf if fewer than k vectors were scanned
    float* mrg = qsm + nw * p.Dp + nw * 64;  // (WPQ > 1) [warps][32 * KPL] floats + [warps][32 * KPL] ids
    if constexpr (WPQ > 1) {
        // the query's k-th smallest upper bound over every warp's share: the first
        // warp folds the others' k smallest values in
        float* mv = mrg + wq * 32 * KPL;
#pragma unroll
        for (int r = 0; r < KPL; ++r) mv[r * 32 + lane] = th.d[r];
        named_bar(4, WPQ * 32 * (nw / WPQ));  // every warp of the block (whole blocks of queries)
        if (ws == 0) {
            for (uint32_t o = 1; o < (uint32_t)WPQ; ++o) {
                const float* ov = mrg + (wq + o) * 32 * KPL;
#pragma unroll
                for (int r = 0; r < KPL; ++r) {
                    const uint32_t e = r * 32 + lane;
                    const float v = ov[r * 32 + lane];
                    const bool pass = e < p.k && th.admits(v, (long long)(o * 4096u + e));
                    unsigned msk = __ballot_sync(0xffffffffu, pass);
                    while (msk) {
                        const int src = __ffs(msk) - 1;
                        msk &= msk - 1;
                        const float bv = __shfl_sync(0xffffffffu, v, src);
                        const long long bi = (long long)(o * 4096u + r * 32 + src);
                        if (th.admits(bv, bi)) th.insert(bv, bi, (int)p.k, lane);
                    }
                }
            }
            if (lane == 0) mrg[wq * 32 * KPL] = fminf(th.thr_d, pre);
        }
        named_bar(4, WPQ * 32 * (nw / WPQ));
        theta = mrg[(wq - ws) * 32 * KPL];
        named_bar(4, WPQ * 32 * (nw / WPQ));  // the merge area is reused below
    }
    // 2. exact top-k over the surviving candidates
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
    uint32_t qn = 0;  // queued candidates (warp-uniform)
    auto flush = [&]() {
        bool ok = lane < qn;
        float dist = 0.f;
        long long id = -1;
        if (ok) {
            const uint32_t c = qc[lane], loc = ql[lane];
            const GroupRef g = ivf_group(p.L, c, p.snap_off[c], p.snap_len[c], loc >> 5);
            dist = p.off_rows ? exact_key_row<MET>(qs, cand_row(p, c, p.snap_off[c], loc >> 5, loc & 31), p.D)
                              : exact_key<MET>(qs, g.base + (loc & 31), p.D);
            id = g.ids[loc & 31];
        }
        offer(dist, id, ok);
        qn = 0;
        __syncwarp();
    };
    // 2b. candidates, 32 runs at a time (lane = run of the contiguous block
    // [P][maxch][2]): counts and candidate loads are independent across lanes,
    // so small batches with many chunks per list do not serialise on latency
    const uint32_t nruns = p.P * p.maxch * 2u;
    const uint64_t rbase = (uint64_t)q * nruns;
    for (uint32_t r0 = 32 * ws; r0 < nruns; r0 += 32 * WPQ) {
        const uint32_t r = r0 + lane;
        uint32_t c = 0, cnt = 0, h = 0;
        bool valid = false;
        if (r < nruns) {
            const uint32_t pi = r / (p.maxch * 2u);
            h = (r >> 1) - pi * p.maxch;
            c = (uint32_t)probes[(uint64_t)q * p.P + pi];
            valid = h < p.nch[c];
            if (valid) cnt = p.ccount[rbase + r];
        }
        // a chunk whose candidate buffer overflowed in either warpgroup run is rescanned
        const uint32_t pcnt = __shfl_xor_sync(0xffffffffu, cnt, 1);
        const bool ovf = valid && (cnt == kOverflow || pcnt == kOverflow);
        unsigned om = __ballot_sync(0xffffffffu, ovf && (r & 1u) == 0);
        while (om) {
            const int src = __ffs(om) - 1;
            om &= om - 1;
            const uint32_t cc = __shfl_sync(0xffffffffu, c, src);
            const uint32_t hh = __shfl_sync(0xffffffffu, h, src);
            const uint32_t off = p.snap_off[cc], len = p.snap_len[cc];
            const uint32_t ng = ivf_ngroups(p.L, off, len);
            const uint32_t g0 = hh * p.gc[cc], g1 = min(ng, g0 + p.gc[cc]);
            for (uint32_t j = g0; j < g1; ++j) {
                const GroupRef g = ivf_group(p.L, cc, off, len, j);
                const bool ok = lane < g.nvalid;
                const float dist = exact_key<MET>(qs, g.base + lane, p.D);
                offer(dist, ok ? g.ids[lane] : -1, ok);
            }
        }
        const uint32_t mycnt = (valid && !ovf) ? cnt : 0u;
        uint32_t mx = mycnt;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        for (uint32_t e = 0; e < mx; ++e) {
            const bool pass = e < mycnt && p.clb[(rbase + r) * kKC + e] <= theta;
            const unsigned msk = __ballot_sync(0xffffffffu, pass);
            const uint32_t np = __popc(msk);
            if (!np) continue;
            if (qn + np > 32) flush();
            if (pass) {
                const uint32_t slot = qn + __popc(msk & ((1u << lane) - 1u));
                qc[slot] = c;
                ql[slot] = p.cloc[(rbase + r) * kKC + e];
            }
            qn += np;
            __syncwarp();
        }
    }
    if (qn) flush();
    if constexpr (WPQ > 1) {  // fold the other warps' exact top-k lists into the first warp's
        float* md = mrg + wq * 32 * KPL * 3;
        long long* mi = reinterpret_cast<long long*>(md + 32 * KPL);
#pragma unroll
        for (int r = 0; r < KPL; ++r) {
            md[r * 32 + lane] = tk.d[r];
            mi[r * 32 + lane] = tk.id[r];
        }
        named_bar(4, WPQ * 32 * (nw / WPQ));
        if (ws != 0) return;
        for (uint32_t o = 1; o < (uint32_t)WPQ; ++o) {
            const float* od = mrg + (wq + o) * 32 * KPL * 3;
            const long long* oi = reinterpret_cast<const long long*>(od + 32 * KPL);
#pragma unroll
            for (int r = 0; r < KPL; ++r) offer(od[r * 32 + lane], oi[r * 32 + lane], oi[r * 32 + lane] >= 0);
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

// Ascending bitonic sort of 32*R keys across a warp: element e = 32 j + lane is
// v[j] of lane `lane` (partners 32 or more apart sit in the same lane).
template <int R>
__device__ __forceinline__ void warp_bitonic(uint64_t (&v)[R], uint32_t lane) {
#pragma unroll
    for (uint32_t sz = 2; sz <= 32u * R; sz <<= 1) {
#pragma unroll
        for (uint32_t st = sz >> 1; st > 0; st >>= 1) {
            if (st >= 32) {
                const uint32_t js = st >> 5;
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    if (j & js) continue;
                    const uint32_t e = 32u * j + lane;
                    const bool up = (e & sz) == 0;
                    const uint64_t a = v[j], b = v[j + js];
                    const uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
                    v[j] = up ? lo : hi;
                    v[j + js] = up ? hi : lo;
                }
            } else {
                const bool lower = (lane & st) == 0;
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    const uint64_t o = __shfl_xor_sync(0xffffffffu, v[j], st);
                    const bool up = ((32u * j + lane) & sz) == 0;
                    v[j] = (lower == up) ? (v[j] < o ? v[j] : o) : (v[j] < o ? o : v[j]);
                }
            }
        }
    }
}
// element e of a warp_bitonic array (warp-uniform e)
template <int R>
__device__ __forceinline__ uint64_t warp_elem(const uint64_t (&v)[R], uint32_t e) {
    // shuffle every register row and keep row e / 32: a register select chain here
    // gets folded into an indexed load, which moves the whole array to local memory
    uint64_t x = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const uint64_t t = __shfl_sync(0xffffffffu, v[j], e & 31);
        if (e >> 5 == (uint32_t)j) x = t;
    }
    return x;
}
// Seed of scan_vm_kernel's per-query thresholds (one warp per query): the exact
// k-th smallest distance (sequential fp32 over the mirror's row copy, the
// reference's bits) among the first two groups (<= 64 stored vectors) met
// walking the query's probes in rank order (rank 0 = its nearest list).  Those
// vectors are probed, so the value bounds the final k-th distance; fewer than k
// vectors leave the threshold at "none".
__global__ void vm_seed_kernel(TcParams p, const long long* probes, uint32_t nq) {
    extern __shared__ float qsm[];  // [warps][Dp]
    const uint32_t nw = blockDim.x >> 5, wq = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t q = blockIdx.x * nw + wq;
    if (q >= nq) return;
    float* qs = qsm + wq * p.Dp;
    for (uint32_t i = lane; i < p.D; i += 32) qs[i] = p.queries[(uint64_t)q * p.Dp + i];
    __syncwarp();
    // the samples (maint.cuh: central offline vectors of every list, interleaved
    // [list][d][slot]) of the query's two nearest probes; an entry deleted before
    // this search's plan snapshot was invalidated before that deletion was
    // published, so every entry read here is a vector the scan probes
    constexpr int kPer = (int)(kSampS / 32), kR = BIVF_VM_SEED_LISTS * kPer;  // 32-sample blocks
    uint64_t v[kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) v[r] = ~0ull;
    uint32_t nvec = 0;
#pragma unroll
    for (int r = 0; r < kR; ++r) {
        if ((uint32_t)(r / kPer) >= p.P) break;
        const uint32_t c = (uint32_t)probes[(uint64_t)q * p.P + r / kPer];
        const uint32_t sl = 32u * (r % kPer) + lane;
        const long long id = *reinterpret_cast<const volatile long long*>(p.samp_ids + (uint64_t)c * kSampS + sl);
        const bool ok = id >= 0;
        const float* x = p.samp_rows + (uint64_t)c * p.D * kSampS + sl;
        float dist = 0.f;  // exact_l2 over the [d][kSampS] sample rows
        for (uint32_t d0 = 0; d0 < p.D; d0 += 16) {
            float xv[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) xv[i] = d0 + i < p.D ? x[(uint64_t)(d0 + i) * kSampS] : 0.f;
#pragma unroll
            for (int i = 0; i < 16; ++i)
                if (d0 + i < p.D) dist = l2_step(dist, qs[d0 + i], xv[i]);
        }
        if (ok) v[r] = ((uint64_t)f2ord(dist) << 32) | (32u * r + lane);  // (r static: unrolled)
        nvec += __popc(__ballot_sync(0xffffffffu, ok));
    }
    if (nvec < p.k) return;  // qthr stays "none"
    warp_bitonic<kR>(v, lane);
    const uint64_t kth = warp_elem<kR>(v, p.k - 1);
    if (lane == 0) p.qthr[q] = __uint_as_float((uint32_t)(kth >> 32));
}
// Bound half-width of a dense-mode approximate key a of slot c (mirror.cuh eps'):
// L2 from |a|, |q|^2 (nqv) and |s|^2; inner product from kEpsIP |q| (nqv) and |x|
// (the wide mirror's norm row, second half), as tc_filter's W pass 2.
template <int MET>
__device__ __forceinline__ float dsel_eps(float a, float nqv, const float* nrm, uint32_t c) {
    if constexpr (MET == kL2) {
        const float ns = nrm[(c >> 5) * kNormFloats + (c & 31)];
        return fmaf(kEpsRel, fabsf(a), fmaf(kEpsT, nqv + ns, 1e-30f));
    } else {
        return fmaf(nqv, nrm[(c >> 5) * kNormFloats + 32 + (c & 31)], 1e-30f);
    }
}

// Fast selection of dense_select_kernel (R pre-threshold keys per lane, lists of
// 32 RL slots; k <= 32R <= n): true when
// the exact top-k was written (false: more than 32R values tie the bounds, the
// caller's general path runs with *pre as its pre-threshold).
template <int R, int RL, int MET, typename UbOf>
__device__ bool dense_select_fast(UbOf&& ub_of, const float* row, const float* nrm, float nqv,
                                  const float* qs, const float* rows, uint32_t D, uint32_t n,
                                  uint32_t k, uint32_t q, uint32_t lane, uint32_t* scratch,
                                  float* out_d, long long* out_i, float* pre,
                                  const float2* gs) {
    const float inf = __int_as_float(0x7f800000);
    // gs: this query's per-group (min upper, min lower) bounds from the TC kernel
    // (null: none).  With them phase A reads one value per group and passes 2 and
    // 3 open only the groups whose minimum can reach the threshold.
    const uint32_t ngq = (n + 31) / 32;
    // the k-th smallest group minimum bounds the k-th upper bound only if k <= groups,
    // and is selective only with several groups per wanted slot
    if (gs && 4 * k > ngq) gs = nullptr;
    // phase A: an upper bound of the k-th smallest upper bound from each lane's
    // R smallest values (32R values sorted across the warp): the k-th smallest
    // of any k values is >= the true k-th smallest
    float m[R];
#pragma unroll
    for (int j = 0; j < R; ++j) m[j] = inf;
    for (uint32_t c = lane; c < (gs ? ngq : n); c += 32) {
        float t = gs ? gs[c].x : ub_of(c);  // a group minimum is a real upper bound of a distinct slot
#pragma unroll
        for (int j = 0; j < R - 1; ++j) {
            const float a = fminf(m[j], t);
            t = fmaxf(m[j], t);
            m[j] = a;
        }
        m[R - 1] = fminf(m[R - 1], t);
    }
    uint64_t v[R];
#pragma unroll
    for (int j = 0; j < R; ++j) v[j] = (uint64_t)f2ord(m[j]) << 32;
    warp_bitonic<R>(v, lane);
    const uint32_t kk = k - 1;
    *pre = ord2f((uint32_t)(warp_elem<R>(v, kk) >> 32));
    uint64_t u[RL];  // the compacted lists (32 RL slots)
    // Fast path (no serialised warp inserts): every upper bound <= pre (>= k of
    // them, <= 32RL expected) compacted and bitonic-sorted -> theta = the k-th;
    // every lower bound <= theta (<= 32RL) recomputed exactly and sorted by the
    // (dist, id) key.  Longer lists fall through to the general path.
    uint32_t* l1 = scratch;  // [32RL] key hi, [32RL] c, [32RL] cand
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t n1 = 0;
    bool ok = true;
    // groups [g0, g0 + 32) at a time; `open` selects the ones to read slot by slot
    auto sweep = [&](auto&& open, auto&& slot) {
        for (uint32_t g0 = 0; g0 < ngq && ok; g0 += 32) {
            unsigned gm = __ballot_sync(0xffffffffu, g0 + lane < ngq && (!gs || open(gs[g0 + lane])));
            while (gm && ok) {
                const uint32_t g = g0 + __ffs(gm) - 1;
                gm &= gm - 1;
                slot(32 * g + lane);
            }
        }
    };
    sweep([&](float2 m) { return m.x <= *pre; }, [&](uint32_t c) {
        const float h = c < n ? ub_of(c) : inf;
        const bool pass = c < n && h <= *pre;
        const unsigned msk = __ballot_sync(0xffffffffu, pass);
        if (n1 + __popc(msk) > 32u * RL) {
            ok = false;
        } else {
            if (pass) {
                const uint32_t pos = n1 + __popc(msk & lt);
                l1[pos] = f2ord(h);
                l1[32 * RL + pos] = c;
            }
            n1 += __popc(msk);
        }
    });
    __syncwarp();
    if (ok && n1 >= k) {
#pragma unroll
        for (int j = 0; j < RL; ++j) {
            const uint32_t e = 32 * j + lane;
            u[j] = e < n1 ? ((uint64_t)l1[e] << 32 | l1[32 * RL + e]) : ~0ull;
        }
        warp_bitonic<RL>(u, lane);
        const float theta = ord2f((uint32_t)(warp_elem<RL>(u, kk) >> 32));
        uint32_t* cq = l1 + 64 * RL;
        uint32_t n2 = 0;
        sweep([&](float2 m) { return m.y <= theta; }, [&](uint32_t c) {
            bool cand = false;
            if (c < n) {
                const float a = row[c];
                cand = a - dsel_eps<MET>(a, nqv, nrm, c) <= theta;
            }
            const unsigned msk = __ballot_sync(0xffffffffu, cand);
            if (n2 + __popc(msk) > 32u * RL) {
                ok = false;
            } else {
                if (cand) cq[n2 + __popc(msk & lt)] = c;
                n2 += __popc(msk);
            }
        });
        __syncwarp();
        if (ok) {
#pragma unroll
            for (int j = 0; j < RL; ++j) {
                const uint32_t e = 32 * j + lane;
                u[j] = ~0ull;
                if (e < n2) {
                    const uint32_t c = cq[e];
                    u[j] = (uint64_t)f2ord(exact_key_row<MET>(qs, rows + (uint64_t)c * D, D)) << 32 | c;
                }
            }
            warp_bitonic<RL>(u, lane);
#pragma unroll
            for (int j = 0; j < RL; ++j) {
                const uint32_t e = 32 * j + lane;
                if (e < k) {
                    out_d[(uint64_t)q * k + e] = ord2f((uint32_t)(u[j] >> 32));
                    out_i[(uint64_t)q * k + e] = (long long)(uint32_t)u[j];
                }
            }
            return true;
        }
    }
    return false;
}

// Dense selection (the coarse quantizer): one warp per query over the n
// approximate distances of the dense mode.  Upper/lower bounds from the same
// eps' as the filter (mirror.cuh), threshold = k-th smallest upper bound, every
// slot whose lower bound is <= it recomputed EXACTLY (sequential fp32 over the
// row-major source rows, the reference's bits) -> exact (dist, id) top-k.
#ifndef BIVF_QSEL_MINB
#define BIVF_QSEL_MINB 6  // 64 registers (measured: quantizer 0.47 -> 0.41 ms at nprobe 64)
#endif
template <int KPL, int MET>
__global__ void __launch_bounds__(128, BIVF_QSEL_MINB) dense_select_kernel(const float* dense, uint32_t ld, const float* dnq,
                                    const float* nrm, const float* rows, const float* queries,
                                    uint32_t Dp, uint32_t D, uint32_t n, uint32_t nq, uint32_t k,
                                    float* out_d, long long* out_i, const float2* gsum) {
    extern __shared__ float qsm[];
    const uint32_t nw = blockDim.x >> 5, wq = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t q = blockIdx.x * nw + wq;
    if (q >= nq) return;
    float* qs = qsm + wq * Dp;
    for (uint32_t i = lane; i < D; i += 32) qs[i] = queries[(uint64_t)q * Dp + i];
    __syncwarp();
    const float nqv = dnq[q];
    const float* row = dense + (uint64_t)q * ld;
    const float inf = __int_as_float(0x7f800000);
    auto ub_of = [&](uint32_t c) {
        const float a = row[c];
        return a + dsel_eps<MET>(a, nqv, nrm, c);
    };
    // phase A (+ the fast selection when <= 32R values tie the bounds): the k-th
    // smallest of each lane's R smallest upper bounds bounds the k-th smallest
    float pre = inf;
    uint32_t* fscr = reinterpret_cast<uint32_t*>(qsm + nw * Dp) + nw * 32 + wq * 768;
    const float2* gs = gsum ? gsum + (uint64_t)q * ((n + 31) / 32) : nullptr;
    if (k <= 32 && n >= 64) {
        if (dense_select_fast<2, 2, MET>(ub_of, row, nrm, nqv, qs, rows, D, n, k, q, lane, fscr, out_d, out_i, &pre, gs))
            return;
    } else if (k <= 64 && n >= 128) {
        if (dense_select_fast<4, 8, MET>(ub_of, row, nrm, nqv, qs, rows, D, n, k, q, lane, fscr, out_d, out_i, &pre, gs))
            return;
    } else if (k <= 128 && n >= 256) {
        if (dense_select_fast<8, 8, MET>(ub_of, row, nrm, nqv, qs, rows, D, n, k, q, lane, fscr, out_d, out_i, &pre, gs))
            return;
    }
    WarpTopK<KPL> th;
    th.init();
    for (uint32_t c0 = 0; c0 < n; c0 += 32) {
        const uint32_t c = c0 + lane;
        const float h = c < n ? ub_of(c) : inf;
        const bool pass = c < n && h <= pre && th.admits(h, (long long)c);
        unsigned m = __ballot_sync(0xffffffffu, pass);
        while (m) {
            const int src = __ffs(m) - 1;
            m &= m - 1;
            const float bh = __shfl_sync(0xffffffffu, h, src);
            const long long bc = __shfl_sync(0xffffffffu, (long long)c, src);
            if (th.admits(bh, bc)) th.insert(bh, bc, (int)k, lane);
        }
    }
    const float theta = fminf(th.thr_d, pre);  // +inf when n < k
    // pass 2: candidates (lower bound <= theta) queued 32 at a time, then one
    // exact distance per lane (parallel sequential chains, not one per chunk)
    WarpTopK<KPL> tk;
    tk.init();
    uint32_t* queue = reinterpret_cast<uint32_t*>(qsm + nw * Dp) + wq * 32;
    uint32_t qn = 0;
    auto flush = [&]() {
        const bool ok = lane < qn;
        const uint32_t c = ok ? queue[lane] : 0u;
        const float dist = ok ? exact_key_row<MET>(qs, rows + (uint64_t)c * D, D) : 0.f;
        const bool pass = ok && tk.admits(dist, (long long)c);
        unsigned m = __ballot_sync(0xffffffffu, pass);
        while (m) {
            const int src = __ffs(m) - 1;
            m &= m - 1;
            const float bd = __shfl_sync(0xffffffffu, dist, src);
            const long long bc = __shfl_sync(0xffffffffu, (long long)c, src);
            if (tk.admits(bd, bc)) tk.insert(bd, bc, (int)k, lane);
        }
        qn = 0;
        __syncwarp();
    };
    for (uint32_t c0 = 0; c0 < n; c0 += 32) {
        const uint32_t c = c0 + lane;
        bool cand = false;
        if (c < n) {
            const float a = row[c];
            cand = a - dsel_eps<MET>(a, nqv, nrm, c) <= theta;
        }
        const unsigned msk = __ballot_sync(0xffffffffu, cand);
        const uint32_t np = __popc(msk);
        if (qn + np > 32) flush();
        if (cand) queue[qn + __popc(msk & ((1u << lane) - 1u))] = c;
        qn += np;
        __syncwarp();
    }
    if (qn) flush();
#pragma unroll
    for (int r = 0; r < KPL; ++r) {
        const uint32_t e = r * 32 + lane;
        if (e < k) {
            out_d[(uint64_t)q * k + e] = tk.d[r];
            out_i[(uint64_t)q * k + e] = tk.id[r];
        }
    }
}

// ---------------------------------------------------------------- dense IVF (k > 32)
// Group g's global index (norms / rows arrays) of group j of list c.
__device__ __forceinline__ uint64_t ivf_group_index(const DevLists& L, uint32_t c, uint32_t off,
                                                    uint32_t j, bool& arena) {
    const uint32_t og = (off + 31u) >> 5;
    if (j < og) {
        arena = false;
        return L.off_start[c] / 32u + j;
    }
    const uint32_t jj = j - og, mid = jj / L.gpb, gi = jj - mid * L.gpb;
    arena = true;
    return (uint64_t)L.rowptr[c][mid] * L.gpb + gi;
}

// One warp per query over the dense approximate distances of all its probed
// lists (TC dense mode, tiled rows at dense_list_base): (A) a pre-threshold from each
// lane's 4 smallest upper bounds (the k-th of any 128 values bounds the k-th
// overall, k <= 128), (B) the exact k-th smallest upper bound, (C) every slot
// whose lower bound reaches it recomputed EXACTLY (mirror rows, the
// reference's sequential fp32 bits) into the (dist, id) top-k.
constexpr uint32_t kSelMetaBytes = 40;  // per-probe metadata of dense_ivf_select_kernel
constexpr uint32_t kSelChunk = 256;     // probes whose metadata one warp holds at a time
#ifndef BIVF_SEL_INFLIGHT
#define BIVF_SEL_INFLIGHT 2
#endif
constexpr int kSelInflight = BIVF_SEL_INFLIGHT;  // group-summary loads in flight per lane

template <int KPL>
#ifndef BIVF_SEL_MINB
#define BIVF_SEL_MINB 6  // 80 registers: 6 blocks of 4 warps per SM
#endif
__global__ void __launch_bounds__(128, BIVF_SEL_MINB) dense_ivf_select_kernel(TcParams p, const long long* probes, float* out_d,
                                        long long* out_i, uint32_t* out_cnt, uint32_t nq) {
    extern __shared__ float qsm[];
    const uint32_t nw = blockDim.x >> 5, wq = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t q = blockIdx.x * nw + wq;
    if (q >= nq) return;
    float* qs = qsm + wq * p.Dp;
    uint32_t* qc = reinterpret_cast<uint32_t*>(qsm + nw * p.Dp) + wq * 64;
    uint32_t* ql = qc + 32;
    for (uint32_t i = lane; i < p.D; i += 32) qs[i] = p.queries[(uint64_t)q * p.Dp + i];
    __syncwarp();
    // per-probe metadata of up to kSelChunk probes, gathered lane-parallel at the
    // start of each chunk of a sweep (the sweeps would otherwise walk probes ->
    // list -> plan position serially for every pair)
    const uint32_t PC = min(p.P, kSelChunk);
    char* meta = reinterpret_cast<char*>(qsm + nw * p.Dp) + nw * 256;
    meta = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(meta) + 15) & ~uintptr_t(15)) +
           (size_t)wq * PC * kSelMetaBytes;
    uint64_t* m_blk = reinterpret_cast<uint64_t*>(meta);  // the pair's tile base in dense_out
    uint64_t* m_g0 = m_blk + PC;                           // its first group summary
    uint32_t* m_c = reinterpret_cast<uint32_t*>(m_g0 + PC);
    uint32_t* m_off = m_c + PC;
    uint32_t* m_len = m_off + PC;
    uint32_t* m_ng = m_len + PC;
    uint32_t* m_row = m_ng + PC;  // the pair's row in its tile
    float* m_nq = reinterpret_cast<float*>(m_row + PC);
    auto gather = [&](uint32_t pb, uint32_t pn) {
        __syncwarp();
        for (uint32_t pi = lane; pi < pn; pi += 32) {
            const uint64_t pair = (uint64_t)q * p.P + pb + pi;
            const uint32_t c = (uint32_t)probes[pair];
            const uint32_t off = p.snap_off[c], len = p.snap_len[c], ng = ivf_ngroups(p.L, off, len);
            const uint32_t pos = p.dense_ppos[pair];
            const uint64_t blk = p.dense_list_base[c] + (uint64_t)(pos / kM) * ng * 32u * kM;
            m_blk[pi] = blk;
            m_g0[pi] = blk / 32u + (uint64_t)(pos % kM) * ng;
            m_c[pi] = c;
            m_off[pi] = off;
            m_len[pi] = len;
            m_ng[pi] = ng;
            m_row[pi] = pos % kM;
            m_nq[pi] = p.dense_nq[pair];
        }
        __syncwarp();
    };
    const float inf = __int_as_float(0x7f800000);
    // the query's groups, a flat index over its probes: lane-strided sweeps read
    // the (min upper, min lower) group summaries, four 32-group chunks in flight;
    // only groups that can matter are opened slot by slot
    auto groups = [&](auto&& f) {  // f(chunk-local probe, group, valid, summary), per lane
        // the order of a query's groups does not matter to any sweep, so each lane
        // walks its own flat index (lane, lane + 32, ...) over the chunk's groups
        // with kSelInflight summary loads in flight
        for (uint32_t pb = 0; pb < p.P; pb += kSelChunk) {
            const uint32_t pn = min(kSelChunk, p.P - pb);
            gather(pb, pn);
            uint32_t pi = 0, j = lane;
            auto norm = [&]() {
                while (pi < pn && j >= m_ng[pi]) {
                    j -= m_ng[pi];
                    ++pi;
                }
            };
            norm();
            while (__any_sync(0xffffffffu, pi < pn)) {
                uint32_t ps[kSelInflight], js[kSelInflight];
                float2 v[kSelInflight];
#pragma unroll
                for (int u = 0; u < kSelInflight; ++u) {
                    ps[u] = pi;
                    js[u] = j;
                    v[u] = pi < pn ? p.dense_gsum[m_g0[pi] + j] : make_float2(inf, inf);
                    j += 32;
                    norm();
                }
#pragma unroll
                for (int u = 0; u < kSelInflight; ++u) f(ps[u], js[u], ps[u] < pn, v[u]);
            }
        }
    };
    // open group j of probe pi: one slot per lane -> (valid, h, l)
    auto open = [&](uint32_t pi, uint32_t j, float& h, float& l) -> bool {
        const uint32_t c = m_c[pi], off = m_off[pi];
        bool ar;
        const uint64_t g = ivf_group_index(p.L, c, off, j, ar);
        const GroupRef gr = ivf_group(p.L, c, off, m_len[pi], j);
        h = inf;
        l = inf;
        if (lane < gr.nvalid) {
            const float a = p.dense_out[m_blk[pi] + ((uint64_t)j * kM + m_row[pi]) * 32u + lane];
            const float ns = (ar ? p.arena_nrm : p.off_nrm)[g * kNormFloats + lane];
            const float e = fmaf(kEpsRel, fabsf(a), fmaf(kEpsT, m_nq[pi] + ns, 1e-30f));
            h = a + e;
            l = a - e;
        }
        return lane < gr.nvalid;
    };
    // (A) pre-threshold: the k-th smallest of the group minima (each a real
    // upper bound of a distinct slot) bounds the k-th smallest upper bound;
    // each lane keeps its 4 smallest, 128 values sorted across the warp
    float pre = inf;
    if (p.k <= 128) {
        float b[4] = {inf, inf, inf, inf};
        groups([&](uint32_t, uint32_t, bool valid, float2 sm) {
            if (!valid) return;
            float x = sm.x;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float lo = fminf(x, b[i]);
                x = fmaxf(x, b[i]);
                b[i] = lo;
            }
        });
        for (uint32_t sz = 2; sz <= 128; sz <<= 1) {
            for (uint32_t st = sz >> 1; st > 0; st >>= 1) {
                if (st >= 32) {
                    const uint32_t rs = st >> 5;
#pragma unroll
                    for (uint32_t r = 0; r < 4; ++r) {
                        if (r & rs) continue;
                        const uint32_t i = r * 32 + lane;
                        const bool up = (i & sz) == 0;
                        const float lo = fminf(b[r], b[r + rs]), hi = fmaxf(b[r], b[r + rs]);
                        b[r] = up ? lo : hi;
                        b[r + rs] = up ? hi : lo;
                    }
                } else {
#pragma unroll
                    for (uint32_t r = 0; r < 4; ++r) {
                        const float o = __shfl_xor_sync(0xffffffffu, b[r], st);
                        const uint32_t i = r * 32 + lane;
                        const bool lower = (lane & st) == 0, up = (i & sz) == 0;
                        b[r] = (lower == up) ? fminf(b[r], o) : fmaxf(b[r], o);
                    }
                }
            }
        }
        const uint32_t kk = p.k - 1;
        const float cand = kk < 32 ? b[0] : kk < 64 ? b[1] : kk < 96 ? b[2] : b[3];
        pre = __shfl_sync(0xffffffffu, cand, kk & 31);
    }
    // (B) the exact k-th smallest upper bound: open the groups whose minimum
    // upper bound is <= pre (values only: ties do not move the k-th value)
    WarpTopVal<KPL> th;
    th.init();
    groups([&](uint32_t gpi, uint32_t gj, bool valid, float2 sm) {
        unsigned gm = __ballot_sync(0xffffffffu, valid && sm.x <= pre);
        while (gm) {
            const int src = __ffs(gm) - 1;
            gm &= gm - 1;
            const uint32_t pi = __shfl_sync(0xffffffffu, gpi, src), j = __shfl_sync(0xffffffffu, gj, src);
            float h, l;
            const bool ok = open(pi, j, h, l);
            const bool pass = ok && h <= pre && th.admits(h);
            unsigned m = __ballot_sync(0xffffffffu, pass);
            while (m) {
                const int s2 = __ffs(m) - 1;
                m &= m - 1;
                const float bh = __shfl_sync(0xffffffffu, h, s2);
                if (th.admits(bh)) th.insert(bh, (int)p.k, lane);
            }
        }
    });
    const float theta = fminf(th.thr, pre);
    // (C) exact top-k over the candidates (groups whose minimum lower bound
    // reaches theta, then their slots), recomputed 32 at a time
    WarpTopK<KPL> tk;
    tk.init();
    uint32_t qn = 0;
    auto flush = [&]() {
        const bool ok = lane < qn;
        float dist = 0.f;
        long long id = -1;
        if (ok) {
            const uint32_t c = qc[lane], loc = ql[lane];
            const GroupRef g = ivf_group(p.L, c, p.snap_off[c], p.snap_len[c], loc >> 5);
            dist = exact_l2_row(qs, cand_row(p, c, p.snap_off[c], loc >> 5, loc & 31), p.D);
            id = g.ids[loc & 31];
        }
        const bool pass = ok && tk.admits(dist, id);
        unsigned m = __ballot_sync(0xffffffffu, pass);
        while (m) {
            const int src = __ffs(m) - 1;
            m &= m - 1;
            const float bd = __shfl_sync(0xffffffffu, dist, src);
            const long long bi = __shfl_sync(0xffffffffu, id, src);
            if (tk.admits(bd, bi)) tk.insert(bd, bi, (int)p.k, lane);
        }
        qn = 0;
        __syncwarp();
    };
    groups([&](uint32_t gpi, uint32_t gj, bool valid, float2 sm) {
        unsigned gm = __ballot_sync(0xffffffffu, valid && sm.y <= theta);
        while (gm) {
            const int src = __ffs(gm) - 1;
            gm &= gm - 1;
            const uint32_t pi = __shfl_sync(0xffffffffu, gpi, src), j = __shfl_sync(0xffffffffu, gj, src);
            float h, l;
            const bool cand = open(pi, j, h, l) && l <= theta;
            const unsigned msk = __ballot_sync(0xffffffffu, cand);
            const uint32_t np = __popc(msk);
            if (!np) continue;
            if (qn + np > 32) flush();
            if (cand) {
                const uint32_t slot = qn + __popc(msk & ((1u << lane) - 1u));
                qc[slot] = m_c[pi];
                ql[slot] = (j << 5) | lane;
            }
            qn += np;
            __syncwarp();
        }
    });
    if (qn) flush();
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

__global__ void dense_list_len_kernel(DevLists L, const uint32_t* snap_off, const uint32_t* snap_len,
                                      const uint32_t* qoff, uint32_t C, uint64_t* len) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    const uint64_t tiles = (qoff[c + 1] - qoff[c] + kM - 1) / kM;
    len[c] = tiles * ivf_ngroups(L, snap_off[c], snap_len[c]) * 32ull * kM;
}

template <int KT, bool W>
constexpr size_t tc_smem_bytes() {
    return 1024 + TcCfg<KT, W>::NS * TcCfg<KT, W>::STAGE + kWG * 32 * kM * 4 + kWG * TcCfg<KT, W>::KC * kM * 8 +
           kNR * kGU * kNormFloats * 4 +
           (2 * TcCfg<KT, W>::NU + 2 * kNB + 2 * kNR + 2 * kRing + 4) * 8 + kRing * sizeof(TcItem) +
           kWG * kMaxD * 4 + 4 * kWG * kM * 4 + 16;
}
static_assert(tc_smem_bytes<16, false>() <= 232448 && tc_smem_bytes<32, false>() <= 232448 &&
                  tc_smem_bytes<16, true>() <= 232448 && tc_smem_bytes<32, true>() <= 232448,
              "smem budget");

constexpr size_t vm_smem_bytes() {
    return 1024 + kVmNS * kVmSlot + 4 * kVmPlane + 4 * kVmWG * 1024 * 4 + 4 * kVmWG * kVmKC * 32 * 8 + kVmNR * 4 * 32 * 4 +
           2 * kVmQ * 4 * 3 + kMaxD * 4 + 16 * kVmQ * 4 + 2 * kVmQ * 4 + 4 * kVmQ * 4 + 2 * 32 * kVmQ * 4 +
           (2 * kVmNS + 2 * kVmNB + 4 + 2 * kRing + 2 * kVmNR) * 8 + kRing * sizeof(TcItem) + 16;
}
static_assert(vm_smem_bytes() <= 232448, "vm smem budget");

template <int KT>
cudaError_t vm_attr() {
    static bool done = false;
    if (done) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(scan_vm_kernel<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)vm_smem_bytes());
    done = e == cudaSuccess;
    return e;
}

template <int KT, bool W>
cudaError_t tc_attr() {
    static bool done = false;
    if (done) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(scan_tc_kernel<KT, W>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)tc_smem_bytes<KT, W>());
    done = e == cudaSuccess;
    return e;
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
    if (k > 32 || D < 8) return false;
    // L2: 3xBF16, D <= 128; inner product: the wide 1xBF16 mode, A (the query
    // rows' hi plane) fits its 384 TMEM columns up to D = 768
    return metric == kL2 ? D <= (uint32_t)kMaxD : mirror_k_wide(D) <= 768;
}

bool tc_dense_supported(uint32_t D, uint32_t k, int metric) {
    return metric == kL2 && D >= 8 && D <= (uint32_t)kMaxD && k > 32 && k <= 256;
}

cudaError_t make_mirror_map(const float* base, uint64_t groups, uint32_t D, bool wide,
                            CUtensorMap* out, bool hi_only) {
    auto enc = get_encode();
    if (!enc) return cudaErrorNotSupported;
    // rows per group: 2K (hi + lo planes) or, wide, K (hi plane) read in chunks;
    // hi_only (scan_vm_kernel): a box of the hi plane's K rows of a 2K-row group
    const uint32_t K = wide ? mirror_k_wide(D) : mirror_k(D);
    const uint32_t rows = wide ? K : 2 * K;
    const uint32_t box_rows = wide ? mirror_chunk_wide(D) : hi_only ? K : 2 * K;
    cuuint64_t dims[2] = {32, std::max<cuuint64_t>(groups * rows, 1)};
    cuuint64_t strides[1] = {64};
    cuuint32_t box[2] = {32, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<float*>(base), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_64B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t make_vm_maps(const float* mir, const float* nrm, uint64_t groups, uint32_t D, CUtensorMap* out3) {
    auto enc = get_encode();
    if (!enc) return cudaErrorNotSupported;
    const uint32_t K = mirror_k(D);
    const cuuint64_t g = std::max<cuuint64_t>(groups, 1);
    cuuint32_t e2[2] = {1, 1}, e3[3] = {1, 1, 1};
    CUresult r;
    {  // one group's hi plane: rows [0, K) of its 2K rows
        cuuint64_t dims[2] = {32, g * 2 * K};
        cuuint64_t str[1] = {64};
        cuuint32_t box[2] = {32, K};
        r = enc(&out3[0], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<float*>(mir), dims, str, box, e2,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
    {  // four consecutive groups' hi planes: {32 slots, K rows, groups}, group stride 2K rows
        cuuint64_t dims[3] = {32, K, g};
        cuuint64_t str[2] = {64, (cuuint64_t)2 * K * 64};
        cuuint32_t box[3] = {32, K, 4};
        r = enc(&out3[1], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<float*>(mir), dims, str, box, e3,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
    {  // the |s|^2 rows (first 32 of each group's 64 norm floats) of four consecutive groups
        cuuint64_t dims[2] = {kNormFloats, g};
        cuuint64_t str[1] = {kNormFloats * 4};
        cuuint32_t box[2] = {32, 4};
        r = enc(&out3[2], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(nrm), dims, str, box, e2,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
    return cudaSuccess;
}

namespace {
__global__ void dense_total_kernel(const uint64_t* off, const uint64_t* len, uint32_t n,
                                   uint64_t* total) {
    *total = n ? off[n - 1] + len[n - 1] : 0;
}
}  // namespace

size_t dense_plan_tmp_bytes(uint32_t nlists) {
    size_t b = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, b, static_cast<const uint64_t*>(nullptr),
                                  static_cast<uint64_t*>(nullptr), (int)nlists);
    return b;
}

cudaError_t launch_dense_plan(const DevLists& L, const PlanBufs& B, const long long* probes,
                              const SearchShape& sh, uint64_t* list_len, uint64_t* list_base,
                              void* tmp, size_t tmp_bytes, uint64_t* total, cudaStream_t s) {
    SearchShape s2 = sh;
    s2.QT = kM;
    cudaError_t e = launch_plan(L, B, probes, s2, s);
    if (e != cudaSuccess) return e;
    dense_list_len_kernel<<<(L.C + 255) / 256, 256, 0, s>>>(L, B.snap_off, B.snap_len, B.qoff, L.C,
                                                            list_len);
    e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, list_len, list_base, (int)L.C, s);
    if (e != cudaSuccess) return e;
    dense_total_kernel<<<1, 1, 0, s>>>(list_base, list_len, L.C, total);
    count_launch(3);
    return cudaGetLastError();
}

// The vector-major path (scan_vm_kernel): plan with kVmQ-pair tiles, exact
// seeds, scan, refine.
static cudaError_t launch_vm(const DevLists& L, const PlanBufs& B, const long long* probes, const float* queries,
                             const float* centroids, const SearchShape& sh, const CUtensorMap* maps_hi,
                             const float* off_nrm, const float* arena_nrm, const float* off_rows,
                             const float* arena_rows, const TcBufs& T, float* out_d, long long* out_i,
                             uint32_t* out_cnt, int num_sms, cudaStream_t s, cudaEvent_t ev0, cudaEvent_t ev1,
                             int max_grid, const float* samp_rows, const long long* samp_ids) {
    SearchShape s2 = sh;
    s2.QT = kVmQ;
    cudaError_t e = launch_plan(L, B, probes, s2, s);
    if (e != cudaSuccess) return e;
    TcParams p{};
    p.L = snapshot_view(L, B);
    p.D = L.D;
    p.Dk = (L.D + 15) & ~15u;
    p.brow = p.Dk;
    p.gstride = 2 * p.Dk;
    p.nkc = 1;
    p.Dp = pad4(L.D);
    p.k = sh.k;
    p.P = sh.P;
    p.maxch = sh.maxch;
    p.qt = kVmQ;
    p.samp_rows = samp_rows;
    p.samp_ids = samp_ids;
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
    p.off_nrm = off_nrm;
    p.arena_nrm = arena_nrm;
    p.off_rows = off_rows;
    p.arena_rows = arena_rows;
    p.qthr = T.qthr;
    p.ub = T.ub;
    p.ccount = T.ccount;
    p.clb = T.clb;
    p.cloc = T.cloc;
    e = sh.k == 10 ? vm_attr<10>() : sh.k <= 16 ? vm_attr<16>() : vm_attr<32>();
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(T.qthr, 0xff, (size_t)sh.nq * 4, s);
    if (e != cudaSuccess) return e;
    if (ev0) cudaEventRecord(ev0, s);
    const uint32_t wpb = 4;
    static const bool seed_env = [] {
        const char* v = std::getenv("BIVF_VM_SEED");  // 0: no seed thresholds (tuning aid)
        return !(v && v[0] == '0');
    }();
    if (seed_env && samp_ids) vm_seed_kernel<<<(sh.nq + wpb - 1) / wpb, wpb * 32, wpb * p.Dp * 4, s>>>(p, probes, sh.nq);
    int grid = std::max(1, std::min(num_sms, max_grid));
    if (const char* g = std::getenv("BIVF_TC_GRID")) grid = std::max(1, atoi(g));  // debugging aid
    VmMaps vmaps;
    for (int a = 0; a < 2; ++a)
        for (int i = 0; i < 3; ++i) vmaps.m[a][i] = maps_hi[3 * a + i];
    // KT = the k-best slots an offer reads: exactly 10 for the common k = 10
    if (sh.k == 10) scan_vm_kernel<10><<<grid, kVmThreads, vm_smem_bytes(), s>>>(p, vmaps);
    else if (sh.k <= 16) scan_vm_kernel<16><<<grid, kVmThreads, vm_smem_bytes(), s>>>(p, vmaps);
    else scan_vm_kernel<32><<<grid, kVmThreads, vm_smem_bytes(), s>>>(p, vmaps);
    count_launch(2);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (ev1) cudaEventRecord(ev1, s);
    // small batches: 8 warps per query (the refine is latency-bound per warp)
    if (sh.nq * 8 <= (uint32_t)num_sms * 16) {
        constexpr int WPQ = 8;
        const size_t sm = WPQ * (p.Dp * 4 + 256) + WPQ * 32 * 1 * 12 + 16;
        refine_kernel<1, kL2, WPQ><<<sh.nq, WPQ * 32, sm, s>>>(p, probes, out_d, out_i, out_cnt, sh.nq);
    } else {
        refine_kernel<1, kL2, 1><<<(sh.nq + wpb - 1) / wpb, wpb * 32, wpb * (p.Dp * 4 + 256), s>>>(
            p, probes, out_d, out_i, out_cnt, sh.nq);
    }
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_ivf_search_tc(const DevLists& L, const PlanBufs& B, const long long* probes,
                                 const float* queries, const float* centroids,
                                 const SearchShape& sh, const CUtensorMap& map_off,
                                 const CUtensorMap& map_arena, const float* off_nrm,
                                 const float* arena_nrm, const float* off_rows,
                                 const float* arena_rows, const TcBufs& T, const TcDense* dense,
                                 float* out_d,
                                 long long* out_i, uint32_t* out_cnt, int num_sms,
                                 cudaStream_t s, cudaEvent_t ev0, cudaEvent_t ev1, int max_grid,
                                 const CUtensorMap* maps_hi, const float* samp_rows, const long long* samp_ids,
                                 int vm_mode) {
    if (sh.nq == 0) return cudaSuccess;
    const bool wide = sh.metric == kIP;  // 1xBF16 inner-product mode (mirror.cuh wide mirror)
    if (wide && dense && dense->list_base) return cudaErrorInvalidValue;  // IVF dense mode: L2 only
    static const bool vm_env = [] {
        const char* v = std::getenv("BIVF_TC_VM");  // 0: the query-major 3xBF16 scan (comparison aid)
        return !(v && v[0] == '0');
    }();
    // the vector-major scan reads a list once per <= 32-query tile and filters
    // with the vectors' bf16 hi plane only: it wins while lists see few queries
    // (the north star: 29 pairs per list); with many pairs per list the
    // query-major kernel's 128-query tiles and 3xBF16 bound (far fewer
    // candidates on dense data) win (measured: cfg1 625 and cfg3 78 pairs per list)
    static const double vm_max_ppl = [] {
        const char* v = std::getenv("BIVF_VM_MAX_PPL");  // tuning aid
        return v ? atof(v) : 48.0;
    }();
    const double ppl = (double)sh.nq * sh.P / std::max<uint32_t>(1u, L.C);
    if (maps_hi && vm_env && !wide && !dense && L.D <= (uint32_t)kMaxD &&
        (vm_mode == 1 || (vm_mode < 0 && ppl <= vm_max_ppl)))
        return launch_vm(L, B, probes, queries, centroids, sh, maps_hi, off_nrm, arena_nrm, off_rows,
                         arena_rows, T, out_d, out_i, out_cnt, num_sms, s, ev0, ev1, max_grid, samp_rows, samp_ids);
    SearchShape s2 = sh;
    s2.QT = kM;
    cudaError_t e = cudaSuccess;
    // Seeded filter scan (batches of >= 512 queries): a seeding pass scans the
    // first unit (2 groups = 64 vectors) of every query's NEAREST list (probe
    // rank 0) and publishes the k-th smallest upper bound as the query's shared
    // threshold (a valid bound: those vectors are probed); the full scan then
    // filters against it from its first group on (no per-run threshold warm-up,
    // far fewer pass-2 slots).  The seeding pass writes no run output.
    static const uint32_t two_min = [] {
        const char* v = std::getenv("BIVF_TC_TWO_PHASE_MIN");  // tuning aid
        return v ? (uint32_t)atoi(v) : 512u;
    }();
    static const uint32_t seed_g = [] {
        const char* v = std::getenv("BIVF_TC_SEED_GROUPS");  // tuning aid
        return v ? std::max(1u, (uint32_t)atoi(v)) : (uint32_t)kGU;
    }();
    // (not for the inner-product wide mode: at D = 768 the seeding pass's item
    // builds cost more than the seeded thresholds save -- measured 2.15 ms seeded
    // vs 1.88 ms unseeded scan per 10K queries, 2M x 768, nprobe 32)
    const bool two = !dense && !wide && sh.P >= 2 && sh.nq >= two_min;
    SearchShape sa = s2;  // seeding pass: rank-0 pairs, one chunk per list
    sa.maxch = 1;
    if (!(dense && dense->list_base)) {  // the IVF dense path planned in launch_dense_plan
        e = two ? launch_plan_ranked(L, B, probes, sa, 0, 1, true, s) : launch_plan(L, B, probes, s2, s);
        if (e != cudaSuccess) return e;
    }
    TcParams p{};
    p.L = snapshot_view(L, B);  // every kernel after the plan reads the plan's snapshot
    p.D = L.D;
    p.Dk = wide ? mirror_k_wide(L.D) : (L.D + 15) & ~15u;
    p.brow = wide ? mirror_chunk_wide(L.D) : 2 * p.Dk;
    p.gstride = wide ? p.Dk : 2 * p.Dk;
    p.nkc = wide ? p.Dk / p.brow : 1;
    p.Dp = pad4(L.D);
    p.k = sh.k;
    p.P = sh.P;
    p.maxch = sh.maxch;
    p.qt = kM;
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
    p.off_nrm = off_nrm;
    p.off_rows = off_rows;
    p.arena_rows = arena_rows;
    p.qthr = T.qthr;
    if (dense) {
        p.dense_out = dense->out;
        p.dense_nq = dense->nq;
        p.dense_ld = dense->ld;
        p.dense_list_base = dense->list_base;
        p.dense_ppos = B.ppos;
        p.dense_gsum = dense->gsum;
    }
    p.arena_nrm = arena_nrm;
    p.ub = T.ub;
    p.ccount = T.ccount;
    p.clb = T.clb;
    p.cloc = T.cloc;
    const size_t sm16 = wide ? tc_smem_bytes<16, true>() : tc_smem_bytes<16, false>();
    const size_t sm32 = wide ? tc_smem_bytes<32, true>() : tc_smem_bytes<32, false>();
    e = wide ? (sh.k <= 16 ? tc_attr<16, true>() : tc_attr<32, true>())
             : (sh.k <= 16 ? tc_attr<16, false>() : tc_attr<32, false>());
    if (e != cudaSuccess) return e;
    // shared per-query thresholds start at "none" (0xffffffff, qthr_dec -> +inf)
    e = cudaMemsetAsync(T.qthr, 0xff, (size_t)sh.nq * 4, s);
    if (e != cudaSuccess) return e;
    if (ev0) cudaEventRecord(ev0, s);
    int grid = std::max(1, std::min(num_sms, max_grid));  // no idle CTAs holding whole SMs
    if (const char* g = std::getenv("BIVF_TC_GRID")) grid = std::max(1, atoi(g));  // debugging aid
    for (int phase = 0; phase < (two ? 2 : 1); ++phase) {
        p.seed_groups = two && phase == 0 ? seed_g : 0u;
        if (two && phase == 1) {
            e = launch_plan(L, B, probes, s2, s);
            if (e != cudaSuccess) return e;
        }
        if (wide) {
            if (sh.k <= 16) scan_tc_kernel<16, true><<<grid, kTcThreads, sm16, s>>>(p, map_off, map_arena);
            else scan_tc_kernel<32, true><<<grid, kTcThreads, sm32, s>>>(p, map_off, map_arena);
        } else {
            if (sh.k <= 16) scan_tc_kernel<16, false><<<grid, kTcThreads, sm16, s>>>(p, map_off, map_arena);
            else scan_tc_kernel<32, false><<<grid, kTcThreads, sm32, s>>>(p, map_off, map_arena);
        }
        count_launch();
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (ev1) cudaEventRecord(ev1, s);
    const uint32_t wpb = 4;
    if (dense && dense->list_base) {
        const size_t sm_sel = wpb * (p.Dp * 4 + 256) + 16 + wpb * std::min(sh.P, kSelChunk) * kSelMetaBytes;
        if (sh.k <= 32)
            dense_ivf_select_kernel<1><<<(sh.nq + wpb - 1) / wpb, wpb * 32, sm_sel, s>>>(
                p, probes, out_d, out_i, out_cnt, sh.nq);
        else if (sh.k <= 64)
            dense_ivf_select_kernel<2><<<(sh.nq + wpb - 1) / wpb, wpb * 32, sm_sel, s>>>(
                p, probes, out_d, out_i, out_cnt, sh.nq);
        else if (sh.k <= 128)
            dense_ivf_select_kernel<4><<<(sh.nq + wpb - 1) / wpb, wpb * 32, sm_sel, s>>>(
                p, probes, out_d, out_i, out_cnt, sh.nq);
        else
            dense_ivf_select_kernel<8><<<(sh.nq + wpb - 1) / wpb, wpb * 32, sm_sel, s>>>(
                p, probes, out_d, out_i, out_cnt, sh.nq);
    } else if (dense) {
        const uint32_t n = dense->n;
        const size_t sm_sel = wpb * (p.Dp * 4 + 128 + 768 * 4);
        if (wide)  // inner-product quantizer (k = nprobe <= 32)
            dense_select_kernel<1, kIP><<<(sh.nq + wpb - 1) / wpb, wpb * 32, sm_sel, s>>>(
                dense->out, dense->ld, dense->nq, off_nrm, off_rows, queries, p.Dp, p.D, n, sh.nq,
                sh.k, out_d, out_i, dense->gsum);
        else if (sh.k <= 32)
            dense_select_kernel<1, kL2><<<(sh.nq + wpb - 1) / wpb, wpb * 32, sm_sel, s>>>(
                dense->out, dense->ld, dense->nq, off_nrm, off_rows, queries, p.Dp, p.D, n, sh.nq,
                sh.k, out_d, out_i, dense->gsum);
        else
            dense_select_kernel<8, kL2><<<(sh.nq + wpb - 1) / wpb, wpb * 32, sm_sel, s>>>(
                dense->out, dense->ld, dense->nq, off_nrm, off_rows, queries, p.Dp, p.D, n, sh.nq,
                sh.k, out_d, out_i, dense->gsum);
    } else {
        if (wide)
            refine_kernel<1, kIP, 1><<<(sh.nq + wpb - 1) / wpb, wpb * 32, wpb * (p.Dp * 4 + 256), s>>>(
                p, probes, out_d, out_i, out_cnt, sh.nq);
        else
            refine_kernel<1, kL2, 1><<<(sh.nq + wpb - 1) / wpb, wpb * 32, wpb * (p.Dp * 4 + 256), s>>>(
                p, probes, out_d, out_i, out_cnt, sh.nq);
    }
    count_launch();
    return cudaGetLastError();
}

}  // namespace bivf
