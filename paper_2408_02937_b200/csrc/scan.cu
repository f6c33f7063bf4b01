// The per-probe list scan + top-k (K3/K4) and the exact CUDA-core coarse
// quantizer (K2), sm_100a.
//
// Reference semantics reproduced (paths under /root/reference/proj):
//   ClusterIndex::search      src/ivf_index.cpp:262-298  (probe, offline scan, online scan)
//   l2_sqr / l2_sqr_strided   include/blockivf/distance.hpp:11-30 (bit-identical sums)
//   TopK + take_sorted        include/blockivf/topk.hpp:14-43  ((dist,id) lexicographic)
//   quantizer partial_sort    src/ivf_index.cpp:271-276   ((dist, cluster id) order)
//
// Design: queries are grouped by the list they probe, so one
// 32-vector group of a list is staged ONCE in shared memory (cp.async.bulk,
// mbarrier ring fed by a producer warp) and scored against every query of the
// tile held in shared memory: HBM/L2 bytes are shared across queries and the
// kernel is bound by the fp32 pipe, not by per-query bytes.  Work items are
// (list, query tile, group chunk), pulled from a device counter by a
// persistent grid.  Each consumer warp keeps a register top-k per query.
#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "launches.h"
#include "scan.cuh"
#include "scan_common.cuh"

namespace bivf {

namespace {

constexpr int kConsumerWarps = 4;
constexpr int kThreads = (kConsumerWarps + 1) * 32;
constexpr int kSlabDims = 128;       // dims per staged slab (16 KB at 32 slots)
constexpr int kItemRing = 2;
constexpr uint32_t kMaxStageBytesTotal = 64 * 1024;

struct ScanParams {
    uint32_t D, Dp, k, P, QT;
    // flat source
    const float* flat;
    uint32_t flat_n, flat_nq, flat_nch, flat_gc;
    // ivf source
    DevLists L;
    const uint32_t* snap_off;
    const uint32_t* snap_len;
    const uint32_t* gc;
    const uint32_t* nch;
    const uint32_t* qoff;
    const uint32_t* item_off;
    const uint32_t* n_items_ptr;
    const uint32_t* plist;
    uint32_t* item_ctr;
    uint32_t maxch;
    const float* queries;  // [nq][Dp]
    float* cand_d;
    long long* cand_i;
    uint32_t NS, nslab;
};

struct ItemDesc {
    uint32_t c, pair0, npairs, g0, g1, chunk, off, len;
    const uint32_t* pairs;  // nullptr in flat mode (pairs are pair0..pair0+npairs-1)
};

template <bool FLAT>
__device__ __forceinline__ ItemDesc decode_item(const ScanParams& p, uint32_t it) {
    ItemDesc d;
    if constexpr (FLAT) {
        const uint32_t tile = it / p.flat_nch, h = it - tile * p.flat_nch;
        d.c = 0;
        d.pair0 = tile * p.QT;
        d.npairs = min(p.QT, p.flat_nq - d.pair0);
        d.pairs = nullptr;
        const uint32_t ng = (p.flat_n + 31u) >> 5;
        d.g0 = h * p.flat_gc;
        d.g1 = min(ng, d.g0 + p.flat_gc);
        d.chunk = h;
        d.off = p.flat_n;
        d.len = 0;
    } else {
        // list owning item `it`: last c with item_off[c] <= it
        uint32_t lo = 0, hi = p.L.C;  // item_off has C+1 entries
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (p.item_off[mid] <= it) lo = mid;
            else hi = mid;
        }
        const uint32_t c = lo;
        const uint32_t local = it - p.item_off[c];
        const uint32_t nch = p.nch[c];
        const uint32_t tile = local / nch, h = local - tile * nch;
        d.c = c;
        const uint32_t q0 = p.qoff[c] + tile * p.QT;
        d.pairs = p.plist + q0;
        d.pair0 = 0;
        d.npairs = min(p.QT, p.qoff[c + 1] - q0);
        d.off = p.snap_off[c];
        d.len = p.snap_len[c];
        const uint32_t ng = ivf_ngroups(p.L, d.off, d.len);
        const uint32_t gc = p.gc[c];
        d.g0 = h * gc;
        d.g1 = min(ng, d.g0 + gc);
        d.chunk = h;
    }
    return d;
}

template <bool FLAT>
__device__ __forceinline__ GroupRef get_group(const ScanParams& p, const ItemDesc& d,
                                              uint32_t j) {
    if constexpr (FLAT) {
        GroupRef g;
        g.base = p.flat + (uint64_t)j * 32u * p.D;
        g.ids = nullptr;
        g.id0 = 32ll * j;
        g.nvalid = min(32u, p.flat_n - 32u * j);
        return g;
    } else {
        return ivf_group(p.L, d.c, d.off, d.len, j);
    }
}

template <int KPL, int M, bool FLAT>
__global__ void __launch_bounds__(kThreads) scan_kernel(const ScanParams p) {
    constexpr int QW = 8 / KPL;  // queries per consumer warp
    constexpr int K = 32 * KPL;
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t NS = p.NS;
    float* stages = reinterpret_cast<float*>(smem);
    const uint32_t stage_floats = kSlabDims * 32;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * stage_floats * 4);
    uint64_t* empty = full + NS;
    uint64_t* it_full = empty + NS;
    uint64_t* it_empty = it_full + kItemRing;
    int* ring = reinterpret_cast<int*>(it_empty + kItemRing);
    float* qreg = reinterpret_cast<float*>(smem + NS * stage_floats * 4 + 256);
    float* scr_d = qreg + kConsumerWarps * QW * p.Dp;
    long long* scr_i = reinterpret_cast<long long*>(scr_d + kConsumerWarps * QW * K);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        for (int s = 0; s < kItemRing; ++s) {
            mbar_init(&it_full[s], 1);
            mbar_init(&it_empty[s], kConsumerWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();

    const uint32_t n_items = FLAT ? ((p.flat_nq + p.QT - 1) / p.QT) * p.flat_nch : *p.n_items_ptr;

    if (warp == kConsumerWarps) {
        // ------------------------------------------------ producer (one lane)
        if (lane != 0) return;
        uint32_t unit = 0;
        for (uint32_t seq = 0;; ++seq) {
            const uint32_t rs = seq % kItemRing;
            mbar_wait(&it_empty[rs], ((seq / kItemRing) & 1) ^ 1);
            uint32_t it = atomicAdd(p.item_ctr, 1u);
            const int v = it < n_items ? (int)it : -1;
            ring[rs] = v;
            mbar_arrive(&it_full[rs]);
            if (v < 0) break;
            const ItemDesc d = decode_item<FLAT>(p, it);
            for (uint32_t j = d.g0; j < d.g1; ++j) {
                const GroupRef g = get_group<FLAT>(p, d, j);
                for (uint32_t s = 0; s < p.nslab; ++s) {
                    const uint32_t st = unit % NS;
                    mbar_wait(&empty[st], ((unit / NS) & 1) ^ 1);
                    const uint32_t d0 = s * kSlabDims;
                    const uint32_t nd = min((uint32_t)kSlabDims, p.D - d0);
                    const uint32_t bytes = nd * 32u * 4u;
                    mbar_arrive_expect_tx(&full[st], bytes);
                    bulk_g2s(stages + st * stage_floats, g.base + (uint64_t)d0 * 32u, bytes,
                             &full[st]);
                    ++unit;
                }
            }
        }
        return;
    }

    // ---------------------------------------------------- consumers
    float* myq = qreg + warp * QW * p.Dp;
    uint32_t unit = 0;
    for (uint32_t seq = 0;; ++seq) {
        const uint32_t rs = seq % kItemRing;
        mbar_wait(&it_full[rs], (seq / kItemRing) & 1);
        const int v = ring[rs];
        __syncwarp();
        if (lane == 0) mbar_arrive(&it_empty[rs]);
        if (v < 0) break;
        const ItemDesc d = decode_item<FLAT>(p, (uint32_t)v);

        const uint32_t nsub = (d.npairs + QW - 1) / QW;
        const uint32_t wps = nsub >= 3 ? 1u : (nsub == 2 ? 2u : 4u);
        const uint32_t sub = warp / wps, part = warp % wps;
        const bool active = sub < nsub;
        const uint32_t qbeg = sub * QW;
        const uint32_t nqw = active ? min((uint32_t)QW, d.npairs - qbeg) : 0u;

        // stage this warp's queries (pair -> query row) into its smem region
        uint32_t mypair[QW];
#pragma unroll
        for (int qi = 0; qi < QW; ++qi) {
            uint32_t pr = 0;
            if (qi < (int)nqw) pr = FLAT ? d.pair0 + qbeg + qi : d.pairs[qbeg + qi];
            mypair[qi] = pr;
            if (qi < (int)nqw) {
                const uint32_t qrow = FLAT ? pr : pr / p.P;
                const float4* src = reinterpret_cast<const float4*>(p.queries + (uint64_t)qrow * p.Dp);
                float4* dst = reinterpret_cast<float4*>(myq + qi * p.Dp);
                for (uint32_t i = lane; i < p.Dp / 4; i += 32) dst[i] = src[i];
            }
        }
        __syncwarp();

        WarpTopK<KPL> tk[QW];
#pragma unroll
        for (int qi = 0; qi < QW; ++qi) tk[qi].init();

        for (uint32_t j = d.g0; j < d.g1; ++j) {
            const bool mine = active && ((j - d.g0) % wps == part);
            float acc[QW];
#pragma unroll
            for (int qi = 0; qi < QW; ++qi) acc[qi] = 0.f;
            for (uint32_t s = 0; s < p.nslab; ++s) {
                const uint32_t st = unit % NS;
                mbar_wait(&full[st], (unit / NS) & 1);
                if (mine) {
                    const float* xs = stages + st * stage_floats;
                    const uint32_t d0 = s * kSlabDims;
                    const uint32_t nd = min((uint32_t)kSlabDims, p.D - d0);
                    uint32_t dd = 0;
                    for (; dd + 4 <= nd; dd += 4) {
                        const float x0 = xs[(dd + 0) * 32 + lane];
                        const float x1 = xs[(dd + 1) * 32 + lane];
                        const float x2 = xs[(dd + 2) * 32 + lane];
                        const float x3 = xs[(dd + 3) * 32 + lane];
                        // all QW chains every step (rows >= nqw hold stale data whose
                        // results are ignored): no per-query branch, so the QW
                        // independent sequential sums interleave (each chain keeps
                        // its ascending-d order, the reference's bits)
                        float4 qv[QW];
#pragma unroll
                        for (int qi = 0; qi < QW; ++qi)
                            qv[qi] = *reinterpret_cast<const float4*>(myq + qi * p.Dp + d0 + dd);
#pragma unroll
                        for (int qi = 0; qi < QW; ++qi) acc[qi] = dstep<M>(acc[qi], qv[qi].x, x0);
#pragma unroll
                        for (int qi = 0; qi < QW; ++qi) acc[qi] = dstep<M>(acc[qi], qv[qi].y, x1);
#pragma unroll
                        for (int qi = 0; qi < QW; ++qi) acc[qi] = dstep<M>(acc[qi], qv[qi].z, x2);
#pragma unroll
                        for (int qi = 0; qi < QW; ++qi) acc[qi] = dstep<M>(acc[qi], qv[qi].w, x3);
                    }
                    for (; dd < nd; ++dd) {
                        const float x = xs[dd * 32 + lane];
#pragma unroll
                        for (int qi = 0; qi < QW; ++qi)
                            if (qi < (int)nqw) acc[qi] = dstep<M>(acc[qi], myq[qi * p.Dp + d0 + dd], x);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[st]);
                ++unit;
            }
            if (mine) {
                const GroupRef g = get_group<FLAT>(p, d, j);
                const bool valid = (uint32_t)lane < g.nvalid;
#pragma unroll
                for (int qi = 0; qi < QW; ++qi) {
                    if (qi >= (int)nqw) continue;
                    const float dist = dfinal<M>(acc[qi]);
                    bool pass = valid && dist <= tk[qi].thr_d;
                    unsigned m = __ballot_sync(0xffffffffu, pass);
                    if (!m) continue;
                    long long myid = 0;
                    if (pass) myid = g.ids ? g.ids[lane] : g.id0 + lane;
                    while (m) {
                        const int src = __ffs(m) - 1;
                        m &= m - 1;
                        const float cd = __shfl_sync(0xffffffffu, dist, src);
                        const long long ci = __shfl_sync(0xffffffffu, myid, src);
                        if (tk[qi].admits(cd, ci)) tk[qi].insert(cd, ci, (int)p.k, lane);
                    }
                }
            }
        }

        // merge the parts of a subset (warps that split the groups).  Warps may
        // already be in different items, so each barrier id has ONE fixed warp
        // set: id 1 = warps {0,1}, id 2 = {2,3} (wps 2), id 3 = {0,1,2,3} (wps 4).
        const uint32_t bar_id = wps == 4 ? 3u : 1u + sub;
        if (active && wps > 1) {
            float* sd = scr_d + warp * QW * K;
            long long* si = scr_i + warp * QW * K;
            if (part != 0) {
#pragma unroll
                for (int qi = 0; qi < QW; ++qi)
#pragma unroll
                    for (int r = 0; r < KPL; ++r) {
                        sd[qi * K + r * 32 + lane] = tk[qi].d[r];
                        si[qi * K + r * 32 + lane] = tk[qi].id[r];
                    }
            }
            asm volatile("barrier.sync %0, %1;" ::"r"(bar_id), "r"(wps * 32) : "memory");
            if (part == 0) {
                for (uint32_t w2 = 1; w2 < wps; ++w2) {
                    const float* od = scr_d + (warp + w2) * QW * K;
                    const long long* oi = scr_i + (warp + w2) * QW * K;
#pragma unroll
                    for (int qi = 0; qi < QW; ++qi) {
                        if (qi >= (int)nqw) continue;
                        for (uint32_t e0 = 0; e0 < p.k; e0 += 32) {
                            const uint32_t e = e0 + lane;
                            const float cd = e < p.k ? od[qi * K + e] : 0.f;
                            const long long ci = e < p.k ? oi[qi * K + e] : -1;
                            bool pass = e < p.k && ci >= 0 && tk[qi].admits(cd, ci);
                            unsigned m = __ballot_sync(0xffffffffu, pass);
                            while (m) {
                                const int src = __ffs(m) - 1;
                                m &= m - 1;
                                const float bd = __shfl_sync(0xffffffffu, cd, src);
                                const long long bi = __shfl_sync(0xffffffffu, ci, src);
                                if (tk[qi].admits(bd, bi)) tk[qi].insert(bd, bi, (int)p.k, lane);
                            }
                        }
                    }
                }
            }
            asm volatile("barrier.sync %0, %1;" ::"r"(bar_id), "r"(wps * 32) : "memory");
        }

        // write the (pair, chunk) candidate runs
        if (active && part == 0) {
#pragma unroll
            for (int qi = 0; qi < QW; ++qi) {
                if (qi >= (int)nqw) continue;
                const uint64_t base = ((uint64_t)mypair[qi] * p.maxch + d.chunk) * p.k;
#pragma unroll
                for (int r = 0; r < KPL; ++r) {
                    const uint32_t e = r * 32 + lane;
                    if (e < p.k) {
                        p.cand_d[base + e] = tk[qi].d[r];
                        p.cand_i[base + e] = tk[qi].id[r];
                    }
                }
            }
        }
    }
}

// ------------------------------------------------------------------ merge
// One warp per query: fold every (probe, chunk) run into one top-k.
template <int KPL, bool FLAT>
__global__ void merge_kernel(uint32_t nq, uint32_t P, uint32_t maxch, uint32_t k,
                             const long long* probes, const uint32_t* nch, uint32_t flat_nch,
                             const float* cand_d, const long long* cand_i, float* out_d,
                             long long* out_i, uint32_t* out_cnt) {
    const uint32_t q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (q >= nq) return;
    WarpTopK<KPL> tk;
    tk.init();
    for (uint32_t pi = 0; pi < P; ++pi) {
        const uint32_t n = FLAT ? flat_nch : nch[(uint32_t)probes[(uint64_t)q * P + pi]];
        const uint64_t pair = (uint64_t)q * P + pi;
        for (uint32_t h = 0; h < n; ++h) {
            const uint64_t base = (pair * maxch + h) * k;
            for (uint32_t e0 = 0; e0 < k; e0 += 32) {
                const uint32_t e = e0 + lane;
                const float cd = e < k ? cand_d[base + e] : 0.f;
                const long long ci = e < k ? cand_i[base + e] : -1;
                const bool pass = e < k && ci >= 0 && tk.admits(cd, ci);
                unsigned m = __ballot_sync(0xffffffffu, pass);
                if (!m) break;  // runs are sorted: nothing later in this run can enter
                while (m) {
                    const int src = __ffs(m) - 1;
                    m &= m - 1;
                    const float bd = __shfl_sync(0xffffffffu, cd, src);
                    const long long bi = __shfl_sync(0xffffffffu, ci, src);
                    if (tk.admits(bd, bi)) tk.insert(bd, bi, (int)k, lane);
                }
            }
        }
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int r = 0; r < KPL; ++r) {
        const uint32_t e = r * 32 + lane;
        const bool ok = e < k && tk.id[r] >= 0;
        cnt += __popc(__ballot_sync(0xffffffffu, ok));
        if (e < k) {
            out_d[(uint64_t)q * k + e] = tk.d[r];
            out_i[(uint64_t)q * k + e] = tk.id[r];
        }
    }
    if (lane == 0 && out_cnt) out_cnt[q] = cnt;
}

// ------------------------------------------------------------------ plan
__global__ void plan_snapshot(DevLists L, uint32_t maxch, uint32_t gcmin, PlanBufs B) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= L.C) return;
    uint32_t off, len;
    uint64_t start, row;
    snapshot_list(L, c, off, len, start, row);
    B.snap_off[c] = off;
    B.snap_len[c] = len;
    B.snap_start[c] = start;
    B.snap_row[c] = row;
    const uint32_t ng = ivf_ngroups(L, off, len);
    uint32_t g = max(gcmin, (ng + maxch - 1) / maxch);
    B.gc[c] = g;
    B.nch[c] = (ng + g - 1) / g;
    B.cnt[c] = 0;
}

// pairs i = q * P + rank with rank in [lo, hi) only (the ranked plans of the
// two-phase TC scan; [0, P) = every pair)
__global__ void plan_count(const long long* probes, uint32_t npairs, uint32_t P, uint32_t lo,
                           uint32_t hi, uint32_t* cnt, uint32_t* ppos) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npairs) return;
    const uint32_t r = i % P;
    if (r < lo || r >= hi) return;
    ppos[i] = atomicAdd(&cnt[(uint32_t)probes[i]], 1u);
}

// single CTA of 1024 threads: exclusive scans over lists
__device__ __forceinline__ void plan_scan_block(uint32_t C, uint32_t QT, const uint32_t* cnt,
                                                const uint32_t* nch, uint32_t* qoff,
                                                uint32_t* item_off, uint32_t* n_items,
                                                uint32_t* item_ctr) {
    __shared__ uint32_t wq[32], wi[32];
    __shared__ uint32_t carry_q, carry_i;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    if (t == 0) {
        carry_q = 0;
        carry_i = 0;
    }
    __syncthreads();
    for (uint32_t base = 0; base < C; base += 1024) {
        const uint32_t c = base + t;
        const uint32_t a = c < C ? cnt[c] : 0u;
        const uint32_t b = c < C ? ((a + QT - 1) / QT) * nch[c] : 0u;
        uint32_t xa = a, xb = b;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t ya = __shfl_up_sync(0xffffffffu, xa, o);
            const uint32_t yb = __shfl_up_sync(0xffffffffu, xb, o);
            if (lane >= o) {
                xa += ya;
                xb += yb;
            }
        }
        if (lane == 31) {
            wq[w] = xa;
            wi[w] = xb;
        }
        __syncthreads();
        if (w == 0) {
            uint32_t sa = wq[lane], sb = wi[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t ya = __shfl_up_sync(0xffffffffu, sa, o);
                const uint32_t yb = __shfl_up_sync(0xffffffffu, sb, o);
                if (lane >= o) {
                    sa += ya;
                    sb += yb;
                }
            }
            wq[lane] = sa;
            wi[lane] = sb;
        }
        __syncthreads();
        const uint32_t pre_a = (w ? wq[w - 1] : 0u) + xa - a + carry_q;
        const uint32_t pre_b = (w ? wi[w - 1] : 0u) + xb - b + carry_i;
        if (c < C) {
            qoff[c] = pre_a;
            item_off[c] = pre_b;
        }
        __syncthreads();
        if (t == 0) {
            carry_q += wq[31];
            carry_i += wi[31];
        }
        __syncthreads();
    }
    if (t == 0) {
        qoff[C] = carry_q;
        item_off[C] = carry_i;
        *n_items = carry_i;
        *item_ctr = 0;
    }
}

__global__ void __launch_bounds__(1024) plan_scan(uint32_t C, uint32_t QT, const uint32_t* cnt,
                                                  const uint32_t* nch, uint32_t* qoff,
                                                  uint32_t* item_off, uint32_t* n_items,
                                                  uint32_t* item_ctr) {
    plan_scan_block(C, QT, cnt, nch, qoff, item_off, n_items, item_ctr);
}

// The whole plan (snapshot, count, scan, scatter) in ONE 1024-thread CTA for
// small batches: the four-launch chain costs more than the work there.
__global__ void __launch_bounds__(1024) plan_fused(DevLists L, uint32_t maxch, uint32_t gcmin,
                                                   const long long* probes, uint32_t npairs,
                                                   uint32_t P, uint32_t lo, uint32_t hi,
                                                   int snapshot, uint32_t QT, PlanBufs B) {
    const uint32_t t = threadIdx.x;
    if (snapshot) {
        // only the lists some pair of the batch probes (any rank: a later ranked
        // plan with snapshot = 0 reuses these) are snapshotted; the others get no
        // work items and nothing after the plan reads their snapshot
        for (uint32_t c = t; c < L.C; c += 1024) {
            B.cnt[c] = 0;
            B.nch[c] = 0;
        }
        __syncthreads();
        for (uint32_t i = t; i < npairs; i += 1024) B.nch[(uint32_t)probes[i]] = 1u;
        __syncthreads();
        for (uint32_t c = t; c < L.C; c += 1024) {
            if (!B.nch[c]) continue;
            uint32_t off, len;
            uint64_t start, row;
            snapshot_list(L, c, off, len, start, row);
            B.snap_off[c] = off;
            B.snap_len[c] = len;
            B.snap_start[c] = start;
            B.snap_row[c] = row;
            const uint32_t ng = ivf_ngroups(L, off, len);
            const uint32_t g = max(gcmin, (ng + maxch - 1) / maxch);
            B.gc[c] = g;
            B.nch[c] = (ng + g - 1) / g;
        }
    } else {
        for (uint32_t c = t; c < L.C; c += 1024) B.cnt[c] = 0;
    }
    __syncthreads();
    for (uint32_t i = t; i < npairs; i += 1024) {
        const uint32_t r = i % P;
        if (r >= lo && r < hi) B.ppos[i] = atomicAdd(&B.cnt[(uint32_t)probes[i]], 1u);
    }
    __syncthreads();
    plan_scan_block(L.C, QT, B.cnt, B.nch, B.qoff, B.item_off, B.n_items, B.item_ctr);
    __syncthreads();
    for (uint32_t i = t; i < npairs; i += 1024) {
        const uint32_t r = i % P;
        if (r >= lo && r < hi) B.plist[B.qoff[(uint32_t)probes[i]] + B.ppos[i]] = i;
    }
}

__global__ void plan_scatter(const long long* probes, uint32_t npairs, uint32_t P, uint32_t lo,
                             uint32_t hi, const uint32_t* qoff, const uint32_t* ppos,
                             uint32_t* plist) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npairs) return;
    const uint32_t r = i % P;
    if (r < lo || r >= hi) return;
    plist[qoff[(uint32_t)probes[i]] + ppos[i]] = i;
}

__global__ void all_probes_kernel(long long* probes, uint32_t nq, uint32_t C) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < (uint64_t)nq * C) probes[i] = (long long)(i % C);
}

__global__ void interleave_kernel(const float* rows, uint32_t n, uint32_t D, float* out) {
    // out[(i/32)*32*D + d*32 + i%32] = rows[i*D + d]; padded slots -> 0
    const uint64_t ngroups = (n + 31u) / 32u;
    const uint64_t total = ngroups * 32ull * D;
    for (uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total;
         o += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t g = o / (32ull * D);
        const uint64_t r = o - g * 32ull * D;
        const uint32_t d = (uint32_t)(r / 32u), s = (uint32_t)(r % 32u);
        const uint64_t i = g * 32u + s;
        out[o] = i < n ? rows[i * D + d] : 0.f;
    }
}

__global__ void pad_rows_kernel(const float* rows, uint32_t n, uint32_t D, uint32_t Dp,
                                float* out) {
    const uint64_t total = (uint64_t)n * Dp;
    for (uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total;
         o += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = o / Dp;
        const uint32_t d = (uint32_t)(o - i * Dp);
        out[o] = d < D ? rows[i * D + d] : 0.f;
    }
}

uint32_t stages_for(uint32_t D) {
    (void)D;
    return kMaxStageBytesTotal / (kSlabDims * 32 * 4);  // 4 stages of 16 KB
}

size_t smem_bytes(int kpl, uint32_t Dp, uint32_t NS) {
    const int QW = 8 / kpl;
    const int K = 32 * kpl;
    return (size_t)NS * kSlabDims * 32 * 4 + 256 + (size_t)kConsumerWarps * QW * Dp * 4 +
           (size_t)kConsumerWarps * QW * K * (4 + 8);
}

template <int KPL, int M, bool FLAT>
cudaError_t launch_scan_t(const ScanParams& p, int num_sms, cudaStream_t s) {
    const size_t sm = smem_bytes(KPL, p.Dp, p.NS);
    static bool attr_set = false;  // per instantiation
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(scan_kernel<KPL, M, FLAT>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             227 * 1024);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, scan_kernel<KPL, M, FLAT>, kThreads,
                                                  sm);
    per_sm = std::max(1, per_sm);
    uint32_t grid = (uint32_t)(num_sms * per_sm);
    if (FLAT) {
        const uint32_t n_items = ((p.flat_nq + p.QT - 1) / p.QT) * p.flat_nch;
        grid = std::min(grid, std::max(1u, n_items));
    }
    scan_kernel<KPL, M, FLAT><<<grid, kThreads, sm, s>>>(p);
    count_launch();
    return cudaGetLastError();
}

template <bool FLAT>
cudaError_t launch_scan(int kpl, int metric, const ScanParams& p, int num_sms, cudaStream_t s) {
#define BIVF_SCAN_CASE(K_)                                                          \
    case K_:                                                                        \
        return metric == kIP ? launch_scan_t<K_, kIP, FLAT>(p, num_sms, s)           \
                             : launch_scan_t<K_, kL2, FLAT>(p, num_sms, s);
    switch (kpl) {
        BIVF_SCAN_CASE(1)
        BIVF_SCAN_CASE(2)
        BIVF_SCAN_CASE(4)
        BIVF_SCAN_CASE(8)
        default:
            return cudaErrorInvalidValue;
    }
#undef BIVF_SCAN_CASE
}

template <bool FLAT>
cudaError_t launch_merge(int kpl, uint32_t nq, uint32_t P, uint32_t maxch, uint32_t k,
                         const long long* probes, const uint32_t* nch, uint32_t flat_nch,
                         const float* cd, const long long* ci, float* od, long long* oi,
                         uint32_t* oc, cudaStream_t s) {
    const uint32_t wpb = 4;
    const uint32_t grid = (nq + wpb - 1) / wpb;
    if (nq == 0) return cudaSuccess;
    count_launch();
    switch (kpl) {
        case 1:
            merge_kernel<1, FLAT><<<grid, wpb * 32, 0, s>>>(nq, P, maxch, k, probes, nch, flat_nch,
                                                           cd, ci, od, oi, oc);
            break;
        case 2:
            merge_kernel<2, FLAT><<<grid, wpb * 32, 0, s>>>(nq, P, maxch, k, probes, nch, flat_nch,
                                                           cd, ci, od, oi, oc);
            break;
        case 4:
            merge_kernel<4, FLAT><<<grid, wpb * 32, 0, s>>>(nq, P, maxch, k, probes, nch, flat_nch,
                                                           cd, ci, od, oi, oc);
            break;
        case 8:
            merge_kernel<8, FLAT><<<grid, wpb * 32, 0, s>>>(nq, P, maxch, k, probes, nch, flat_nch,
                                                           cd, ci, od, oi, oc);
            break;
        default:
            return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace

int kpl_for(uint32_t k) {
    if (k <= 32) return 1;
    if (k <= 64) return 2;
    if (k <= 128) return 4;
    if (k <= 256) return 8;
    return 0;
}

uint32_t qt_for(uint32_t k, uint32_t D) {
    (void)D;
    const int kpl = kpl_for(k);
    return kpl ? (uint32_t)(kConsumerWarps * (8 / kpl)) : 0u;
}

cudaError_t launch_flat_topk(const float* flat_il, uint32_t n, uint32_t D, const float* queries,
                             uint32_t nq, uint32_t k, int metric, uint32_t nch, float* cand_d,
                             long long* cand_i, float* out_d, long long* out_i, uint32_t* out_cnt,
                             uint32_t* item_ctr, int num_sms, cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    const int kpl = kpl_for(k);
    if (!kpl) return cudaErrorInvalidValue;
    ScanParams p{};
    p.D = D;
    p.Dp = pad4(D);
    p.k = k;
    p.P = 1;
    p.QT = qt_for(k, D);
    p.flat = flat_il;
    p.flat_n = n;
    p.flat_nq = nq;
    const uint32_t ng = (n + 31) / 32;
    nch = std::max(1u, std::min(nch, ng));
    p.flat_gc = (ng + nch - 1) / nch;
    p.flat_nch = (ng + p.flat_gc - 1) / p.flat_gc;
    p.item_ctr = item_ctr;
    p.maxch = p.flat_nch;
    p.queries = queries;
    p.cand_d = cand_d;
    p.cand_i = cand_i;
    p.NS = stages_for(D);
    p.nslab = (D + kSlabDims - 1) / kSlabDims;
    cudaError_t e = cudaMemsetAsync(item_ctr, 0, sizeof(uint32_t), s);
    if (e != cudaSuccess) return e;
    e = launch_scan<true>(kpl, metric, p, num_sms, s);
    if (e != cudaSuccess) return e;
    return launch_merge<true>(kpl, nq, 1, p.maxch, k, nullptr, nullptr, p.flat_nch, cand_d, cand_i,
                              out_d, out_i, out_cnt, s);
}

cudaError_t launch_plan(const DevLists& L, const PlanBufs& B, const long long* probes,
                        const SearchShape& sh, cudaStream_t s) {
    return launch_plan_ranked(L, B, probes, sh, 0, sh.P, true, s);
}

cudaError_t launch_plan_ranked(const DevLists& L, const PlanBufs& B, const long long* probes,
                               const SearchShape& sh, uint32_t lo, uint32_t hi, bool snapshot,
                               cudaStream_t s) {
    const uint32_t npairs = sh.nq * sh.P;
    if (npairs <= 8192 && L.C <= 8192) {  // small batch: one launch
        plan_fused<<<1, 1024, 0, s>>>(L, sh.maxch, sh.gcmin, probes, npairs, sh.P, lo, hi,
                                      snapshot ? 1 : 0, sh.QT, B);
        count_launch(1);
        return cudaGetLastError();
    }
    if (snapshot) {
        plan_snapshot<<<(L.C + 255) / 256, 256, 0, s>>>(L, sh.maxch, sh.gcmin, B);
    } else {
        cudaError_t e = cudaMemsetAsync(B.cnt, 0, (size_t)L.C * 4, s);
        if (e != cudaSuccess) return e;
    }
    plan_count<<<(npairs + 255) / 256, 256, 0, s>>>(probes, npairs, sh.P, lo, hi, B.cnt, B.ppos);
    plan_scan<<<1, 1024, 0, s>>>(L.C, sh.QT, B.cnt, B.nch, B.qoff, B.item_off, B.n_items,
                                 B.item_ctr);
    plan_scatter<<<(npairs + 255) / 256, 256, 0, s>>>(probes, npairs, sh.P, lo, hi, B.qoff,
                                                      B.ppos, B.plist);
    count_launch(snapshot ? 4 : 3);
    return cudaGetLastError();
}

cudaError_t launch_ivf_search(const DevLists& L, const PlanBufs& B, const long long* probes,
                              const float* queries, const SearchShape& sh, float* cand_d,
                              long long* cand_i, float* out_d, long long* out_i,
                              uint32_t* out_cnt, int num_sms, cudaStream_t s,
                              cudaEvent_t ev_scan0, cudaEvent_t ev_scan1) {
    if (sh.nq == 0) return cudaSuccess;
    const int kpl = kpl_for(sh.k);
    if (!kpl) return cudaErrorInvalidValue;
    const uint32_t npairs = sh.nq * sh.P;
    plan_snapshot<<<(L.C + 255) / 256, 256, 0, s>>>(L, sh.maxch, sh.gcmin, B);
    plan_count<<<(npairs + 255) / 256, 256, 0, s>>>(probes, npairs, sh.P, 0, sh.P, B.cnt, B.ppos);
    plan_scan<<<1, 1024, 0, s>>>(L.C, sh.QT, B.cnt, B.nch, B.qoff, B.item_off, B.n_items,
                                 B.item_ctr);
    plan_scatter<<<(npairs + 255) / 256, 256, 0, s>>>(probes, npairs, sh.P, 0, sh.P, B.qoff,
                                                      B.ppos, B.plist);
    count_launch(4);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    ScanParams p{};
    p.D = L.D;
    p.Dp = pad4(L.D);
    p.k = sh.k;
    p.P = sh.P;
    p.QT = sh.QT;
    p.L = snapshot_view(L, B);
    p.snap_off = B.snap_off;
    p.snap_len = B.snap_len;
    p.gc = B.gc;
    p.nch = B.nch;
    p.qoff = B.qoff;
    p.item_off = B.item_off;
    p.n_items_ptr = B.n_items;
    p.plist = B.plist;
    p.item_ctr = B.item_ctr;
    p.maxch = sh.maxch;
    p.queries = queries;
    p.cand_d = cand_d;
    p.cand_i = cand_i;
    p.NS = stages_for(L.D);
    p.nslab = (L.D + kSlabDims - 1) / kSlabDims;
    if (ev_scan0) cudaEventRecord(ev_scan0, s);
    e = launch_scan<false>(kpl, sh.metric, p, num_sms, s);
    if (e != cudaSuccess) return e;
    if (ev_scan1) cudaEventRecord(ev_scan1, s);
    return launch_merge<false>(kpl, sh.nq, sh.P, sh.maxch, sh.k, probes, B.nch, 0, cand_d, cand_i,
                               out_d, out_i, out_cnt, s);
}

cudaError_t launch_all_probes(long long* probes, uint32_t nq, uint32_t C, cudaStream_t s) {
    const uint64_t total = (uint64_t)nq * C;
    if (!total) return cudaSuccess;
    all_probes_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(probes, nq, C);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_interleave(const float* rows, uint32_t n, uint32_t D, float* out,
                              cudaStream_t s) {
    if (!n) return cudaSuccess;
    interleave_kernel<<<1184, 256, 0, s>>>(rows, n, D, out);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_pad_rows(const float* rows, uint32_t n, uint32_t D, uint32_t Dp, float* out,
                            cudaStream_t s) {
    if (!n) return cudaSuccess;
    pad_rows_kernel<<<1184, 256, 0, s>>>(rows, n, D, Dp, out);
    count_launch();
    return cudaGetLastError();
}

}  // namespace bivf
