// Maintenance kernels: in-place rearrangement data moves (Alg. 3, K7),
// delete (K6: locate + tail-into-hole compaction moves), the multi-GPU top-k
// merge (K8) and small glue kernels.  sm_100a.
//
// Reference semantics:
//   swap_blocks data part       src/ivf_index.cpp:381-384 (save_to_scratch / copy_block_data / restore)
//   delete                      none in the reference; rules: DESIGN.md §Delete
// Moves are planned on the host mirror.  Concurrent searches are never fenced:
// new versions of the touched blocks / segments are built in storage no
// published state references (scratch blocks past the pool, free offline
// regions), published per list through the DevLists seqlock
// (publish_lists_kernel), and the old storage is reused only after a grace
// period (GpuIndex::grace).  The in-place gather/scatter kernels below remain
// for the quiescent fallback path.
#include <algorithm>

#include "common.cuh"
#include "launches.h"
#include "maint.cuh"

namespace bivf {

namespace {

__global__ void make_asg_kernel(const long long* nearest, const long long* ids, uint32_t n,
                                uint32_t* asg) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) asg[i] = ids[i] < 0 ? 0xffffffffu : (uint32_t)nearest[i];
}

// whole-block moves: phase 0 src -> scratch[m], phase 1 scratch[m] -> dst
__global__ void block_move_kernel(float* arena, long long* bids, uint64_t PS, uint32_t T,
                                  const int32_t* src, const int32_t* dst, uint32_t nmoves,
                                  float* scr_pay, long long* scr_ids, int phase) {
    const uint32_t m = blockIdx.y;
    if (m >= nmoves) return;
    const uint64_t b = phase == 0 ? (uint64_t)src[m] : (uint64_t)dst[m];
    float* blk_pay = arena + b * PS;
    long long* blk_ids = bids ? bids + b * T : nullptr;
    float* sp = scr_pay + (uint64_t)m * PS;
    long long* si = scr_ids ? scr_ids + (uint64_t)m * T : nullptr;
    const float4* from4 = reinterpret_cast<const float4*>(phase == 0 ? blk_pay : sp);
    float4* to4 = reinterpret_cast<float4*>(phase == 0 ? sp : blk_pay);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < PS / 4;
         i += (uint64_t)gridDim.x * blockDim.x)
        to4[i] = from4[i];
    if (!bids) return;  // payload-only move (the scan mirror)
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < T;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (phase == 0) si[i] = blk_ids[i];
        else blk_ids[i] = si[i];
    }
}

// slot moves (delete compaction).  A slot address is the float offset of its
// dimension-0 element within its pool (offline segments or arena; bit 63
// selects the arena) and the index of its id.
__device__ __forceinline__ float* slot_pay(float* off_pay, float* arena, uint64_t a) {
    return (a >> 63) ? arena + (a & ~(1ull << 63)) : off_pay + a;
}
__device__ __forceinline__ long long* slot_id(long long* off_ids, long long* bids, uint64_t a) {
    return (a >> 63) ? bids + (a & ~(1ull << 63)) : off_ids + a;
}

__global__ void slot_move_kernel(float* off_pay, long long* off_ids, float* arena,
                                 long long* bids, uint32_t D, const uint64_t* pay_addr,
                                 const uint64_t* id_addr, uint32_t nmoves, float* scr_pay,
                                 long long* scr_ids, int phase) {
    // pay_addr/id_addr: [2*nmoves] = src..., dst...
    const uint64_t total = (uint64_t)nmoves * D;
    for (uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total;
         o += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t m = (uint32_t)(o / D), d = (uint32_t)(o - (uint64_t)m * D);
        if (phase == 0) {
            scr_pay[o] = slot_pay(off_pay, arena, pay_addr[m])[(uint64_t)d * 32u];
            if (d == 0) scr_ids[m] = *slot_id(off_ids, bids, id_addr[m]);
        } else {
            slot_pay(off_pay, arena, pay_addr[nmoves + m])[(uint64_t)d * 32u] = scr_pay[o];
            if (d == 0) *slot_id(off_ids, bids, id_addr[nmoves + m]) = scr_ids[m];
        }
    }
}

__global__ void clear_ids_kernel(long long* off_ids, long long* bids, const uint64_t* id_addr,
                                 uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) *slot_id(off_ids, bids, id_addr[i]) = -1;
}

__global__ void set_u32_kernel(uint32_t* arr, const uint32_t* idx, const uint32_t* val,
                               uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) arr[idx[i]] = val[i];
}

// Copy-on-write block copies (disjoint source / destination sets: pool
// blocks <-> scratch blocks past the pool): n copies of `bytes` each (a
// multiple of 8), block x at base + x * bytes.
__global__ void copy_blocks_kernel(char* base, uint64_t bytes, const int32_t* src,
                                   const int32_t* dst, uint32_t n) {
    const uint32_t m = blockIdx.y;
    if (m >= n) return;
    const char* from = base + (uint64_t)src[m] * bytes;
    char* to = base + (uint64_t)dst[m] * bytes;
    if ((bytes & 15) == 0) {
        const uint4* f = reinterpret_cast<const uint4*>(from);
        uint4* t = reinterpret_cast<uint4*>(to);
        for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < bytes / 16;
             i += (uint64_t)gridDim.x * blockDim.x)
            t[i] = f[i];
    } else {
        const uint2* f = reinterpret_cast<const uint2*>(from);
        uint2* t = reinterpret_cast<uint2*>(to);
        for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < bytes / 8;
             i += (uint64_t)gridDim.x * blockDim.x)
            t[i] = f[i];
    }
}

// Publish new versions of lists (DevLists seqlock): ver odd, the fields, ver
// even.  Everything the new versions point to was written by earlier work on
// this stream.  A null field array leaves that field unchanged.
__global__ void publish_lists_kernel(uint32_t n, const uint32_t* idx, const uint64_t* start,
                                     const uint32_t* count, const uint64_t* row,
                                     const uint32_t* len, uint64_t* L_start, uint32_t* L_count,
                                     uint64_t* L_row, uint32_t* L_len, uint32_t* L_ver) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t c = idx[i];
    const uint32_t v = L_ver[c];
    *reinterpret_cast<volatile uint32_t*>(L_ver + c) = v + 1;
    __threadfence();
    if (start) *reinterpret_cast<volatile uint64_t*>(L_start + c) = start[i];
    if (count) *reinterpret_cast<volatile uint32_t*>(L_count + c) = count[i];
    if (row) *reinterpret_cast<volatile uint64_t*>(L_row + c) = row[i];
    if (len) *reinterpret_cast<volatile uint32_t*>(L_len + c) = len[i];
    __threadfence();
    st_release_u32(L_ver + c, v + 2);
}

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}

// locate: every live id (offline slots, then pool slots) probed against the
// request hash table; a hit records the slot's global address.
__global__ void locate_kernel(const long long* ids, uint64_t nslots, uint64_t arena_flag,
                              const long long* hkeys, const uint32_t* hvals, uint32_t hmask,
                              uint64_t* loc) {
    for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nslots;
         s += (uint64_t)gridDim.x * blockDim.x) {
        const long long id = ids[s];
        if (id < 0) continue;
        uint32_t h = (uint32_t)mix64((uint64_t)id) & hmask;
        for (;;) {
            const long long k = hkeys[h];
            if (k < 0) break;
            if (k == id) {
                loc[hvals[h]] = s | arena_flag;
                break;
            }
            h = (h + 1) & hmask;
        }
    }
}

// K8: merge G shard runs per query ([G][nq][k]) into the global top-k.
template <int KPL>
__global__ void merge_shards_kernel(const float* dists, const long long* ids, uint32_t G,
                                    uint32_t nq, uint32_t k, float* out_d, long long* out_i,
                                    uint32_t* out_cnt) {
    const uint32_t q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (q >= nq) return;
    WarpTopK<KPL> tk;
    tk.init();
    for (uint32_t g = 0; g < G; ++g) {
        const uint64_t base = ((uint64_t)g * nq + q) * k;
        for (uint32_t e0 = 0; e0 < k; e0 += 32) {
            const uint32_t e = e0 + lane;
            const float cd = e < k ? dists[base + e] : 0.f;
            const long long ci = e < k ? ids[base + e] : -1;
            const bool pass = e < k && ci >= 0 && tk.admits(cd, ci);
            unsigned m = __ballot_sync(0xffffffffu, pass);
            if (!m) break;
            while (m) {
                const int src = __ffs(m) - 1;
                m &= m - 1;
                const float bd = __shfl_sync(0xffffffffu, cd, src);
                const long long bi = __shfl_sync(0xffffffffu, ci, src);
                if (tk.admits(bd, bi)) tk.insert(bd, bi, (int)k, lane);
            }
        }
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int r = 0; r < KPL; ++r) {
        const uint32_t e = r * 32 + lane;
        cnt += __popc(__ballot_sync(0xffffffffu, e < k && tk.id[r] >= 0));
        if (e < k) {
            out_d[(uint64_t)q * k + e] = tk.d[r];
            out_i[(uint64_t)q * k + e] = tk.id[r];
        }
    }
    if (lane == 0 && out_cnt) out_cnt[q] = cnt;
}

unsigned grid_for(uint64_t work, unsigned cap = 148 * 16) {
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((work + 255) / 256, cap));
}

}  // namespace

cudaError_t launch_make_asg(const long long* nearest, const long long* ids, uint32_t n,
                            uint32_t* asg, cudaStream_t s) {
    if (!n) return cudaSuccess;
    make_asg_kernel<<<(n + 255) / 256, 256, 0, s>>>(nearest, ids, n, asg);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_block_moves(float* arena, long long* bids, uint64_t PS, uint32_t T,
                               const int32_t* src, const int32_t* dst, uint32_t nmoves,
                               float* scr_pay, long long* scr_ids, cudaStream_t s) {
    if (!nmoves) return cudaSuccess;
    const unsigned gx = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((PS / 4 + 255) / 256, 64));
    for (int phase = 0; phase < 2; ++phase) {
        block_move_kernel<<<dim3(gx, nmoves), 256, 0, s>>>(arena, bids, PS, T, src, dst, nmoves,
                                                           scr_pay, scr_ids, phase);
        count_launch();
    }
    return cudaGetLastError();
}

cudaError_t launch_slot_moves(float* off_pay, long long* off_ids, float* arena, long long* bids,
                              uint32_t D, const uint64_t* pay_addr, const uint64_t* id_addr,
                              uint32_t nmoves, float* scr_pay, long long* scr_ids,
                              cudaStream_t s) {
    if (!nmoves) return cudaSuccess;
    for (int phase = 0; phase < 2; ++phase) {
        slot_move_kernel<<<grid_for((uint64_t)nmoves * D), 256, 0, s>>>(
            off_pay, off_ids, arena, bids, D, pay_addr, id_addr, nmoves, scr_pay, scr_ids, phase);
        count_launch();
    }
    return cudaGetLastError();
}

cudaError_t launch_clear_ids(long long* off_ids, long long* bids, const uint64_t* id_addr,
                             uint32_t n, cudaStream_t s) {
    if (!n) return cudaSuccess;
    clear_ids_kernel<<<(n + 255) / 256, 256, 0, s>>>(off_ids, bids, id_addr, n);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_set_u32(uint32_t* arr, const uint32_t* idx, const uint32_t* val, uint32_t n,
                           cudaStream_t s) {
    if (!n) return cudaSuccess;
    set_u32_kernel<<<(n + 255) / 256, 256, 0, s>>>(arr, idx, val, n);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_locate(const long long* ids, uint64_t nslots, bool arena,
                          const long long* hkeys, const uint32_t* hvals, uint32_t hmask,
                          uint64_t* loc, cudaStream_t s) {
    if (!nslots) return cudaSuccess;
    locate_kernel<<<grid_for(nslots, 148 * 32), 256, 0, s>>>(ids, nslots, arena ? (1ull << 63) : 0,
                                                             hkeys, hvals, hmask, loc);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_copy_blocks(void* base, uint64_t bytes, const int32_t* src, const int32_t* dst,
                               uint32_t n, cudaStream_t s) {
    if (!n || !base || !bytes) return cudaSuccess;
    if (bytes & 7) return cudaErrorInvalidValue;
    const uint64_t units = bytes / ((bytes & 15) == 0 ? 16 : 8);
    const unsigned gx = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((units + 255) / 256, 64));
    copy_blocks_kernel<<<dim3(gx, n), 256, 0, s>>>(static_cast<char*>(base), bytes, src, dst, n);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_publish_lists(uint32_t n, const uint32_t* idx, const uint64_t* start,
                                 const uint32_t* count, const uint64_t* row, const uint32_t* len,
                                 uint64_t* L_start, uint32_t* L_count, uint64_t* L_row,
                                 uint32_t* L_len, uint32_t* L_ver, cudaStream_t s) {
    if (!n) return cudaSuccess;
    publish_lists_kernel<<<(n + 255) / 256, 256, 0, s>>>(n, idx, start, count, row, len, L_start,
                                                         L_count, L_row, L_len, L_ver);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_merge_shards(const float* dists, const long long* ids, uint32_t G, uint32_t nq,
                                uint32_t k, float* out_d, long long* out_i, uint32_t* out_cnt,
                                cudaStream_t s) {
    if (!nq) return cudaSuccess;
    const unsigned grid = (nq + 3) / 4;
    if (k <= 32) merge_shards_kernel<1><<<grid, 128, 0, s>>>(dists, ids, G, nq, k, out_d, out_i, out_cnt);
    else if (k <= 64) merge_shards_kernel<2><<<grid, 128, 0, s>>>(dists, ids, G, nq, k, out_d, out_i, out_cnt);
    else if (k <= 128) merge_shards_kernel<4><<<grid, 128, 0, s>>>(dists, ids, G, nq, k, out_d, out_i, out_cnt);
    else if (k <= 256) merge_shards_kernel<8><<<grid, 128, 0, s>>>(dists, ids, G, nq, k, out_d, out_i, out_cnt);
    else return cudaErrorInvalidValue;
    count_launch();
    return cudaGetLastError();
}

// ---- seed samples (scan_tc.cu vm_seed_kernel) ----------------------------
// Per list, kSampS stored vectors of its offline segment with small residual
// norms |x - c|^2 (each of 512 threads keeps its 2 best, the block sorts the 1024
// and takes the first kSampS), copied in the interleaved group layout
// [list][d][slot] with their ids.  Any stored vectors make a valid seed; central
// ones make a tight one (their distance to a query is close to |q - c|^2).
namespace {
__global__ void __launch_bounds__(512) sample_build_kernel(const float* off_pay, const long long* off_ids,
                                                           const uint64_t* off_start, const uint32_t* off_count,
                                                           const float* cent, uint32_t D, float* rows,
                                                           long long* ids) {
    __shared__ uint64_t key[1024];
    const uint32_t c = blockIdx.x, t = threadIdx.x;
    const uint32_t n = off_count[c];
    const uint64_t start = off_start[c];
    const float* cc = cent + (uint64_t)c * D;
    uint64_t b0 = ~0ull, b1 = ~0ull;
    for (uint32_t v = t; v < n; v += 512) {
        const uint64_t slot = start + v;
        const float* x = off_pay + (slot >> 5) * 32ull * D + (slot & 31u);
        float s2 = 0.f;
        for (uint32_t d = 0; d < D; ++d) {
            const float r = x[(uint64_t)d * 32] - cc[d];
            s2 = fmaf(r, r, s2);
        }
        const uint64_t k = ((uint64_t)__float_as_uint(s2) << 32) | v;  // s2 >= 0: bits order as values
        if (k < b0) {
            b1 = b0;
            b0 = k;
        } else if (k < b1) {
            b1 = k;
        }
    }
    key[2 * t] = b0;
    key[2 * t + 1] = b1;
    __syncthreads();
    for (uint32_t sz = 2; sz <= 1024; sz <<= 1)  // bitonic sort, ascending
        for (uint32_t st = sz >> 1; st > 0; st >>= 1) {
            for (uint32_t i = t; i < 1024; i += 512) {
                const uint32_t j = i ^ st;
                if (j > i) {
                    const bool up = (i & sz) == 0;
                    const uint64_t a = key[i], b = key[j];
                    if ((a > b) == up) {
                        key[i] = b;
                        key[j] = a;
                    }
                }
            }
            __syncthreads();
        }
    for (uint32_t e = t; e < kSampS * D; e += 512) {  // e = d * kSampS + slot
        const uint32_t d = e / kSampS, sl = e % kSampS;
        const uint64_t k = key[sl];
        const bool ok = k != ~0ull;
        const uint64_t slot = start + (uint32_t)k;
        rows[((uint64_t)c * D + d) * kSampS + sl] =
            ok ? off_pay[(slot >> 5) * 32ull * D + (uint64_t)d * 32 + (slot & 31u)] : 0.f;
        if (d == 0) ids[(uint64_t)c * kSampS + sl] = ok ? off_ids[slot] : -1;
    }
}

// a deleted id leaves every list's sample (gone: ascending)
__global__ void sample_invalidate_kernel(long long* ids, uint64_t n, const long long* gone, uint32_t ng) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const long long v = ids[i];
    if (v < 0) return;
    uint32_t lo = 0, hi = ng;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (gone[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    if (lo < ng && gone[lo] == v) ids[i] = -1;
}
}  // namespace

cudaError_t launch_sample_build(const float* off_pay, const long long* off_ids, const uint64_t* off_start,
                                const uint32_t* off_count, const float* cent, uint32_t C, uint32_t D,
                                float* rows, long long* ids, cudaStream_t s) {
    if (!C) return cudaSuccess;
    sample_build_kernel<<<C, 512, 0, s>>>(off_pay, off_ids, off_start, off_count, cent, D, rows, ids);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_sample_invalidate(long long* ids, uint64_t n, const long long* gone, uint32_t ng,
                                     cudaStream_t s) {
    if (!n || !ng) return cudaSuccess;
    sample_invalidate_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(ids, n, gone, ng);
    count_launch();
    return cudaGetLastError();
}

}  // namespace bivf
