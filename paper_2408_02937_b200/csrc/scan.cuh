// Host-visible declarations for the scan/merge/plan kernels (scan.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace bivf {

// Device view of the index's storage (all pointers device memory).
// Live view: the index's published per-list state.  A search reads it ONCE, in
// its plan (snapshot_list: a per-list seqlock against maintenance publishes), and
// every later kernel of the search gets a snapshot view (snapshot_view) whose
// off_start / rowptr are the plan's copies: maintenance (delete, rearrangement)
// never edits storage a published state points to; it writes new versions
// elsewhere, publishes them, and reuses the old storage only after every search
// that may have snapshotted it has finished (GpuIndex::grace).
struct DevLists {
    uint32_t C, D, T, gpb;   // clusters, dim, block capacity, groups per block
    uint64_t PS;             // payload scalars per block = gpb*32*D
    const float* off_payload;     // offline segments, interleaved, group-aligned
    const long long* off_ids;     // per slot
    const uint64_t* off_start;    // per cluster, slot offset (multiple of 32)
    const uint32_t* off_count;    // per cluster
    const float* arena;           // pool payload, (num_blocks + scratch) * PS
    const long long* bids;        // pool ids, (num_blocks + scratch) * T
    const int32_t* const* rowptr; // per cluster: its block-table row (logical order)
    const uint32_t* len;          // per-list online length (published, acquire)
    const uint32_t* ver;          // per-list seqlock: odd while a publish rewrites the list
};

// Per-search scratch (lease workspace), device pointers.
struct PlanBufs {
    uint32_t* snap_off;   // [C]
    uint32_t* snap_len;   // [C]
    uint64_t* snap_start; // [C] offline segment start at plan time
    uint64_t* snap_row;   // [C] block-table row pointer at plan time
    uint32_t* gc;         // [C] groups per chunk
    uint32_t* nch;        // [C] chunks
    uint32_t* cnt;        // [C] pairs per list
    uint32_t* qoff;       // [C+1]
    uint32_t* item_off;   // [C+1]
    uint32_t* n_items;    // [1]
    uint32_t* item_ctr;   // [1]
    uint32_t* ppos;       // [npairs]
    uint32_t* plist;      // [npairs]
};

struct SearchShape {
    uint32_t nq, k, P, maxch, gcmin, QT;
    int metric;
};

// The view every post-plan kernel of a search uses: the plan's snapshot of
// the lists' offline starts and block-table rows.
inline DevLists snapshot_view(const DevLists& L, const PlanBufs& B) {
    DevLists v = L;
    v.off_start = B.snap_start;
    v.rowptr = reinterpret_cast<const int32_t* const*>(B.snap_row);
    return v;
}

// Picks the device top-k width for k (1,2,4,8 registers per lane).
int kpl_for(uint32_t k);
uint32_t qt_for(uint32_t k, uint32_t D);

// Coarse quantizer on CUDA cores (K2 semantics, exact): probes[q*P + p] are
// the P lowest (key, cluster) pairs; cand_* is scratch of nq*flat_nch*P.
cudaError_t launch_flat_topk(const float* flat_il, uint32_t n, uint32_t D, const float* queries,
                             uint32_t nq, uint32_t k, int metric, uint32_t nch, float* cand_d,
                             long long* cand_i, float* out_d, long long* out_i, uint32_t* out_cnt,
                             uint32_t* item_ctr, int num_sms, cudaStream_t s);

// The list scan: plan (snapshot, invert probe map, items) + scan + merge.
cudaError_t launch_ivf_search(const DevLists& L, const PlanBufs& B, const long long* probes,
                              const float* queries, const SearchShape& sh, float* cand_d,
                              long long* cand_i, float* out_d, long long* out_i,
                              uint32_t* out_cnt, int num_sms, cudaStream_t s,
                              cudaEvent_t ev_scan0 = nullptr, cudaEvent_t ev_scan1 = nullptr);

cudaError_t launch_all_probes(long long* probes, uint32_t nq, uint32_t C, cudaStream_t s);

// Only the plan kernels (snapshot, count, scan, scatter) of launch_ivf_search.
cudaError_t launch_plan(const DevLists& L, const PlanBufs& B, const long long* probes,
                        const SearchShape& sh, cudaStream_t s);
// Plan over the pairs of probe rank [lo, hi) only; snapshot = false reuses the
// previous plan's list snapshot (snap_off/snap_len/gc/nch) and only re-counts.
cudaError_t launch_plan_ranked(const DevLists& L, const PlanBufs& B, const long long* probes,
                               const SearchShape& sh, uint32_t lo, uint32_t hi, bool snapshot,
                               cudaStream_t s);

// Copy row-major fp32 rows [n][D] into the 32-interleaved group layout
// (block_store.hpp:37-40), zero-padding the last group; and the query
// staging layout [n][Dp] (Dp = D rounded up to 4, zero padded).
cudaError_t launch_interleave(const float* rows, uint32_t n, uint32_t D, float* out,
                              cudaStream_t s);
cudaError_t launch_pad_rows(const float* rows, uint32_t n, uint32_t D, uint32_t Dp, float* out,
                            cudaStream_t s);

inline uint32_t pad4(uint32_t d) { return (d + 3u) & ~3u; }

}  // namespace bivf
