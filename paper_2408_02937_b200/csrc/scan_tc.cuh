// Host-visible declarations for the tensor-core filtered scan (scan_tc.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "scan.cuh"

namespace bivf {

// candidate slots per run (query, list chunk, warpgroup): 40 for k <= 16, 56 for
// k <= 32 (inner-product wide mode: 64, 72); global buffers use the largest stride
constexpr uint32_t kKC = 72;
constexpr uint32_t kOverflow = 0xffffffffu;  // ccount marker: buffer overflowed -> exact rescan

// per-search scratch of the TC path (lease workspace)
// runs = pairs * maxch * 2 (one per chunk and math warpgroup)
struct TcBufs {
    float* ub;          // [runs][k]  upper bounds (k smallest)
    uint32_t* ccount;   // [runs]     candidates kept (kOverflow -> exact rescan)
    float* clb;         // [runs][kKC] lower bounds
    uint32_t* cloc;     // [runs][kKC] group << 5 | slot
    float* qthr;        // [nq]       shared per-query threshold (reset per launch)
};

bool tc_supported(uint32_t D, uint32_t k, int metric);
bool tc_dense_supported(uint32_t D, uint32_t k, int metric);

// Dense mode of the TC scan (coarse quantizer): the single list's n slots,
// approximate distances -> out[nq][ld], query norms -> nq; the selection
// kernel then returns the exact top-k (dist, slot).
struct TcDense {
    float* out;
    float* nq;
    uint32_t ld, n;
    const uint64_t* list_base = nullptr;  // IVF dense mode (k > 32): per-list tile block offsets
    float2* gsum = nullptr;               // IVF dense mode: per-(pair, group) bound minima
};

// IVF dense mode (k > 32, exact top-k through the TC distances): plan + per-list
// tile-block sizes (tiles x groups x 32 slots x 128 rows) + exclusive scan;
// *total (device) = floats the dense blocks need.
size_t dense_plan_tmp_bytes(uint32_t nlists);
cudaError_t launch_dense_plan(const DevLists& L, const PlanBufs& B, const long long* probes,
                              const SearchShape& sh, uint64_t* list_len, uint64_t* list_base,
                              void* tmp, size_t tmp_bytes, uint64_t* total, cudaStream_t s);

// 2-D TMA map over a scan mirror region (mirror.cuh: `groups` groups of 2K rows
// of 32 bf16, box = {32, 2K}; wide: K rows, box = {32, min(K, 128)}), SWIZZLE_64B.
cudaError_t make_mirror_map(const float* base, uint64_t groups, uint32_t D, bool wide,
                            CUtensorMap* out, bool hi_only = false);

// the vector-major scan's maps over one mirror region (offline segments or the
// arena): out3[0] one group's hi plane, out3[1] four consecutive groups' hi
// planes (3-D), out3[2] their |s|^2 rows; launch_ivf_search_tc takes six
// (offline then arena) as maps_hi.  vm_mode: -1 choose by pairs per list, 1 the
// vector-major scan whenever maps_hi allows it, 0 never (query-major).
cudaError_t make_vm_maps(const float* mir, const float* nrm, uint64_t groups, uint32_t D, CUtensorMap* out3);

cudaError_t launch_ivf_search_tc(const DevLists& L, const PlanBufs& B, const long long* probes,
                                 const float* queries, const float* centroids,
                                 const SearchShape& sh, const CUtensorMap& map_off,
                                 const CUtensorMap& map_arena, const float* off_nrm,
                                 const float* arena_nrm, const float* off_rows,
                                 const float* arena_rows, const TcBufs& T, const TcDense* dense,
                                 float* out_d,
                                 long long* out_i, uint32_t* out_cnt, int num_sms,
                                 cudaStream_t s, cudaEvent_t ev0 = nullptr,
                                 cudaEvent_t ev1 = nullptr, int max_grid = 1 << 30,
                                 const CUtensorMap* maps_hi = nullptr, const float* samp_rows = nullptr,
                                 const long long* samp_ids = nullptr, int vm_mode = -1);

}  // namespace bivf
