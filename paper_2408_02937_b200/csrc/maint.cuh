// Host-visible declarations for maint.cu.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace bivf {

cudaError_t launch_make_asg(const long long* nearest, const long long* ids, uint32_t n,
                            uint32_t* asg, cudaStream_t s);
cudaError_t launch_block_moves(float* arena, long long* bids, uint64_t PS, uint32_t T,
                               const int32_t* src, const int32_t* dst, uint32_t nmoves,
                               float* scr_pay, long long* scr_ids, cudaStream_t s);
// pay_addr/id_addr hold 2*nmoves entries: sources then destinations
cudaError_t launch_slot_moves(float* off_pay, long long* off_ids, float* arena, long long* bids,
                              uint32_t D, const uint64_t* pay_addr, const uint64_t* id_addr,
                              uint32_t nmoves, float* scr_pay, long long* scr_ids,
                              cudaStream_t s);
cudaError_t launch_clear_ids(long long* off_ids, long long* bids, const uint64_t* id_addr,
                             uint32_t n, cudaStream_t s);
cudaError_t launch_set_u32(uint32_t* arr, const uint32_t* idx, const uint32_t* val, uint32_t n,
                           cudaStream_t s);
cudaError_t launch_locate(const long long* ids, uint64_t nslots, bool arena,
                          const long long* hkeys, const uint32_t* hvals, uint32_t hmask,
                          uint64_t* loc, cudaStream_t s);
cudaError_t launch_merge_shards(const float* dists, const long long* ids, uint32_t G, uint32_t nq,
                                uint32_t k, float* out_d, long long* out_i, uint32_t* out_cnt,
                                cudaStream_t s);

// n whole-block copies of `bytes` (multiple of 8) from block src[i] to dst[i]
// of the array at `base` (source and destination sets disjoint).
cudaError_t launch_copy_blocks(void* base, uint64_t bytes, const int32_t* src, const int32_t* dst,
                               uint32_t n, cudaStream_t s);
// publish new list versions (DevLists seqlock); null field arrays stay unchanged
cudaError_t launch_publish_lists(uint32_t n, const uint32_t* idx, const uint64_t* start,
                                 const uint32_t* count, const uint64_t* row, const uint32_t* len,
                                 uint64_t* L_start, uint32_t* L_count, uint64_t* L_row,
                                 uint32_t* L_len, uint32_t* L_ver, cudaStream_t s);

constexpr uint64_t kArenaBit = 1ull << 63;

// seed samples of the vector-major scan: kSampS offline vectors per list with
// small residual norms, [list][d][slot] + ids (-1 = empty / deleted)
#ifndef BIVF_SAMP_S
#define BIVF_SAMP_S 32
#endif
constexpr uint32_t kSampS = BIVF_SAMP_S;
static_assert(kSampS % 32 == 0 && kSampS <= 1024, "seed samples: whole warps, <= the build's 1024 sorted keys");
cudaError_t launch_sample_build(const float* off_pay, const long long* off_ids, const uint64_t* off_start,
                                const uint32_t* off_count, const float* cent, uint32_t C, uint32_t D,
                                float* rows, long long* ids, cudaStream_t s);
cudaError_t launch_sample_invalidate(long long* ids, uint64_t n, const long long* gone, uint32_t ng,
                                     cudaStream_t s);

}  // namespace bivf
