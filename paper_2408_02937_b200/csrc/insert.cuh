// Host-visible declarations for the insert / bulk-load / k-means kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "mirror.cuh"

namespace bivf {

// Mutable device state touched by an insert batch (device pointers).
struct InsertState {
    uint32_t C, D, T, MLB, num_blocks;
    uint64_t PS;
    float* arena;
    long long* bids;
    int32_t* owner;
    uint32_t* cursor;
    uint32_t* len;
    uint32_t* nblocks;
    uint8_t* fail;
    int32_t* const* rowptr;   // per list: its live block-table row (MLB = row capacity)
    // per-batch scratch, [C] each
    uint32_t *run, *fail_from, *newlen;
};

// asg[i] = cluster of vector i (0xffffffff = rejected before assignment).
// out_blk[i] = pool block the vector landed in (-1 = failed), out_did[i] =
// its position in the list.  The scan mirror (if any) is written with the
// payload.  Release-publishes the list lengths last.
// Block headers (prev/next/head/tail) are derived on the host from the new
// blocks' owners, in allocation order (GpuIndex::absorb_new_blocks).
cudaError_t launch_insert(const InsertState& S, uint32_t n, const float* x, const long long* ids,
                          const uint32_t* asg, int32_t* out_blk, uint32_t* out_did,
                          const MirrorView* mirror, cudaStream_t s);

// offline segment build: row i -> slot dest[i] of the concatenated,
// group-aligned offline segments (ivf_index.cpp:61-82 layout).
cudaError_t launch_scatter_rows(const float* x, uint32_t n, uint32_t D, const uint64_t* dest,
                                const long long* ids, float* off_payload, long long* off_ids,
                                cudaStream_t s);

// k-means++ seeding distance fold (kmeans.cpp:47-68).
cudaError_t launch_seed_update(const float* pts_il, uint32_t n, uint32_t D, const float* cent,
                               double* min_d2, int first, cudaStream_t s);

}  // namespace bivf
