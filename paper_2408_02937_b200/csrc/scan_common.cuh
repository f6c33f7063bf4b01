// Device helpers shared by the CUDA-core scan (scan.cu) and the tensor-core
// scan (scan_tc.cu): where group j of list c lives (offline segment groups
// first, then the online blocks through the list's block table).
#pragma once

#include <cstdint>

#include "common.cuh"
#include "scan.cuh"

namespace bivf {

struct GroupRef {
    const float* base;
    const long long* ids;  // nullptr -> implicit id0 + slot
    long long id0;
    uint32_t nvalid;
};

__device__ __forceinline__ uint32_t ivf_ngroups(const DevLists& L, uint32_t off, uint32_t len) {
    const uint32_t og = (off + 31u) >> 5;
    const uint32_t full = len / L.T, rem = len - full * L.T;
    return og + full * L.gpb + ((rem + 31u) >> 5);
}

__device__ __forceinline__ GroupRef ivf_group(const DevLists& L, uint32_t c, uint32_t off,
                                              uint32_t len, uint32_t j) {
    GroupRef g;
    const uint32_t og = (off + 31u) >> 5;
    if (j < og) {
        const uint64_t slot0 = L.off_start[c] + 32ull * j;
        g.base = L.off_payload + slot0 * L.D;
        g.ids = L.off_ids + slot0;
        g.nvalid = min(32u, off - 32u * j);
    } else {
        const uint32_t jj = j - og;
        const uint32_t mid = jj / L.gpb, gi = jj - mid * L.gpb;
        const int32_t blk = L.rowptr[c][mid];
        const uint32_t cnt_mid = min(L.T, len - mid * L.T);
        g.base = L.arena + (uint64_t)blk * L.PS + (uint64_t)gi * 32u * L.D;
        g.ids = L.bids + (uint64_t)blk * L.T + 32u * gi;
        g.nvalid = min(32u, cnt_mid - 32u * gi);
    }
    g.id0 = 0;
    return g;
}


// One list's published state, consistent against maintenance publishes
// (maint.cu publish_lists: ver odd -> fields -> ver even).  Inserts only append
// (entries past the old block count, slots past the old length) and release
// the length, so they need no seqlock.
__device__ __forceinline__ void snapshot_list(const DevLists& L, uint32_t c, uint32_t& off,
                                              uint32_t& len, uint64_t& start, uint64_t& row) {
    for (;;) {
        const uint32_t v1 = ld_acquire_u32(L.ver + c);
        if (v1 & 1u) continue;  // a publish kernel is rewriting this list right now
        // the fields as relaxed loads, all in flight together (the acquire on the
        // version keeps them after it); the fence below turns them into an
        // acquire pattern, so a length read here synchronizes with the insert's
        // release-publish of it and later kernels see the payload it covers
        off = *reinterpret_cast<const volatile uint32_t*>(L.off_count + c);
        len = *reinterpret_cast<const volatile uint32_t*>(L.len + c);
        start = *reinterpret_cast<const volatile uint64_t*>(L.off_start + c);
        row = *reinterpret_cast<const volatile uint64_t*>(reinterpret_cast<const uint64_t*>(L.rowptr) + c);
        __threadfence();
        if (*reinterpret_cast<const volatile uint32_t*>(L.ver + c) == v1) return;
    }
}

}  // namespace bivf
