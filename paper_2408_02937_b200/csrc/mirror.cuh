// The tensor-core scan mirror.
//
// For every stored vector x of list c the index keeps, next to the
// reference-layout payload (which stays the source of truth and of every exact
// distance), the list-centred residual s = fl(x - c) pre-split for 3xTF32:
// s_hi = TF32 truncation of s, s_lo = s - s_hi (exact in fp32), plus |s|^2 and
// |s|.  Layout per 32-vector group (same group indexing as the payload, so
// slot/block moves map one-to-one), rows of 32 floats (one per slot):
//     rows [0, D)        s_hi, dim d
//     row  D             |s|^2   (sequential fp32)
//     rows [D+1, 2D+1)   s_lo, dim d
//     row  2D+1          |s|
// Two TMA boxes of {32, D+1} rows stage a group's B operands + norms.  The
// mirror is written by the same data-lane operations that write the payload
// (bulk load, insert, delete slot moves, rearrangement block moves), before
// the list length that exposes the slots is release-published.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace bivf {

struct MirrorView {
    float* off_mir;        // offline groups x GF
    float* arena_mir;      // num_blocks x MPS
    const float* cent;     // [C][D] row-major centroids
    uint32_t D, T, gpb;
    uint64_t GF;           // floats per group  = (2D+2)*32
    uint64_t MPS;          // floats per block  = gpb*GF
};

inline uint64_t mirror_group_floats(uint32_t D) { return (2ull * D + 2) * 32ull; }

// insert: vector i (row-major x[i*D..]) landed in block out_blk[i] (-1 = failed)
// at list position out_did[i]; its list is asg[i].
cudaError_t launch_mirror_insert(const MirrorView& M, uint32_t n, const float* x,
                                 const uint32_t* asg, const int32_t* out_blk,
                                 const uint32_t* out_did, cudaStream_t s);
// bulk load: row i -> offline slot dest[i] of list asg[i].
cudaError_t launch_mirror_offline(const MirrorView& M, uint32_t n, const float* x,
                                  const uint64_t* dest, const uint32_t* asg, cudaStream_t s);
// rebuild whole groups from the payload: group g (offline group index, or
// arena group index block*gpb + j when arena) of list cl[i].
cudaError_t launch_mirror_groups(const MirrorView& M, const float* payload, bool arena,
                                 uint64_t PS, const uint64_t* groups, const uint32_t* cl,
                                 uint32_t n, cudaStream_t s);
// delete compaction: the same moves as launch_slot_moves, on the mirror
// (id_addr[2n] = sources then destinations; bit 63 = arena, value = the slot's
// id index).  scratch: n * (2D+2) floats.
cudaError_t launch_mirror_slot_moves(const MirrorView& M, const uint64_t* id_addr, uint32_t n,
                                     float* scratch, cudaStream_t s);

}  // namespace bivf
