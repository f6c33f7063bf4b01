// The tensor-core scan mirror.
//
// For every stored vector x of list c the index keeps, next to the
// reference-layout payload (which stays the source of truth and of every exact
// distance), the list-centred residual s = fl(x - c) pre-split for 3xBF16:
// s_hi = bf16_rn(s), s_lo = bf16_rn(s - s_hi) (s - s_hi is exact in fp32), plus
// |s|^2.  Same group indexing as the payload, so slot/block moves map one-to-one.
// Planes, per 32-vector group, rows of 32 bf16 (64 bytes, one element per slot),
// K = D rounded up to 16 (rows D..K-1 stay zero: the MMA's K padding):
//     rows [0, K)      s_hi, dim d
//     rows [K, 2K)     s_lo, dim d
// A group's planes occupy 2K*64 bytes = K*32 "floats" of the float-typed buffers.
// Wide mode (inner product, D <= 768; scan_tc.cu's 1xFP16 filter): the UNcentred
// vector scaled by 2^ev (max |x_d| 2^ev in [2^13, 2^14): fp16 keeps its 11-bit
// relative precision, no overflow) in one fp16 plane (K rows, K = D rounded up to
// 16, or to 128 when D > 128 so that 128-row K-chunks tile it), norms
// [2^-ev x32][|x| x32]; K*16 floats per group.
// Norms, per group, a separate array of 64 floats: [|s|^2 (sequential fp32) x 32]
// [kVScale * |s|^2 x 32] (the per-slot term of the scan's pass-1 threshold, scan_tc.cu).
// Rows, per group, a slot-major copy of the exact payload (32 x D fp32): the
// refine's candidate gathers read 4 contiguous 128-byte lines per vector instead
// of D scattered 32-byte sectors of the interleaved layout.
// One TMA box of {32, 2K} bf16 rows (SWIZZLE_64B) stages a group's two B operands.  The
// mirror is written by the same data-lane operations that write the payload
// (bulk load, insert, delete slot moves, rearrangement block moves), before
// the list length that exposes the slots is release-published.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>

namespace bivf {

struct MirrorView {
    float* off_mir;        // offline groups x GF (bf16 planes, see above)
    float* arena_mir;      // num_blocks x MPS
    float* off_nrm;        // offline groups x 64
    float* arena_nrm;      // num_blocks x gpb x 64
    float* off_rows;       // offline groups x 32 x D
    float* arena_rows;     // num_blocks x gpb x 32 x D
    const float* cent;     // [C][D] row-major centroids
    uint32_t D, K, T, gpb; // K = D rounded up to 16 (wide: mirror_k_wide)
    uint32_t wide;         // 1: inner-product wide mode (hi plane only, uncentred)
    uint64_t GF;           // floats per group  = K*32 (2K*32 bf16)
    uint64_t MPS;          // floats per block  = gpb*GF
};

// Error-bound constants of the tensor-core filter (D <= 128):
//   |a - e| <= kEpsCross*|r||s| + kEpsRel*(|r|^2+|s|^2) + kEpsRel*|a|  (>= 2x margin), and with
//   |r||s| <= (|r|^2+|s|^2)/2:  eps' = kEpsT*(nq+ns) + kEpsRel*|a|,  kEpsT = kEpsRel + kEpsCross/2.
// For a >= 0 the lower bound a - eps' <= ubk  <=>  dot >= kVScale*(nq+ns) - ubk/(2(1-kEpsRel)).
// 3xBF16 (scan_tc.cu): |P - r.s| <= (3.01*2^-16 + 24*2^-24)|r||s| <= 2^-14.3 |r||s|, so the
// cross term of a = nq + ns - 2P is off by <= 2^-13.3 |r||s|; 2^-12 carries a 2.5x margin.
constexpr float kEpsCross = 1.0f / 4096.0f;
constexpr float kEpsRel = 1.0f / 32768.0f;    // 2^-15 on (nq+ns) and on |a|
constexpr float kEpsT = kEpsRel + 0.5f * kEpsCross;
constexpr float kVScale = (1.0f - kEpsRel - kEpsT) / (2.0f * (1.0f - kEpsRel));

inline uint32_t mirror_k(uint32_t D) { return (D + 15u) & ~15u; }
inline uint64_t mirror_group_floats(uint32_t D) { return (uint64_t)mirror_k(D) * 32ull; }
// wide mode: K-chunks of min(K, 128) rows
inline uint32_t mirror_k_wide(uint32_t D) { return D <= 128 ? mirror_k(D) : (D + 127u) & ~127u; }
inline uint32_t mirror_chunk_wide(uint32_t D) { return std::min<uint32_t>(mirror_k_wide(D), 128u); }
inline uint64_t mirror_group_floats_wide(uint32_t D) { return (uint64_t)mirror_k_wide(D) * 16ull; }
// the 1xFP16 inner-product filter over 2^e-scaled operands (max |v_d| in [2^13, 2^14)):
// |fl(v) - v| <= 2^-11 |v| + 2^-25, so |P' - q'.x'| <= (2^-10 + 2^-22)|q'||x'| +
// 2^-24.9 sqrt(D)(|q'| + |x'|) + D 2^-50, and with |q'|, |x'| >= 2^13 the last two
// terms are < 2^-30 |q'||x'| (D <= 768): |P - q.x| <= 2^-9.99 |q||x| unscaled, plus
// fp32 accumulation (48 K-steps) <= 2^-19 |q||x|; 2^-9 carries a ~2x margin.
constexpr float kEpsIP = 1.0f / 512.0f;
// the scale exponent: max |v_d| * 2^e in [2^13, 2^14) (e = 0 for a zero vector)
__host__ __device__ inline int wide_scale_exp(float mx) {
    if (!(mx > 0.f)) return 0;
    int e = 0;
    (void)frexpf(mx, &e);  // mx = f * 2^e, f in [0.5, 1): mx in [2^(e-1), 2^e)
    return 14 - e;
}
constexpr uint32_t kNormFloats = 64;  // per group

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
// id index).  scratch: n * (2K+2+D) floats (one per moved bf16 plane element).
cudaError_t launch_mirror_slot_moves(const MirrorView& M, const uint64_t* id_addr, uint32_t n,
                                     float* scratch, cudaStream_t s);

}  // namespace bivf
