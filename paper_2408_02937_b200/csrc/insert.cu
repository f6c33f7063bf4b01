// Real-time insert (K5), bulk load and the k-means helpers, sm_100a.
//
// The reference inserts a batch sequentially (src/ivf_index.cpp:122-229):
// per vector, did = length++ of its cluster, block mid = did / T_m; the
// vector with did % T_m == 0 ("designated writer") allocates a pool block by
// bumping the cursor (block_store.cpp:31-48) and links it after the tail
// (block_store.cpp:55-65); every vector then writes its interleaved slot and
// publishes the committed prefix (block_store.cpp:67-90).  On exhaustion the
// cluster is poisoned and the batch continues (ivf_index.cpp:180-193).
//
// Batch-parallel restatement (validated against the
// reference in tests/test_oracle_vs_ref.py and on device in tests/test_gpu_*):
//   (i)   stable per-cluster rank in batch order  -> did = len_c + rank
//   (ii)  openers: did % T_m == 0 and mid >= blocks already in the list
//   (iii) openers of non-poisoned lists, in batch order, take consecutive
//         pool indices from the cursor while blocks remain
//   (iv)  a cluster's vectors from its first failed opener onward fail and
//         poison it
// One CTA runs (i)-(iv) over 1024-vector chunks (cub stable radix sort for the
// rank, block scans for opener order); a grid-wide kernel writes the payload;
// a third kernel release-publishes the list lengths so concurrent scans on
// other streams only ever see committed prefixes.
#include <algorithm>

#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "insert.cuh"
#include "launches.h"

namespace bivf {

namespace {

constexpr uint32_t kInvalid = 0xffffffffu;
constexpr int kLayoutThreads = 1024;

__global__ void reset_scratch(uint32_t C, uint32_t* run, uint32_t* fail_from, uint32_t* newlen,
                              const uint32_t* len) {
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
        run[c] = 0;
        fail_from[c] = kInvalid;
        newlen[c] = len[c];
    }
}

__global__ void __launch_bounds__(kLayoutThreads) layout_kernel(InsertState S, uint32_t n,
                                                                const uint32_t* asg,
                                                                int32_t* out_blk,
                                                                uint32_t* out_did) {
    using Sort = cub::BlockRadixSort<uint32_t, kLayoutThreads, 1, uint32_t>;
    using ScanU = cub::BlockScan<uint32_t, kLayoutThreads>;
    __shared__ union {
        typename Sort::TempStorage sort;
        typename ScanU::TempStorage scan;
    } tmp;
    __shared__ uint32_t skey[kLayoutThreads];
    __shared__ uint32_t srank[kLayoutThreads];
    __shared__ uint32_t s_obase, s_R;

    const uint32_t t = threadIdx.x;
    if (t == 0) {
        s_obase = 0;
        const uint32_t cur = *S.cursor;
        s_R = cur < S.num_blocks ? S.num_blocks - cur : 0u;
    }
    __syncthreads();
    const uint32_t cursor0 = *S.cursor;

    for (uint32_t base = 0; base < n; base += kLayoutThreads) {
        const uint32_t i = base + t;
        const uint32_t a = i < n ? asg[i] : kInvalid;

        // (i) stable rank among equal clusters within the chunk
        uint32_t key[1] = {a};
        uint32_t val[1] = {t};
        Sort(tmp.sort).Sort(key, val);
        skey[t] = key[0];
        __syncthreads();
        const uint32_t head_pos = (t == 0 || skey[t - 1] != key[0]) ? t : 0u;
        uint32_t seg_start;
        ScanU(tmp.scan).InclusiveScan(head_pos, seg_start, cub::Max());
        srank[val[0]] = t - seg_start;
        const bool seg_last = (t == kLayoutThreads - 1) || skey[t + 1] != key[0];
        __syncthreads();

        // (ii)/(iii) openers in batch order
        uint32_t did = 0, mid = 0;
        bool opener = false, consuming = false;
        if (a != kInvalid) {
            did = S.len[a] + S.run[a] + srank[t];
            mid = did / S.T;
            opener = (did % S.T == 0) && (mid >= S.nblocks[a]);
            consuming = opener && !S.fail[a] && mid < S.MLB;
        }
        uint32_t cidx, ctotal;
        ScanU(tmp.scan).ExclusiveSum(consuming ? 1u : 0u, cidx, ctotal);
        const uint32_t gidx = s_obase + cidx;
        const bool ok_open = consuming && gidx < s_R;
        int32_t blk = -1;
        if (ok_open) {
            blk = (int32_t)(cursor0 + gidx);
            S.rowptr[a][mid] = blk;  // appended past every published entry
            S.owner[blk] = (int32_t)a;
            atomicMax(&S.nblocks[a], mid + 1);
        } else if (opener) {
            atomicMin(&S.fail_from[a], i);  // (iv)
            S.fail[a] = 1;
        }
        __syncthreads();
        // rank bases for the next chunk (one writer per cluster segment)
        if (seg_last && key[0] != kInvalid) S.run[key[0]] += t - seg_start + 1;
        if (t == 0) s_obase += ctotal;
        __syncthreads();
        if (i < n) {
            bool ok = a != kInvalid && i < S.fail_from[a];
            out_blk[i] = ok ? S.rowptr[a][mid] : -1;
            out_did[i] = did;
            if (ok) atomicMax(&S.newlen[a], did + 1);
        }
        __syncthreads();
    }
    if (t == 0) {
        const uint32_t used = s_obase < s_R ? s_obase : s_R;
        *S.cursor = cursor0 + used;
    }
}

// payload + id writes: thread per (vector, dim); interleaved offset
// (block_store.hpp:37-40).
__global__ void write_kernel(InsertState S, uint32_t n, const float* x, const long long* ids,
                             const int32_t* out_blk, const uint32_t* out_did) {
    const uint64_t total = (uint64_t)n * S.D;
    for (uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total;
         o += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t i = (uint32_t)(o / S.D), d = (uint32_t)(o - (uint64_t)i * S.D);
        const int32_t b = out_blk[i];
        if (b < 0) continue;
        const uint32_t slot = out_did[i] % S.T;
        S.arena[(uint64_t)b * S.PS + (uint64_t)(slot / 32u) * 32u * S.D + (uint64_t)d * 32u +
                (slot % 32u)] = x[o];
        if (d == 0) S.bids[(uint64_t)b * S.T + slot] = ids[i];
    }
}

// release-publish: the list length, by the list's last new vector, after the
// payload kernel completed (stream order) — a scan that acquires the new
// length sees every slot below it (block_store.cpp:83-90 prefix commit).
__global__ void publish_kernel(InsertState S, uint32_t n, const uint32_t* asg,
                               const int32_t* out_blk, const uint32_t* out_did) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (out_blk[i] < 0) return;
    const uint32_t a = asg[i];
    const uint32_t nl = S.newlen[a];
    if (out_did[i] + 1 == nl) {
        __threadfence();
        st_release_u32(S.len + a, nl);
    }
}

// --------------------------------------------------------------- bulk load
__global__ void scatter_rows(const float* x, uint32_t n, uint32_t D, const uint64_t* dest,
                             const long long* ids, float* off_payload, long long* off_ids) {
    const uint64_t total = (uint64_t)n * D;
    for (uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total;
         o += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = o / D;
        const uint32_t d = (uint32_t)(o - i * D);
        const uint64_t s = dest[i];
        off_payload[(s / 32u) * 32u * D + (uint64_t)d * 32u + (s % 32u)] = x[o];
        if (d == 0) off_ids[s] = ids[i];
    }
}

// --------------------------------------------------------------- k-means++
// d2 of every point to centroid `cent` (exact l2_sqr, distance.hpp:11-18; the
// reference computes l2_sqr(point, centroid), kmeans.cpp:50/65), folded into
// min_d2 as double exactly like kmeans.cpp:64-66.
__global__ void seed_update(const float* pts_il, uint32_t n, uint32_t D, const float* cent,
                            double* min_d2, int first) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* base = pts_il + (uint64_t)(i / 32u) * 32u * D + (i % 32u);
    float acc = 0.f;
    for (uint32_t d = 0; d < D; ++d) acc = l2_step(acc, base[(uint64_t)d * 32u], cent[d]);
    const double v = (double)acc;
    if (first || v < min_d2[i]) min_d2[i] = v;
}

}  // namespace

cudaError_t launch_insert(const InsertState& S, uint32_t n, const float* x, const long long* ids,
                          const uint32_t* asg, int32_t* out_blk, uint32_t* out_did,
                          const MirrorView* mirror, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    reset_scratch<<<(S.C + 255) / 256, 256, 0, s>>>(S.C, S.run, S.fail_from, S.newlen, S.len);
    layout_kernel<<<1, kLayoutThreads, 0, s>>>(S, n, asg, out_blk, out_did);
    const uint64_t total = (uint64_t)n * S.D;
    const unsigned wg = (unsigned)std::min<uint64_t>((total + 255) / 256, 148ull * 16);
    write_kernel<<<wg, 256, 0, s>>>(S, n, x, ids, out_blk, out_did);
    if (mirror) {
        const cudaError_t e = launch_mirror_insert(*mirror, n, x, asg, out_blk, out_did, s);
        if (e != cudaSuccess) return e;
    }
    publish_kernel<<<(n + 255) / 256, 256, 0, s>>>(S, n, asg, out_blk, out_did);
    count_launch(4);
    return cudaGetLastError();
}

cudaError_t launch_scatter_rows(const float* x, uint32_t n, uint32_t D, const uint64_t* dest,
                                const long long* ids, float* off_payload, long long* off_ids,
                                cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const uint64_t total = (uint64_t)n * D;
    const unsigned g = (unsigned)std::min<uint64_t>((total + 255) / 256, 148ull * 32);
    scatter_rows<<<g, 256, 0, s>>>(x, n, D, dest, ids, off_payload, off_ids);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_seed_update(const float* pts_il, uint32_t n, uint32_t D, const float* cent,
                               double* min_d2, int first, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    seed_update<<<(n + 255) / 256, 256, 0, s>>>(pts_il, n, D, cent, min_d2, first);
    count_launch();
    return cudaGetLastError();
}

}  // namespace bivf
