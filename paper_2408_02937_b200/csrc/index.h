// GpuIndex — host runtime of the B200-native online IVF-Flat path.
//
// Ownership split:
//   device  : centroids (+ interleaved copy), offline segments, pool arena +
//             ids, per-list block table / length / block count / fail flag,
//             allocation cursor, block owners.  Everything the scan and the
//             insert kernels read or write.
//   host    : the block-header mirror (prev/next/owner/merged, derived
//             committed), list head/tail, id bookkeeping (auto ranges,
//             supplied ids), counters, rearrangement planning.  Updated from
//             the device's own results after every insert (new block owners
//             + lengths), never guessed.
// Concurrency (the reference's contract, block_store.hpp:56-59):
//   search || search, search || insert: searches run on leased streams and
//     read only release-published prefixes (len) of append-only storage.
//   insert / remove / rearrange: serialized on the data stream (data_mu_),
//     like the reference's single data lane + insert_gate_.
//   remove / rearrange vs search: read-copy-update, searches never wait.  A
//     search snapshots every list's (offline start, count, block-table row,
//     length) once, in its plan, under a per-list seqlock (scan_common.cuh
//     snapshot_list).  Maintenance builds the new versions of the touched
//     blocks / segments in storage no published state references (scratch
//     blocks past the pool, free offline regions, the inactive copy of each
//     double-buffered block-table row), publishes them (maint.cu
//     publish_lists), and reuses old storage only after a grace period: the
//     data stream waits, on the device, for every search enqueued before the
//     publish (grace()).  Rearrangement and online deletes move data back into
//     the reference's block positions in a second phase (layout parity).
//     Oversized operations fall back to quiescence (begin/end_maintenance).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <memory>
#include <map>
#include <mutex>
#include <shared_mutex>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <vector>

#include "../../include/bivf.h"
#include "insert.cuh"
#include "mirror.cuh"
#include "scan.cuh"
#include "scan_tc.cuh"

namespace bivf {

struct Error : std::runtime_error {
    bivf_status code;
    uint64_t inserted = 0;
    Error(bivf_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char* what);
#define BIVF_CUDA(x) ::bivf::cuda_check((x), #x)

extern std::atomic<uint64_t> g_launches;

// RAII device allocation
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf();
    void alloc(size_t n);         // exact size, contents undefined
    void ensure(size_t n);        // grow (no copy)
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

struct PinBuf {
    void* p = nullptr;
    size_t bytes = 0;
    PinBuf() = default;
    PinBuf(const PinBuf&) = delete;
    PinBuf& operator=(const PinBuf&) = delete;
    ~PinBuf();
    void ensure(size_t n);
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

// A search lease: one stream + its device workspace + pinned staging
// (Alg. 4's per-request resource).
struct Lease {
    int id = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;
    cudaEvent_t t0 = nullptr, t1 = nullptr, t2 = nullptr, t3 = nullptr, t4 = nullptr;
    DevBuf ws;
    PinBuf pin;
    DevBuf dense, dense_aux;  // k > 32 TC path: dense distance rows + per-pair offsets
    PinBuf dpin;
    uint64_t seen_maint = 0;
    bool busy = false;
    // small-batch searches replayed as CUDA graphs (GpuIndex::search): one entry
    // per (batch shape, workspace, index device-buffer signature)
    struct Graph {
        uint32_t m, k, P;
        void* ws;
        uint64_t sig;
        cudaGraphExec_t exec;
        uint64_t launches;
    };
    std::vector<Graph> graphs;
};

struct Workspace {  // carved from Lease::ws
    float* queries;        // [nq][Dp]
    float* qraw;           // [nq][D] (H2D target)
    long long* probes;     // [nq][P]
    float* pdist;          // [nq][P] probe keys
    float* fcand_d;        // quantizer candidates
    long long* fcand_i;
    float* cand_d;         // scan candidates
    long long* cand_i;
    float* out_d;
    long long* out_i;
    uint32_t* out_cnt;
    uint32_t* ctr;
    PlanBufs plan;
    TcBufs tc;
    float* qdense;         // TC quantizer: [qslice][ceil(C/32)*32] approximate distances
    float* qdense_nq;      // [nq] query norms
    float2* qgsum;         // TC quantizer: [qslice][ceil(C/32)] per-group (min upper, min lower) bounds
};

struct RearrangeEvent {
    uint32_t cluster;
    uint64_t hops_before, hops_after, merges;
    double duration_us;
};

class GpuIndex {
public:
    explicit GpuIndex(const bivf_config& cfg);
    ~GpuIndex();

    const bivf_config& config() const { return cfg_; }
    uint32_t C() const { return C_; }
    uint32_t D() const { return D_; }

    void train(const float* x, uint64_t n);
    void set_centroids(const float* c);
    void get_centroids(float* out) const;
    void bulk_load(const float* x, uint64_t n, const uint32_t* assignment, const int64_t* ids);

    uint64_t insert(const float* x, uint64_t n, const int64_t* ids, int64_t* out_ids);
    void search(const float* q, uint64_t nq, uint64_t k, uint64_t nprobe, int64_t* out_ids,
                float* out_d, uint32_t* out_cnt);
    // one zero-query search of this shape on every lease (serving start-up)
    void prewarm(uint64_t nq, uint64_t k, uint64_t nprobe);
    void search_device(const float* q_dev, uint64_t nq, uint64_t k, uint64_t nprobe,
                       int64_t* ids_dev, float* d_dev, uint32_t* cnt_dev, cudaStream_t user);
    void assign(const float* y, uint64_t n, uint32_t* out);
    void probes(const float* q, uint64_t nq, uint64_t nprobe, uint32_t* out);
    uint64_t remove(const int64_t* ids, uint64_t n, uint8_t* found);

    bool exceed(uint32_t c) const;
    void rearrange(uint32_t c);
    void rearrange_sweep();
    std::vector<RearrangeEvent> take_events(size_t cap = SIZE_MAX);
    uint64_t cow_ops() const { return cow_ops_; }
    uint64_t quiescent_ops() const { return quiescent_ops_; }

    uint64_t size() const;
    uint64_t scalars_copied() const { return scalars_copied_; }
    uint64_t reallocations() const { return reallocations_; }
    // The copy-based baseline backend (baseline_index.cpp:51-103, the paper's
    // Faiss/RAFT-style extend) on device: every affected list is re-allocated at
    // old + new, its old contents copied, the new vectors appended, the old space
    // dropped.  Lists live in the offline-segment area (searched as usual).
    uint64_t extend_copy(const float* x, uint64_t n, const int64_t* ids, int64_t* out_ids);
    uint64_t list_length(uint32_t c) const;
    uint64_t offline_count(uint32_t c) const;
    uint64_t hop_count(uint32_t c) const;
    int32_t online_head(uint32_t c) const;
    uint64_t allocated_blocks() const;
    void block_header(int32_t b, int32_t* out5) const;
    void block_ids(int32_t b, int64_t* out) const;
    void block_payload(int32_t b, float* out) const;
    uint64_t cluster_contents(uint32_t c, int64_t* ids, float* vecs) const;
    std::string dump_pool() const;
    int64_t next_id() const { return next_id_; }

    void save(const std::string& path) const;
    // shard/nshards: keep only the ids with id mod nshards == shard (one shard of
    // a vector-sharded group); nshards 1 = the whole snapshot
    static std::unique_ptr<GpuIndex> load(const std::string& path, const bivf_config* ov,
                                          uint32_t shard = 0, uint32_t nshards = 1);
    // one-shot utilization alert (block_store.cpp:41-46): fired, blocks used when it fired
    void alert_state(int32_t* fired, uint64_t* used_at) const;
    // block_store.hpp set_next: raw header mutation (the reference's pool test hook)
    void block_set_next(int32_t b, int32_t next);

    // ---- one shard's part of a vector-sharded search (group.cpp), on one of
    // this index's leases: open (lease, workspace for nq rounded up to G slices,
    // gate shared) -> queries -> quantize one slice of the queries -> (the
    // caller all-gathers the probe rows) -> scan all queries -> close.
    struct ShardCtx {
        Lease* lease = nullptr;
        Workspace w{};
        std::shared_lock<std::shared_mutex> gate;
        uint32_t nq = 0, nq_pad = 0, k = 0, P = 0, slice = 0;
    };
    void shard_open(ShardCtx& s, uint64_t nq, uint64_t k, uint64_t nprobe, uint32_t G);
    void shard_quantize(ShardCtx& s, uint32_t g);  // pads every query; probes of slice g
    void shard_scan(ShardCtx& s);                  // plan + scan + refine -> s.w.out_*
    void shard_close(ShardCtx& s);
    int device() const { return device_; }

    void set_timing(bool on) { timing_ = on; }
    void set_scan_mode(int m) { scan_mode_ = m; }
    bool use_tc(uint32_t k) const;
    bool use_tc_dense(uint32_t k) const;
    void last_timings(float* out4) const;
    void record_timings(Lease& l);

private:
    // --- device storage (copies/memsets stream-ordered on data_stream_, then synced)
    cudaError_t h2d(void* dst, const void* src, size_t n) const;
    cudaError_t d2h(void* dst, const void* src, size_t n) const;
    cudaError_t dset(void* p, int v, size_t n) const;
    void alloc_device();
    void ensure_offline_capacity(uint64_t slots);
    DevLists dev_lists() const;
    InsertState insert_state();
    MirrorView mirror_view() const;
    const MirrorView* mirror_ptr() const { return mir_on_ ? &mirror_ : nullptr; }
    void rebuild_mirror();
    void build_quantizer_mirror(const float* centroids_host);
    bool use_tc_quantizer(uint32_t P) const;
    uint32_t quantizer_maxch(uint32_t nq) const;
    uint32_t quantizer_slice() const;
    DevLists quantizer_lists() const;
    void enqueue_quantizer(cudaStream_t s, uint32_t nq, uint32_t P, uint32_t fnch, Workspace& w,
                           uint32_t qbase = 0);
    void upload_centroids();

    // --- leases / maintenance fencing
    Lease* acquire_lease();
    void release_lease(Lease* l);
    Workspace carve(Lease& l, uint32_t nq, uint32_t k, uint32_t P, uint32_t maxch,
                    uint32_t fnch);
    void enqueue_probes(Lease& l, const float* q_dev_raw_piece, uint32_t q0, uint32_t m,
                        uint32_t P, uint32_t fnch, Workspace& w);
    void enqueue_scan(Lease& l, uint32_t nq, uint32_t k, uint32_t P, Workspace& w);
    // the search's device work for a small batch as a cached CUDA graph
    // (returns false when the shape is not graph-eligible: caller enqueues)
    bool graph_search(Lease& l, uint32_t m, uint32_t k, uint32_t P, Workspace& w);
    uint64_t graph_sig() const;
    void search_on(Lease* l, const float* q, uint64_t nq, uint64_t k, uint64_t nprobe, int64_t* out_ids,
                   float* out_d, uint32_t* out_cnt, double us_lease);
    void enqueue_search(Lease& l, const float* q_dev_raw, uint32_t nq, uint32_t k,
                        uint32_t P, Workspace& w);
    void begin_maintenance();   // caller holds data_mu_; takes gate_ exclusively
    void end_maintenance();
    // read-copy-update maintenance (caller holds data_mu_)
    void grace();                                   // see the header comment
    void reclaim() { if (grace_pending_) grace(); } // before reusing scratch / inactive rows
    struct ListPub {                                // a list's new published state
        uint32_t c;
        uint64_t start;
        uint32_t count;
        uint64_t row;
        uint32_t len;
    };
    void publish(const std::vector<ListPub>& pubs);
    ListPub current_pub(uint32_t c) const;
    uint64_t row_addr(uint32_t c, uint32_t sel) const;
    // write rows (logical block order) into the given row copies of lists
    void write_rows(const std::vector<uint32_t>& lists, const std::vector<std::vector<int32_t>>& rows,
                    const std::vector<uint8_t>& sel);
    void grow_rows(uint32_t need);                  // row capacity (MLB_) >= need
    void apply_block_moves(const std::vector<int32_t>& src, const std::vector<int32_t>& dst,
                           const std::vector<uint32_t>& lists);
    void copy_block_set(const std::vector<int32_t>& src, const std::vector<int32_t>& dst);
    // offline free space (slots, group aligned)
    uint64_t off_alloc(uint64_t slots);             // ~0 when none
    void off_free_add(uint64_t start, uint64_t slots);
    uint32_t off_owner(uint64_t slot) const;        // cluster whose segment holds the slot

    // --- host mirror
    void absorb_new_blocks(uint32_t cursor_old, uint32_t cursor_new);
    void refresh_lengths();
    uint32_t committed_of(int32_t b) const;
    void check_block(int32_t b) const;
    bool is_duplicate_id(int64_t id);
    void validate_search(uint64_t k, uint64_t nprobe) const;

    bivf_config cfg_;
    uint32_t C_, D_, Dp_, T_, gpb_, NB_, MLB_, MLB_cap_;
    uint32_t NS_ = 0;  // scratch blocks past the pool (arena block ids NB_ .. NB_+NS_-1)
    uint64_t PS_;
    int device_;
    int num_sms_ = 148;

    // device
    DevBuf d_cent_, d_cent_il_;
    DevBuf d_off_pay_, d_off_ids_, d_off_start_, d_off_count_;
    uint64_t off_slots_cap_ = 0;
    DevBuf d_arena_, d_bids_, d_owner_;
    // tensor-core scan mirror (mirror.cuh); allocated when the TC scan can serve this index
    DevBuf d_off_mir_, d_arena_mir_, d_off_nrm_, d_arena_nrm_, d_off_rows_, d_arena_rows_;
    bool mir_on_ = false;
    uint64_t GF_ = 0, MPS_ = 0;
    MirrorView mirror_{};
    // tensor-core coarse quantizer: the centroid set as ONE list (centred at the
    // centroid mean mu, its own scan mirror) searched by the TC filter + exact refine
    DevBuf d_q_mir_, d_q_nrm_, d_q_ids_, d_q_meta_, d_q_zero_, d_q_mu_;
    CUtensorMap map_q_{};
    bool q_tc_ok_ = false;
    DevBuf d_cursor_, d_len_, d_nblocks_, d_fail_;
    // per-list block-table rows, double buffered: [2][C][MLB_] int32; d_rowptr_[c]
    // points at copy h_sel_[c] of row c; d_ver_ is the per-list seqlock
    DevBuf d_rows_, d_rowptr_, d_ver_;
    std::vector<std::unique_ptr<DevBuf>> retired_;  // outgrown row buffers (searches may hold them)
    std::vector<uint8_t> h_sel_;
    bool grace_pending_ = false;
    uint64_t cow_ops_ = 0, quiescent_ops_ = 0;  // maintenance ops by path (tests, bench)
    void rearrange_lists(const std::vector<uint32_t>& lists);  // caller holds data_mu_  // scratch / inactive rows may still be read by searches
    bool cow_on_ = true;          // BIVF_COW=0: quiescence for every maintenance op
    bool copy_backend_ = false;   // extend_copy owns the offline area (no free-space COW)
    DevBuf s_pub_, s_rows_;
    PinBuf h_pub_;
    DevBuf d_run_, d_failfrom_, d_newlen_;
    // data-lane staging
    cudaStream_t data_stream_ = nullptr;
    int prio_hi_ = 0;
    DevBuf d_x_, d_ids_, d_asg_, d_blk_, d_did_, d_qtmp_, d_fc_d_, d_fc_i_, d_fo_d_, d_fo_i_,
        d_ctr_;
    PinBuf h_stage_;
    Lease data_lease_;  // the data lane's own workspace (insert-path TC quantizer); stream = data_stream_
    // maintenance scratch (rearrangement block moves, delete), grow-only; used
    // under data_mu_ only
    DevBuf s_rr_src_, s_rr_dst_, s_rr_pay_, s_rr_ids_;
    DevBuf s_rm_[12];

    // host mirror
    std::vector<uint32_t> h_len_, h_off_count_, h_nblocks_;
    std::vector<uint64_t> h_off_start_;
    std::map<uint64_t, uint64_t> off_free_;                       // start -> slots
    std::vector<std::pair<uint64_t, uint64_t>> off_pending_;      // retired, freed at the next grace
    std::map<uint64_t, std::pair<uint32_t, uint64_t>> off_region_;  // start -> (cluster, slots)
    std::vector<int32_t> h_prev_, h_next_, h_owner_, h_mid_;
    std::vector<uint8_t> h_merged_;
    std::vector<int32_t> h_head_, h_tail_;
    std::vector<std::vector<int32_t>> h_blocks_;  // per list, logical order (table row)
    uint32_t h_cursor_ = 0;
    bool alert_fired_ = false;
    uint64_t alert_used_ = 0;
    bool trained_ = false;

    // ids (ivf_index.cpp:107-141)
    int64_t next_id_ = 0, offline_end_ = 0;
    std::vector<std::pair<int64_t, int64_t>> auto_ranges_;
    std::unordered_set<int64_t> supplied_;
    uint64_t scalars_copied_ = 0, reallocations_ = 0;
    void grow_offline_preserving(uint64_t slots);  // copy-based extend: keep contents

    std::vector<RearrangeEvent> events_;
    std::mutex events_mu_;

    // concurrency
    mutable std::mutex data_mu_;
    std::shared_mutex gate_;
    std::mutex lease_mu_;
    std::condition_variable lease_cv_;
    std::vector<std::unique_ptr<Lease>> leases_;
    cudaEvent_t maint_evt_ = nullptr;
    std::atomic<uint64_t> maint_gen_{0};
    std::atomic<uint64_t> gen_{0};  // device-buffer generation (graph_sig)
    std::atomic<uint64_t> size_total_{0};  // stored vectors (size(), lock-free)
    void refresh_size();

    CUtensorMap map_off_{}, map_arena_{};
    CUtensorMap maps_h_[6]{};  // scan_vm_kernel's maps (make_vm_maps): offline [0, 3), arena [3, 6)
    CUtensorMap q_vm_maps_[6]{};       // scan_vm_kernel's maps over the quantizer mirror (L2)
    bool q_vm_ok_ = false;
    DevBuf d_samp_rows_, d_samp_ids_;  // seed samples (maint.cuh kSampS per list), built by bulk_load
    bool samp_on_ = false;

public:
    uint64_t seed_samples(int64_t* out, uint64_t cap) const;

private:
    bool maps_h_ok_ = false;
    bool tc_ok_ = false;
    int scan_mode_ = 0;  // 0 auto, 1 CUDA-core only, 2 tensor-core when supported,
                         // 3 / 4 auto with the list scan forced vector- / query-major
    std::atomic<bool> graphs_on_{true};  // BIVF_GRAPHS=0 disables; a failed capture too
    bool timing_ = false;
    float last_ms_[4] = {-1, -1, -1, -1};
};

// helpers implemented in host_algos.cpp
void synthetic_dataset(uint64_t n, uint64_t dim, uint64_t comps, uint64_t seed, float* out);
uint64_t kmeans_gpu(const float* points, uint64_t n, uint64_t dim, uint64_t k, uint64_t iters,
                    uint64_t seed, int device, float* centroids, uint32_t* assignment);
float host_l2(const float* a, const float* b, uint32_t dim);
void exact_knn_gpu(const float* base, uint64_t n, uint64_t dim, const float* q, uint64_t nq, uint64_t k,
                   int metric, int device, int64_t* ids, float* d, uint32_t* cnt);

}  // namespace bivf
