/*
 * bivf.h — C-ABI of the B200-native online IVF-Flat path (libbivf_gpu.so).
 *
 * This is the drop-in boundary for the reference's index plugin API
 * (blockivf::VectorIndex, /root/reference/proj/include/blockivf/vector_index.hpp:19-44,
 * and the concrete ClusterIndex surface, include/blockivf/ivf_index.hpp:47-103).
 * Every entry point cites the reference interface it replaces.  Plain
 * pointers and sizes only; all array arguments are HOST memory unless the
 * name says _device.  No exceptions cross the ABI: every call returns a
 * bivf_status and bivf_last_error() holds the thread-local message.
 *
 * Status -> reference exception (so C++/Python wrappers can rethrow):
 *   BIVF_EINVAL   std::invalid_argument          (ivf_index.cpp:126-129, :266-269)
 *   BIVF_EPOOL    PoolExhaustedError(inserted)    (types.hpp:19-30)
 *   BIVF_ECORRUPT CorruptListError                (types.hpp:34-36)
 *   BIVF_ERANGE   std::out_of_range               (ivf_index.cpp:477, block_store.cpp:51)
 *   BIVF_ELOGIC   std::logic_error                (block_store.cpp:58-62)
 *   BIVF_EIO      std::runtime_error (snapshot)   (ivf_index.cpp:537, :569-575)
 *   BIVF_ECUDA    CUDA/driver failure (no GPU, launch error) — no CPU fallback exists
 *   BIVF_EBUSY    all leases busy (executor fail-fast reject, executor.cpp:165-170)
 */
#ifndef BIVF_H
#define BIVF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    BIVF_OK = 0,
    BIVF_EINVAL = 1,
    BIVF_EPOOL = 2,
    BIVF_ECORRUPT = 3,
    BIVF_ERANGE = 4,
    BIVF_ELOGIC = 5,
    BIVF_EIO = 6,
    BIVF_ECUDA = 7,
    BIVF_EBUSY = 8,
    BIVF_ENOMEM = 9
} bivf_status;

typedef enum { BIVF_METRIC_L2 = 0, BIVF_METRIC_IP = 1 } bivf_metric;

/* IndexConfig + PoolConfig (ivf_index.hpp:20-30, block_store.hpp:16-33), plus
 * device placement.  Zero fields take the reference defaults noted. */
typedef struct {
    uint64_t num_clusters;        /* N (default 100) */
    uint64_t dim;                 /* D (required) */
    uint64_t nprobe_default;      /* default 8 */
    uint64_t rearrange_threshold; /* T'_m (default 256) */
    uint64_t kmeans_iters;        /* default 25 */
    uint64_t kmeans_seed;         /* default 42 (use kmeans_seed_set=1 to pass 0) */
    uint64_t num_blocks;          /* |P| (default 1024) */
    uint64_t block_capacity;      /* T_m (default 64) */
    double alert_watermark;       /* default 0.9 */
    int32_t metric;               /* bivf_metric (extension; default L2) */
    int32_t device;               /* CUDA device ordinal (default 0) */
    uint32_t num_leases;          /* search leases = streams+workspaces (default 32) */
    uint32_t max_list_blocks;     /* per-list block-table row length (default num_blocks) */
    uint32_t kmeans_seed_set;     /* 1: kmeans_seed is explicit even if 0 */
    uint32_t reserved[7];
} bivf_config;

typedef struct bivf_index bivf_index;

/* thread-local message of the last failing call on this thread */
const char* bivf_last_error(void);
/* "bivf <version> sm_100a" */
const char* bivf_version(void);
/* number of visible CUDA devices (0 on a host without GPU) */
int bivf_device_count(void);
/* Page-locked host memory for search inputs/outputs: bivf_search DMAs such
 * buffers directly (no staging copy).  Plain host memory works too. */
bivf_status bivf_host_alloc(size_t bytes, void** out);
bivf_status bivf_host_free(void* p);

/* ---- lifecycle ------------------------------------------------------- */
/* ClusterIndex(IndexConfig) storage (ivf_index.cpp:36-45): allocates the whole
 * device arena up front (block_store.cpp:19-29). */
bivf_status bivf_create(const bivf_config* cfg, bivf_index** out);
bivf_status bivf_destroy(bivf_index* h);
bivf_status bivf_get_config(const bivf_index* h, bivf_config* out);

/* ClusterIndex(offline, n, cfg) (ivf_index.cpp:47-59): k-means (kmeans.cpp:31-142,
 * assignment sweeps on the GPU, bit-identical to the reference) then the
 * offline bulk load; ids 0..n-1, auto ids continue at n. */
bivf_status bivf_train(bivf_index* h, const float* x, uint64_t n);
/* centroids row-major [num_clusters x dim] (ClusterIndex::centroids()) */
bivf_status bivf_set_centroids(bivf_index* h, const float* centroids);
bivf_status bivf_get_centroids(const bivf_index* h, float* out);
/* build_offline (ivf_index.cpp:61-82).  assignment NULL -> assign on device;
 * ids NULL -> 0..n-1 (offline range, like the trained constructor), else the
 * given ids are recorded as supplied ids. */
bivf_status bivf_bulk_load(bivf_index* h, const float* x, uint64_t n, const uint32_t* assignment,
                           const int64_t* ids);

/* BIVFSNAP v1 (ivf_index.cpp:515-619; format proj/README.md:132-150) */
bivf_status bivf_save_snapshot(const bivf_index* h, const char* path);
/* cfg_override may be NULL; its device / num_leases / max_list_blocks fields apply */
bivf_status bivf_load_snapshot(const char* path, const bivf_config* cfg_override,
                               bivf_index** out);

/* One shard of a vector-sharded group from a whole-index snapshot: only the
 * vectors with id mod nshards == shard are loaded (every shard
 * keeps all centroids and the snapshot's next_id). */
bivf_status bivf_load_snapshot_shard(const char* path, uint32_t shard, uint32_t nshards,
                                     const bivf_config* cfg_override, bivf_index** out);

/* ---- the hot path ----------------------------------------------------- */
/* VectorIndex::insert (vector_index.hpp:25-27, ivf_index.cpp:122-164).
 * ids NULL -> contiguous auto ids.  out_ids[i] = id or -1 (rejected duplicate
 * or failed on pool exhaustion).  Returns BIVF_EPOOL with *inserted set when
 * the pool ran out mid-batch (PoolExhaustedError(inserted)). */
bivf_status bivf_add(bivf_index* h, const float* x, uint64_t n, const int64_t* ids,
                     int64_t* out_ids, uint64_t* inserted);
/* Batched VectorIndex::search (vector_index.hpp:28-29, ivf_index.cpp:262-298):
 * nq queries, row-major.  out_ids/out_dists are [nq x k]; out_counts[q] =
 * min(k, scanned); unused tail entries are id -1.  Distances are
 * bit-identical to l2_sqr_strided (L2) or -<q,x> (IP).  k <= 256, and nprobe
 * <= 256 or nprobe == num_clusters. */
bivf_status bivf_search(bivf_index* h, const float* queries, uint64_t nq, uint64_t k,
                        uint64_t nprobe, int64_t* out_ids, float* out_dists, uint32_t* out_counts);
/* Same with device-resident inputs/outputs on the caller's CUDA stream
 * (cudaStream_t passed as void*; NULL = legacy default).  Asynchronous. */
bivf_status bivf_search_device(bivf_index* h, const float* queries_device, uint64_t nq,
                               uint64_t k, uint64_t nprobe, int64_t* out_ids_device,
                               float* out_dists_device, uint32_t* out_counts_device,
                               void* stream);
/* ClusterIndex::assign (ivf_index.cpp:93-105) for n vectors */
bivf_status bivf_assign(bivf_index* h, const float* y, uint64_t n, uint32_t* out);
/* probe sets (ivf_index.cpp:271-276): out [nq x nprobe] ascending by (key, cluster)
 * (nprobe == num_clusters > 256: every cluster, in cluster-id order) */
bivf_status bivf_probes(bivf_index* h, const float* queries, uint64_t nq, uint64_t nprobe,
                        uint32_t* out);
/* Delete (extension; the reference has none; rules in DESIGN.md
 * §Delete): in request order, fill each hole with the last vector of its part
 * (offline segment or online list).  found may be NULL. */
/* The copy-based baseline backend (blockivf::BaselineIndex::insert,
 * baseline_index.cpp:51-103) on device: each affected list is re-allocated at
 * old + new, the old contents copied, the new vectors appended.  Searched by
 * bivf_search like any index.  Counters: bivf_scalars_copied, bivf_reallocations. */
bivf_status bivf_extend_copy(bivf_index* h, const float* x, uint64_t n, const int64_t* ids,
                             int64_t* out_ids, uint64_t* inserted);
bivf_status bivf_reallocations(const bivf_index* h, uint64_t* out);
bivf_status bivf_remove(bivf_index* h, const int64_t* ids, uint64_t n, uint64_t* removed,
                        uint8_t* found);

/* ---- rearrangement (Alg. 3) -------------------------------------------- */
bivf_status bivf_exceed(const bivf_index* h, uint32_t cluster, int* out);     /* ivf_index.cpp:300-311 */
bivf_status bivf_rearrange(bivf_index* h, uint32_t cluster);                  /* ivf_index.cpp:476-505 */
bivf_status bivf_rearrange_sweep(bivf_index* h);                              /* ivf_index.cpp:507-511 */
/* RearrangeEvent (ivf_index.hpp:33-39): 5 doubles per event (cluster,
 * hops_before, hops_after, merges, duration_us).  Takes the oldest
 * min(cap, pending) events (count via *n); the rest stay queued, so a caller
 * loops until *n < cap. */
bivf_status bivf_take_rearrange_events(bivf_index* h, double* out5, uint64_t cap, uint64_t* n);

/* ---- introspection (ivf_index.hpp:84-103, block_store.hpp:75-132) -------- */
bivf_status bivf_size(const bivf_index* h, uint64_t* out);
bivf_status bivf_scalars_copied(const bivf_index* h, uint64_t* out);
/* maintenance operations (delete / rearrangement batches) that ran as
 * read-copy-update (searches never wait) and that fell back to quiescence
 * (oversized: more blocks than the scratch area, no free offline region) */
bivf_status bivf_cow_ops(const bivf_index* h, uint64_t* out);
bivf_status bivf_quiescent_ops(const bivf_index* h, uint64_t* out);
bivf_status bivf_list_length(const bivf_index* h, uint32_t cluster, uint64_t* out);
bivf_status bivf_offline_count(const bivf_index* h, uint32_t cluster, uint64_t* out);
bivf_status bivf_hop_count(const bivf_index* h, uint32_t cluster, uint64_t* out);
bivf_status bivf_online_head(const bivf_index* h, uint32_t cluster, int32_t* out);
bivf_status bivf_allocated_blocks(const bivf_index* h, uint64_t* out);
/* header: prev, next, size(committed), owner, merged_with_prev */
bivf_status bivf_block_header(const bivf_index* h, int32_t block, int32_t* out5);
bivf_status bivf_block_ids(const bivf_index* h, int32_t block, int64_t* out /* [T_m] */);
bivf_status bivf_block_payload(const bivf_index* h, int32_t block,
                               float* out /* [ceil(T_m/32)*32*D] */);
/* offline then online contents (ivf_index.cpp:505-523); ids NULL -> count only */
bivf_status bivf_cluster_contents(const bivf_index* h, uint32_t cluster, int64_t* ids,
                                  float* vecs, uint64_t* count);
/* dump_pool text (block_store.cpp:188-201); *len = bytes needed incl. NUL */
bivf_status bivf_dump_pool(const bivf_index* h, char* buf, uint64_t cap, uint64_t* len);
bivf_status bivf_next_id(const bivf_index* h, int64_t* out);
/* one-shot utilization alert (block_store.cpp:41-46): *fired, and the number of
 * blocks in use at the allocation that first exceeded the watermark */
bivf_status bivf_pool_alert(const bivf_index* h, int32_t* fired, uint64_t* used_at);
/* the list scan's seed samples: per list up to 32 ids of
 * central offline vectors, -1 for empty / deleted entries; writes
 * min(cap, num_clusters * 32) ids (list-major), *n = num_clusters * 32, or 0
 * when the index keeps no samples */
bivf_status bivf_seed_samples(const bivf_index* h, int64_t* out, uint64_t cap, uint64_t* n);
/* block_store.hpp set_next: raw header-link mutation (the reference pool's test
 * hook; traversals then report cycles as BIVF_ECORRUPT) */
bivf_status bivf_block_set_next(bivf_index* h, int32_t block, int32_t next);

/* ---- data helpers (either side of the path) ----------------------------- */
/* synthetic_dataset (dataset.cpp:92-112): same std::mt19937_64 stream, same
 * libstdc++ distributions -> identical bits to the reference on this image. */
bivf_status bivf_synthetic_dataset(uint64_t n, uint64_t dim, uint64_t components, uint64_t seed,
                                   float* out);
/* k-means (kmeans.cpp:31-142): seeding + assignment sweeps on device, the
 * double-precision updates on the host in the reference's order. */
bivf_status bivf_kmeans(const float* points, uint64_t n, uint64_t dim, uint64_t k,
                        uint64_t max_iters, uint64_t seed, int32_t device, float* centroids,
                        uint32_t* assignment, uint64_t* iters_run);

/* Exact k nearest neighbours by brute force (oracle.cpp:11-49 exact_knn):
 * sequential fp32 distances (L2: distance.hpp:11-18; IP: key = -q.x) over rows
 * 0..n-1, ordered by (key, row id); counts = min(k, n).  k <= 256.  Ground
 * truth for recall@k at scale, on the GPU (host buffers). */
bivf_status bivf_exact_knn(const float* base, uint64_t n, uint64_t dim, const float* queries,
                           uint64_t nq, uint64_t k, int32_t metric, int32_t device, int64_t* out_ids,
                           float* out_dists, uint32_t* out_counts);

/* ---- multi-GPU merge (north star (5)) ------------------------------------ */
/* Merge G per-shard top-k lists ([G][nq][k], ascending runs, id -1 = empty)
 * into the global top-k under (dist, id) order — the step after the NCCL
 * all-gather of per-GPU results.  Device pointers, async on `stream`. */
bivf_status bivf_merge_topk_device(int32_t device, const float* dists, const int64_t* ids,
                                   uint64_t G, uint64_t nq, uint64_t k, float* out_dists,
                                   int64_t* out_ids, uint32_t* out_counts, void* stream);

/* ---- vector-sharded groups (north star (5)) ------------------ */
/* Shard g of a G-shard group owns the ids with id mod G == g; every shard holds
 * all centroids, so the merged top-k equals the single index's bit for bit.
 * A search splits the coarse quantizer by queries (shard g computes the probes
 * of query slice g), all-gathers the probe rows, scans every shard's lists for
 * the whole batch, all-gathers the local top-k lists and merges them on device
 * (bivf_merge_topk_device's kernel).  Transports:
 *   bivf_group_create_local: G shard handles of this process (any devices, one
 *     device repeated included); peer copies between the shards' lease streams.
 *   bivf_group_create_nccl: this process's shard is rank `rank` of `nranks`;
 *     ncclAllGather / ncclAllReduce on the lease stream (libnccl loaded at run
 *     time).  `uid128` = bivf_nccl_unique_id() of rank 0, broadcast by the caller.
 *     `channels` communicators (ncclCommSplit): calls on one channel must be
 *     issued in the same order on every rank; concurrent callers use distinct
 *     channels (channel 0 also carries the all-reduces of inserts / deletes).  Every rank passes the same queries / insert batch / delete ids
 *     and receives the whole result.
 * Inserts: auto ids are the group's contiguous next_id range (ivf_index.cpp:
 * 133-141); each shard inserts its rows with explicit ids.  The group does not
 * own its shards: destroy the group first. */
typedef struct bivf_group bivf_group;
bivf_status bivf_nccl_unique_id(void* out128);
bivf_status bivf_group_create_local(bivf_index* const* shards, uint32_t nshards, bivf_group** out);
bivf_status bivf_group_create_nccl(bivf_index* shard, const void* uid128, int32_t nranks, int32_t rank,
                                   uint32_t channels, bivf_group** out);
void bivf_group_destroy(bivf_group* g);
bivf_status bivf_group_size(const bivf_group* g, uint32_t* out);
bivf_status bivf_group_search(bivf_group* g, const float* queries, uint64_t nq, uint64_t k,
                              uint64_t nprobe, int64_t* out_ids, float* out_dists,
                              uint32_t* out_counts, uint32_t channel);
/* NCCL groups: device buffers on this rank's device, ordered after / before `stream` */
bivf_status bivf_group_search_device(bivf_group* g, const float* queries_dev, uint64_t nq,
                                     uint64_t k, uint64_t nprobe, int64_t* ids_dev, float* dists_dev,
                                     uint32_t* counts_dev, void* stream, uint32_t channel);
bivf_status bivf_group_insert(bivf_group* g, const float* vectors, uint64_t n, const int64_t* ids,
                              int64_t* out_ids, uint64_t* inserted);
bivf_status bivf_group_remove(bivf_group* g, const int64_t* ids, uint64_t n, uint64_t* removed,
                              uint8_t* found);

/* ---- executor: the multi-lane resource pool (Alg. 4) ---------------------- */
/* Mirrors blockivf::Executor (include/blockivf/executor.hpp:21-196,
 * src/executor.cpp): search lanes (thread + GPU lease each) with fail-fast
 * reject, a dedicated insertion lane with the 128-multiple / cap / interval
 * batcher, serialized FIFO mode, tickets with submit/start/end stamps. */
typedef struct bivf_executor bivf_executor;
typedef struct bivf_ticket bivf_ticket;
typedef struct {
    uint32_t num_lanes;          /* default 32 */
    uint32_t central_grants;     /* default 4 */
    uint64_t lane_cache_bytes;   /* default 512 KiB (paper 50 MB) */
    uint64_t central_grant_bytes;/* default 2 MiB (paper 200 MB) */
    uint32_t flush_interval_ms;  /* default 1000 */
    uint32_t batch_multiple;     /* default 128 */
    uint32_t batch_cap;          /* default 1024 */
    uint32_t max_search_batch;   /* default 10 */
    int32_t serialized;          /* 0 parallel, 1 serialized FIFO */
    uint32_t reserved[5];
} bivf_executor_config;
typedef struct {
    int32_t status;   /* 0 pending, 1 done, 2 rejected, 3 error */
    int32_t type;     /* 0 search, 1 insert */
    int32_t lane;     /* search lane, num_lanes = data lane */
    uint32_t nq, k;   /* search shape */
    uint64_t n;       /* insert: vectors */
    double latency_us, queue_us, exec_us;
} bivf_ticket_info;
typedef struct {
    double qps_search, qps_insert, duration_s;
    uint32_t search_batch, insert_batch, k, nprobe;
    uint64_t seed;
    int32_t poisson;
    uint32_t reserved[5];
} bivf_replay_spec;

bivf_status bivf_executor_create(bivf_index* h, const bivf_executor_config* cfg,
                                 bivf_executor** out);                        /* Executor ctor */
bivf_status bivf_executor_destroy(bivf_executor* e);                          /* shutdown + free */
bivf_status bivf_executor_submit_search(bivf_executor* e, const float* queries, uint64_t nq,
                                        uint64_t k, uint64_t nprobe, bivf_ticket** out);
bivf_status bivf_executor_submit_insert(bivf_executor* e, const float* x, uint64_t n,
                                        const int64_t* ids, bivf_ticket** out);
bivf_status bivf_executor_flush(bivf_executor* e);                            /* flush_insertions */
bivf_status bivf_executor_set_mode(bivf_executor* e, int serialized);         /* set_mode */
bivf_status bivf_executor_shutdown(bivf_executor* e);
/* rejected, completed, in_flight, grants_outstanding, grants_total,
 * lane_cache_allocations, lane_double_hold_violations, largest_flush */
bivf_status bivf_executor_stats(const bivf_executor* e, uint64_t* out8);
bivf_status bivf_ticket_wait(bivf_ticket* t, bivf_ticket_info* info);       /* Ticket::get */
/* search: ids/dists [nq x k] + counts [nq]; insert: ids [n] (dists/counts ignored) */
bivf_status bivf_ticket_results(bivf_ticket* t, int64_t* ids, float* dists, uint32_t* counts);
bivf_status bivf_ticket_error(bivf_ticket* t, char* buf, uint64_t cap);
bivf_status bivf_ticket_free(bivf_ticket* t);
/* open-loop replay (workload.cpp:114-269): per-request latencies in us
 * (-1 rejected, -2 error), issue order */
bivf_status bivf_replay(bivf_executor* e, const bivf_replay_spec* spec, const float* queries,
                        uint64_t nqueries, const float* inserts, uint64_t ninserts,
                        double* search_lat_us, uint64_t search_cap, uint64_t* n_search,
                        double* insert_lat_us, uint64_t insert_cap, uint64_t* n_insert,
                        uint64_t* rejected, uint64_t* errors);

/* ---- instrumentation ------------------------------------------------------ */
/* kernel launches issued by this library since load (bench's gpu_launches) */
uint64_t bivf_kernel_launches(void);
/* serving start-up: one search of nq zero queries (k, nprobe) on every lease,
 * all leases held at once, so each lease's stream, workspace, pinned staging and
 * CUDA graph for that request shape exist before traffic (no first-use stalls
 * when load first spreads over many leases).  Replaces nothing in the reference
 * (its executor creates every lane and its cached scratch up front,
 * executor.cpp:103-125). */
bivf_status bivf_prewarm(bivf_index* h, uint64_t nq, uint64_t k, uint64_t nprobe);
/* scan kernel selection: 0 auto (tensor-core filtered scan when supported:
 * L2, k <= 32, 8 <= D <= 128), 1 CUDA-core exact scan only, 2 = auto,
 * 3 / 4 = auto with the L2 list scan forced onto the vector-major /
 * query-major tensor-core kernel (auto picks by pairs per list) */
bivf_status bivf_set_scan_mode(bivf_index* h, int mode);
/* enable CUDA-event timing of the search phases (on the lease stream) */
bivf_status bivf_set_timing(bivf_index* h, int enable);
/* device ms of the last timed search slice: quantizer, plan, scan kernel, merge */
bivf_status bivf_last_timings(const bivf_index* h, float* out4);

#ifdef __cplusplus
}
#endif
#endif /* BIVF_H */
