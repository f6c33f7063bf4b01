// extern "C" boundary (include/bivf.h).  Every entry point catches and maps
// C++ exceptions to bivf_status + a thread-local message; nothing throws
// across the ABI.
#include <cstring>
#include <functional>
#include <string>

#include "../../include/bivf.h"
#include "executor.h"
#include "index.h"
#include "launches.h"
#include "maint.cuh"

using bivf::Error;
using bivf::GpuIndex;

struct bivf_index {
    std::unique_ptr<GpuIndex> impl;
};
struct bivf_executor {
    std::unique_ptr<bivf::Executor> impl;
};
struct bivf_ticket {
    bivf::Ticket t;
};

namespace {
thread_local std::string g_err;

bivf_status fail(bivf_status s, const char* m) {
    g_err = m;
    return s;
}

template <class F>
bivf_status guard(F&& f) {
    try {
        f();
        return BIVF_OK;
    } catch (const Error& e) {
        return fail(e.code, e.what());
    } catch (const std::bad_alloc&) {
        return fail(BIVF_ENOMEM, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(BIVF_ELOGIC, e.what());
    }
}

GpuIndex& I(bivf_index* h) {
    if (!h || !h->impl) throw Error(BIVF_EINVAL, "null index handle");
    return *h->impl;
}
const GpuIndex& I(const bivf_index* h) {
    if (!h || !h->impl) throw Error(BIVF_EINVAL, "null index handle");
    return *h->impl;
}
template <class T>
void need(const T* p, const char* what) {
    if (!p) throw Error(BIVF_EINVAL, std::string(what) + " must not be NULL");
}
}  // namespace

namespace bivf {
// shared with group.cpp
GpuIndex& index_of(bivf_index* h) { return I(h); }
bivf_status run_guarded(const std::function<void()>& f) { return guard(f); }
}  // namespace bivf

extern "C" {

const char* bivf_last_error(void) { return g_err.c_str(); }
const char* bivf_version(void) { return "bivf 0.1.0 sm_100a"; }
int bivf_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}
uint64_t bivf_kernel_launches(void) { return bivf::g_launches.load(); }

bivf_status bivf_host_alloc(size_t bytes, void** out) {
    return guard([&] {
        need(out, "out");
        *out = nullptr;
        const cudaError_t e = cudaHostAlloc(out, std::max<size_t>(bytes, 1), cudaHostAllocPortable);
        if (e != cudaSuccess) {
            cudaGetLastError();
            throw bivf::Error(BIVF_ECUDA, std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
        }
    });
}

bivf_status bivf_host_free(void* p) {
    return guard([&] {
        if (p) cudaFreeHost(p);
    });
}

bivf_status bivf_create(const bivf_config* cfg, bivf_index** out) {
    return guard([&] {
        need(cfg, "cfg");
        need(out, "out");
        *out = nullptr;
        auto h = new bivf_index;
        try {
            h->impl = std::make_unique<GpuIndex>(*cfg);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

bivf_status bivf_destroy(bivf_index* h) {
    return guard([&] { delete h; });
}

bivf_status bivf_get_config(const bivf_index* h, bivf_config* out) {
    return guard([&] {
        need(out, "out");
        *out = I(h).config();
    });
}

bivf_status bivf_train(bivf_index* h, const float* x, uint64_t n) {
    return guard([&] {
        need(x, "x");
        I(h).train(x, n);
    });
}

bivf_status bivf_set_centroids(bivf_index* h, const float* c) {
    return guard([&] {
        need(c, "centroids");
        I(h).set_centroids(c);
    });
}

bivf_status bivf_get_centroids(const bivf_index* h, float* out) {
    return guard([&] {
        need(out, "out");
        I(h).get_centroids(out);
    });
}

bivf_status bivf_bulk_load(bivf_index* h, const float* x, uint64_t n, const uint32_t* asg,
                           const int64_t* ids) {
    return guard([&] {
        if (n) need(x, "x");
        I(h).bulk_load(x, n, asg, ids);
    });
}

bivf_status bivf_save_snapshot(const bivf_index* h, const char* path) {
    return guard([&] {
        need(path, "path");
        I(h).save(path);
    });
}

bivf_status bivf_load_snapshot(const char* path, const bivf_config* ov, bivf_index** out) {
    return guard([&] {
        need(path, "path");
        need(out, "out");
        *out = nullptr;
        auto h = new bivf_index;
        try {
            h->impl = GpuIndex::load(path, ov);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

bivf_status bivf_load_snapshot_shard(const char* path, uint32_t shard, uint32_t nshards,
                                     const bivf_config* ov, bivf_index** out) {
    return guard([&] {
        need(path, "path");
        need(out, "out");
        *out = nullptr;
        auto h = new bivf_index;
        try {
            h->impl = GpuIndex::load(path, ov, shard, nshards);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

bivf_status bivf_seed_samples(const bivf_index* h, int64_t* out, uint64_t cap, uint64_t* n) {
    return guard([&] {
        need(n, "n");
        *n = I(h).seed_samples(out, cap);
    });
}

bivf_status bivf_pool_alert(const bivf_index* h, int32_t* fired, uint64_t* used_at) {
    return guard([&] { I(h).alert_state(fired, used_at); });
}

bivf_status bivf_block_set_next(bivf_index* h, int32_t block, int32_t next) {
    return guard([&] { I(h).block_set_next(block, next); });
}

bivf_status bivf_exact_knn(const float* base, uint64_t n, uint64_t dim, const float* queries,
                           uint64_t nq, uint64_t k, int32_t metric, int32_t device, int64_t* out_ids,
                           float* out_d, uint32_t* out_counts) {
    return guard([&] {
        if (n) need(base, "base");
        if (nq) {
            need(queries, "queries");
            need(out_ids, "out_ids");
            need(out_d, "out_dists");
        }
        bivf::exact_knn_gpu(base, n, dim, queries, nq, k, metric, device, out_ids, out_d, out_counts);
    });
}

bivf_status bivf_add(bivf_index* h, const float* x, uint64_t n, const int64_t* ids,
                     int64_t* out_ids, uint64_t* inserted) {
    if (inserted) *inserted = 0;
    try {
        if (n) {
            need(x, "x");
            need(out_ids, "out_ids");
        }
        const uint64_t r = I(h).insert(x, n, ids, out_ids);
        if (inserted) *inserted = r;
        return BIVF_OK;
    } catch (const Error& e) {
        if (inserted) *inserted = e.inserted;
        return fail(e.code, e.what());
    } catch (const std::exception& e) {
        return fail(BIVF_ELOGIC, e.what());
    }
}

bivf_status bivf_extend_copy(bivf_index* h, const float* x, uint64_t n, const int64_t* ids,
                             int64_t* out_ids, uint64_t* inserted) {
    if (inserted) *inserted = 0;
    return guard([&] {
        if (n) {
            need(x, "x");
            need(out_ids, "out_ids");
        }
        const uint64_t r = I(h).extend_copy(x, n, ids, out_ids);
        if (inserted) *inserted = r;
    });
}

bivf_status bivf_search(bivf_index* h, const float* q, uint64_t nq, uint64_t k, uint64_t nprobe,
                        int64_t* out_ids, float* out_d, uint32_t* out_cnt) {
    return guard([&] {
        if (nq) {
            need(q, "queries");
            need(out_ids, "out_ids");
            need(out_d, "out_dists");
        }
        I(h).search(q, nq, k, nprobe, out_ids, out_d, out_cnt);
    });
}

bivf_status bivf_search_device(bivf_index* h, const float* q, uint64_t nq, uint64_t k,
                               uint64_t nprobe, int64_t* ids, float* d, uint32_t* cnt,
                               void* stream) {
    return guard([&] {
        if (nq) {
            need(q, "queries_device");
            need(ids, "out_ids_device");
            need(d, "out_dists_device");
        }
        I(h).search_device(q, nq, k, nprobe, ids, d, cnt, static_cast<cudaStream_t>(stream));
    });
}

bivf_status bivf_assign(bivf_index* h, const float* y, uint64_t n, uint32_t* out) {
    return guard([&] {
        if (n) {
            need(y, "y");
            need(out, "out");
        }
        I(h).assign(y, n, out);
    });
}

bivf_status bivf_probes(bivf_index* h, const float* q, uint64_t nq, uint64_t nprobe,
                        uint32_t* out) {
    return guard([&] {
        if (nq) {
            need(q, "queries");
            need(out, "out");
        }
        I(h).probes(q, nq, nprobe, out);
    });
}

bivf_status bivf_remove(bivf_index* h, const int64_t* ids, uint64_t n, uint64_t* removed,
                        uint8_t* found) {
    return guard([&] {
        if (n) need(ids, "ids");
        const uint64_t r = I(h).remove(ids, n, found);
        if (removed) *removed = r;
    });
}

bivf_status bivf_exceed(const bivf_index* h, uint32_t c, int* out) {
    return guard([&] {
        need(out, "out");
        *out = I(h).exceed(c) ? 1 : 0;
    });
}

bivf_status bivf_rearrange(bivf_index* h, uint32_t c) {
    return guard([&] { I(h).rearrange(c); });
}

bivf_status bivf_rearrange_sweep(bivf_index* h) {
    return guard([&] { I(h).rearrange_sweep(); });
}

bivf_status bivf_take_rearrange_events(bivf_index* h, double* out5, uint64_t cap, uint64_t* n) {
    return guard([&] {
        need(n, "n");
        auto ev = I(h).take_events(out5 ? (size_t)cap : 0);
        uint64_t m = 0;
        for (auto& e : ev) {
            out5[5 * m + 0] = e.cluster;
            out5[5 * m + 1] = (double)e.hops_before;
            out5[5 * m + 2] = (double)e.hops_after;
            out5[5 * m + 3] = (double)e.merges;
            out5[5 * m + 4] = e.duration_us;
            ++m;
        }
        *n = m;
    });
}

#define BIVF_GETTER(name, expr)                          \
    bivf_status name(const bivf_index* h, uint64_t* out) { \
        return guard([&] {                               \
            need(out, "out");                            \
            *out = (expr);                               \
        });                                              \
    }
BIVF_GETTER(bivf_size, I(h).size())
BIVF_GETTER(bivf_scalars_copied, I(h).scalars_copied())
BIVF_GETTER(bivf_reallocations, I(h).reallocations())
BIVF_GETTER(bivf_cow_ops, I(h).cow_ops())
BIVF_GETTER(bivf_quiescent_ops, I(h).quiescent_ops())
BIVF_GETTER(bivf_allocated_blocks, I(h).allocated_blocks())
#undef BIVF_GETTER

bivf_status bivf_list_length(const bivf_index* h, uint32_t c, uint64_t* out) {
    return guard([&] {
        need(out, "out");
        *out = I(h).list_length(c);
    });
}
bivf_status bivf_offline_count(const bivf_index* h, uint32_t c, uint64_t* out) {
    return guard([&] {
        need(out, "out");
        *out = I(h).offline_count(c);
    });
}
bivf_status bivf_hop_count(const bivf_index* h, uint32_t c, uint64_t* out) {
    return guard([&] {
        need(out, "out");
        *out = I(h).hop_count(c);
    });
}
bivf_status bivf_online_head(const bivf_index* h, uint32_t c, int32_t* out) {
    return guard([&] {
        need(out, "out");
        *out = I(h).online_head(c);
    });
}
bivf_status bivf_block_header(const bivf_index* h, int32_t b, int32_t* out5) {
    return guard([&] {
        need(out5, "out");
        I(h).block_header(b, out5);
    });
}
bivf_status bivf_block_ids(const bivf_index* h, int32_t b, int64_t* out) {
    return guard([&] {
        need(out, "out");
        I(h).block_ids(b, out);
    });
}
bivf_status bivf_block_payload(const bivf_index* h, int32_t b, float* out) {
    return guard([&] {
        need(out, "out");
        I(h).block_payload(b, out);
    });
}
bivf_status bivf_cluster_contents(const bivf_index* h, uint32_t c, int64_t* ids, float* vecs,
                                  uint64_t* count) {
    return guard([&] {
        need(count, "count");
        if (ids) need(vecs, "vecs");
        *count = I(h).cluster_contents(c, ids, vecs);
    });
}
bivf_status bivf_dump_pool(const bivf_index* h, char* buf, uint64_t cap, uint64_t* len) {
    return guard([&] {
        const std::string s = I(h).dump_pool();
        if (len) *len = s.size() + 1;
        if (buf && cap) {
            const size_t m = std::min<size_t>(cap - 1, s.size());
            std::memcpy(buf, s.data(), m);
            buf[m] = 0;
        }
    });
}
bivf_status bivf_next_id(const bivf_index* h, int64_t* out) {
    return guard([&] {
        need(out, "out");
        *out = I(h).next_id();
    });
}

bivf_status bivf_synthetic_dataset(uint64_t n, uint64_t dim, uint64_t comps, uint64_t seed,
                                   float* out) {
    return guard([&] {
        if (n) need(out, "out");
        bivf::synthetic_dataset(n, dim, comps, seed, out);
    });
}

bivf_status bivf_kmeans(const float* pts, uint64_t n, uint64_t dim, uint64_t k, uint64_t iters,
                        uint64_t seed, int32_t device, float* cent, uint32_t* asg,
                        uint64_t* iters_run) {
    return guard([&] {
        need(pts, "points");
        need(cent, "centroids");
        need(asg, "assignment");
        const uint64_t r = bivf::kmeans_gpu(pts, n, dim, k, iters, seed, device, cent, asg);
        if (iters_run) *iters_run = r;
    });
}

bivf_status bivf_merge_topk_device(int32_t device, const float* dists, const int64_t* ids,
                                   uint64_t G, uint64_t nq, uint64_t k, float* od, int64_t* oi,
                                   uint32_t* oc, void* stream) {
    return guard([&] {
        if (k < 1 || k > 256) throw Error(BIVF_EINVAL, "merge_topk: k out of [1, 256]");
        BIVF_CUDA(cudaSetDevice(device));
        BIVF_CUDA(bivf::launch_merge_shards(dists, reinterpret_cast<const long long*>(ids),
                                            (uint32_t)G, (uint32_t)nq, (uint32_t)k, od,
                                            reinterpret_cast<long long*>(oi), oc,
                                            static_cast<cudaStream_t>(stream)));
    });
}

bivf_status bivf_executor_create(bivf_index* h, const bivf_executor_config* cfg,
                                 bivf_executor** out) {
    return guard([&] {
        need(out, "out");
        *out = nullptr;
        bivf::ExecConfig c;
        if (cfg) {
            if (cfg->num_lanes) c.num_lanes = cfg->num_lanes;
            if (cfg->central_grants) c.central_grants = cfg->central_grants;
            if (cfg->lane_cache_bytes) c.lane_cache_bytes = cfg->lane_cache_bytes;
            if (cfg->central_grant_bytes) c.central_grant_bytes = cfg->central_grant_bytes;
            if (cfg->flush_interval_ms) c.flush_interval_ms = cfg->flush_interval_ms;
            if (cfg->batch_multiple) c.batch_multiple = cfg->batch_multiple;
            if (cfg->batch_cap) c.batch_cap = cfg->batch_cap;
            if (cfg->max_search_batch) c.max_search_batch = cfg->max_search_batch;
            c.serialized = cfg->serialized != 0;
        }
        auto e = new bivf_executor;
        try {
            e->impl = std::make_unique<bivf::Executor>(I(h), c);
        } catch (...) {
            delete e;
            throw;
        }
        *out = e;
    });
}

namespace {
bivf::Executor& X(bivf_executor* e) {
    if (!e || !e->impl) throw Error(BIVF_EINVAL, "null executor handle");
    return *e->impl;
}
}  // namespace

bivf_status bivf_executor_destroy(bivf_executor* e) {
    return guard([&] { delete e; });
}

bivf_status bivf_executor_submit_search(bivf_executor* e, const float* q, uint64_t nq, uint64_t k,
                                        uint64_t nprobe, bivf_ticket** out) {
    return guard([&] {
        need(q, "queries");
        need(out, "out");
        auto t = X(e).submit_search(q, (uint32_t)nq, (uint32_t)k, (uint32_t)nprobe);
        *out = new bivf_ticket{t};
    });
}

bivf_status bivf_executor_submit_insert(bivf_executor* e, const float* x, uint64_t n,
                                        const int64_t* ids, bivf_ticket** out) {
    return guard([&] {
        need(x, "x");
        need(out, "out");
        auto t = X(e).submit_insert(x, n, ids);
        *out = new bivf_ticket{t};
    });
}

bivf_status bivf_executor_flush(bivf_executor* e) {
    return guard([&] { X(e).flush_insertions(); });
}

bivf_status bivf_executor_set_mode(bivf_executor* e, int serialized) {
    return guard([&] { X(e).set_mode(serialized != 0); });
}

bivf_status bivf_executor_shutdown(bivf_executor* e) {
    return guard([&] { X(e).shutdown(); });
}

bivf_status bivf_executor_stats(const bivf_executor* e, uint64_t* out8) {
    return guard([&] {
        need(out8, "out");
        X(const_cast<bivf_executor*>(e)).stats(out8);
    });
}

bivf_status bivf_ticket_wait(bivf_ticket* t, bivf_ticket_info* info) {
    return guard([&] {
        if (!t || !t->t) throw Error(BIVF_EINVAL, "null ticket");
        t->t->wait();
        if (info) {
            auto& s = *t->t;
            info->status = (int32_t)s.status;
            info->type = (int32_t)s.type;
            info->lane = s.lane;
            info->nq = s.nq;
            info->k = s.k;
            info->n = s.type == bivf::RequestType::Insert ? s.ids.size() : 0;
            info->latency_us = s.latency_us();
            info->queue_us = s.queue_us();
            info->exec_us = s.exec_us();
        }
    });
}

bivf_status bivf_ticket_results(bivf_ticket* t, int64_t* ids, float* dists, uint32_t* counts) {
    return guard([&] {
        if (!t || !t->t) throw Error(BIVF_EINVAL, "null ticket");
        auto& s = *t->t;
        s.wait();
        if (ids && !s.ids.empty()) std::memcpy(ids, s.ids.data(), s.ids.size() * 8);
        if (dists && !s.dists.empty()) std::memcpy(dists, s.dists.data(), s.dists.size() * 4);
        if (counts && !s.counts.empty()) std::memcpy(counts, s.counts.data(), s.counts.size() * 4);
    });
}

bivf_status bivf_ticket_error(bivf_ticket* t, char* buf, uint64_t cap) {
    return guard([&] {
        if (!t || !t->t) throw Error(BIVF_EINVAL, "null ticket");
        if (buf && cap) {
            const std::string& m = t->t->error;
            const size_t n = std::min<size_t>(cap - 1, m.size());
            std::memcpy(buf, m.data(), n);
            buf[n] = 0;
        }
    });
}

bivf_status bivf_ticket_free(bivf_ticket* t) {
    return guard([&] { delete t; });
}

bivf_status bivf_replay(bivf_executor* e, const bivf_replay_spec* spec, const float* queries,
                        uint64_t nqueries, const float* inserts, uint64_t ninserts,
                        double* slat, uint64_t scap, uint64_t* ns, double* ilat, uint64_t icap,
                        uint64_t* ni, uint64_t* rejected, uint64_t* errors) {
    return guard([&] {
        need(spec, "spec");
        bivf::ReplaySpec r;
        r.qps_search = spec->qps_search;
        r.qps_insert = spec->qps_insert;
        r.duration_s = spec->duration_s;
        r.search_batch = spec->search_batch ? spec->search_batch : 1;
        r.insert_batch = spec->insert_batch ? spec->insert_batch : 1;
        r.k = spec->k ? spec->k : 10;
        r.nprobe = spec->nprobe ? spec->nprobe : 8;
        r.seed = spec->seed;
        r.poisson = spec->poisson != 0;
        auto out = bivf::replay(X(e), r, queries, nqueries, inserts, ninserts);
        if (ns) *ns = out.search_us.size();
        if (ni) *ni = out.insert_us.size();
        if (slat) std::memcpy(slat, out.search_us.data(), std::min<uint64_t>(scap, out.search_us.size()) * 8);
        if (ilat) std::memcpy(ilat, out.insert_us.data(), std::min<uint64_t>(icap, out.insert_us.size()) * 8);
        if (rejected) *rejected = out.rejected;
        if (errors) *errors = out.errors;
    });
}

bivf_status bivf_prewarm(bivf_index* h, uint64_t nq, uint64_t k, uint64_t nprobe) {
    return guard([&] { I(h).prewarm(nq, k, nprobe); });
}

bivf_status bivf_set_scan_mode(bivf_index* h, int mode) {
    return guard([&] {
        if (mode < 0 || mode > 4) throw Error(BIVF_EINVAL, "scan mode must be 0..4");
        I(h).set_scan_mode(mode);
    });
}

bivf_status bivf_set_timing(bivf_index* h, int enable) {
    return guard([&] { I(h).set_timing(enable != 0); });
}

bivf_status bivf_last_timings(const bivf_index* h, float* out4) {
    return guard([&] {
        need(out4, "out");
        I(h).last_timings(out4);
    });
}

}  // extern "C"
