// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (blockivf, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It
// lets the Python tests and bench.py's reference arm drive the reference's
// own ClusterIndex / kmeans / synthetic_dataset / exact_knn / Executor with
// plain pointers.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs load it.
//
// Reference entry points wrapped (file:line under /root/reference/proj):
//   ClusterIndex ctor/insert/search/assign/exceed/rearrange   src/ivf_index.cpp:47,122,262,93,300,476
//   pool().header/ids/payload/allocated_blocks                  include/blockivf/block_store.hpp:75,113-132
//   save/load (BIVFSNAP v1)                                     src/ivf_index.cpp:535,567
//   kmeans                                                      src/kmeans.cpp:31
//   synthetic_dataset                                           src/dataset.cpp:92
//   exact_knn                                                   src/oracle.cpp:11
//   Executor + replay                                           src/executor.cpp, src/workload.cpp
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "blockivf/dataset.hpp"
#include "blockivf/executor.hpp"
#include "blockivf/ivf_index.hpp"
#include "blockivf/kmeans.hpp"
#include "blockivf/oracle.hpp"

using namespace blockivf;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

// 0 ok, 1 invalid_argument, 2 pool exhausted, 3 corrupt, 4 out_of_range,
// 5 logic_error, 6 runtime_error (io), 9 other
#define REF_GUARD(...)                                               \
    try {                                                            \
        __VA_ARGS__;                                                 \
        return 0;                                                    \
    } catch (const PoolExhaustedError& e) {                          \
        return fail(e, 2);                                           \
    } catch (const CorruptListError& e) {                            \
        return fail(e, 3);                                           \
    } catch (const std::invalid_argument& e) {                       \
        return fail(e, 1);                                           \
    } catch (const std::out_of_range& e) {                           \
        return fail(e, 4);                                           \
    } catch (const std::logic_error& e) {                            \
        return fail(e, 5);                                           \
    } catch (const std::runtime_error& e) {                          \
        return fail(e, 6);                                           \
    } catch (const std::exception& e) {                              \
        return fail(e, 9);                                           \
    }

ClusterIndex* I(void* h) { return static_cast<ClusterIndex*>(h); }
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Train through the reference constructor (kmeans + build_offline).
int ref_create(const float* x, uint64_t n, uint64_t dim, uint64_t clusters, uint64_t block_cap,
               uint64_t rearrange_threshold, uint64_t num_blocks, uint64_t kmeans_iters,
               uint64_t seed, uint64_t nprobe_default, void** out) {
    REF_GUARD({
        IndexConfig cfg;
        cfg.num_clusters = clusters;
        cfg.dim = dim;
        cfg.nprobe_default = nprobe_default;
        cfg.rearrange_threshold = rearrange_threshold;
        cfg.kmeans_iters = kmeans_iters;
        cfg.kmeans_seed = seed;
        cfg.pool = PoolConfig{.num_blocks = num_blocks, .block_capacity = block_cap, .dim = dim};
        *out = new ClusterIndex(std::span<const float>(x, n * dim), n, cfg);
    })
}

int ref_load(const char* path, void** out) {
    REF_GUARD({ *out = ClusterIndex::load(path).release(); })
}

int ref_save(void* h, const char* path) { REF_GUARD({ I(h)->save(path); }) }

void ref_destroy(void* h) { delete I(h); }

int ref_insert(void* h, const float* x, uint64_t n, const int64_t* ids, int64_t* out,
               uint64_t* inserted) {
    *inserted = 0;
    for (uint64_t i = 0; i < n; ++i) out[i] = -1;
    try {
        std::span<const vector_id> sp;
        if (ids) sp = {ids, n};
        auto r = I(h)->insert(std::span<const float>(x, n * I(h)->dim()), n, sp);
        uint64_t c = 0;
        for (uint64_t i = 0; i < n; ++i) {
            out[i] = r[i];
            if (r[i] >= 0) ++c;
        }
        *inserted = c;
        return 0;
    } catch (const PoolExhaustedError& e) {
        *inserted = e.inserted();
        return fail(e, 2);
    } catch (const std::invalid_argument& e) {
        return fail(e, 1);
    } catch (const std::exception& e) {
        return fail(e, 9);
    }
}

int ref_search(void* h, const float* q, uint64_t k, uint64_t nprobe, int64_t* ids, float* d,
               uint64_t* count) {
    REF_GUARD({
        auto r = I(h)->search(std::span<const float>(q, I(h)->dim()), k, nprobe);
        *count = r.ids.size();
        for (size_t i = 0; i < r.ids.size(); ++i) {
            ids[i] = r.ids[i];
            d[i] = r.distances[i];
        }
    })
}

int ref_assign(void* h, const float* y, uint32_t* out) {
    REF_GUARD({ *out = I(h)->assign(std::span<const float>(y, I(h)->dim())); })
}

int ref_exceed(void* h, uint32_t c, int* out) { REF_GUARD({ *out = I(h)->exceed(c) ? 1 : 0; }) }
int ref_rearrange(void* h, uint32_t c) { REF_GUARD({ I(h)->rearrange(c); }) }
int ref_rearrange_sweep(void* h) { REF_GUARD({ I(h)->rearrange_sweep(); }) }

// events: up to cap records of (cluster, hops_before, hops_after, merges)
uint64_t ref_take_events(void* h, uint64_t* out4, uint64_t cap) {
    auto ev = I(h)->take_rearrange_events();
    uint64_t n = 0;
    for (auto& e : ev) {
        if (n >= cap) break;
        out4[4 * n + 0] = e.cluster;
        out4[4 * n + 1] = e.hops_before;
        out4[4 * n + 2] = e.hops_after;
        out4[4 * n + 3] = e.merges;
        ++n;
    }
    return n;
}

uint64_t ref_dim(void* h) { return I(h)->dim(); }
uint64_t ref_num_clusters(void* h) { return I(h)->num_clusters(); }
uint64_t ref_size(void* h) { return I(h)->size(); }
uint64_t ref_scalars_copied(void* h) { return I(h)->scalars_copied(); }
uint64_t ref_list_length(void* h, uint32_t c) { return I(h)->list_length(c); }
uint64_t ref_offline_count(void* h, uint32_t c) { return I(h)->offline_count(c); }
uint64_t ref_hop_count(void* h, uint32_t c) { return I(h)->hop_count(c); }
int32_t ref_online_head(void* h, uint32_t c) { return I(h)->online_head(c); }
uint64_t ref_allocated_blocks(void* h) { return I(h)->pool().allocated_blocks(); }
void ref_centroids(void* h, float* out) {
    auto c = I(h)->centroids();
    std::memcpy(out, c.data(), c.size() * sizeof(float));
}

// header: prev, next, size(committed), owner, merged
void ref_block_header(void* h, int32_t b, int32_t* out5) {
    auto hd = I(h)->pool().header(b);
    out5[0] = hd.prev;
    out5[1] = hd.next;
    out5[2] = static_cast<int32_t>(hd.size);
    out5[3] = hd.owner;
    out5[4] = hd.merged_with_prev ? 1 : 0;
}
void ref_block_ids(void* h, int32_t b, int64_t* out) {
    const auto& p = I(h)->pool();
    std::memcpy(out, p.ids(b), p.config().block_capacity * sizeof(int64_t));
}
void ref_block_payload(void* h, int32_t b, float* out) {
    const auto& p = I(h)->pool();
    std::memcpy(out, p.payload(b), p.config().payload_scalars() * sizeof(float));
}

// cluster_contents: first call with ids=NULL to get the count.
uint64_t ref_cluster_contents(void* h, uint32_t c, int64_t* ids, float* vecs) {
    auto v = I(h)->cluster_contents(c);
    if (ids) {
        const size_t dim = I(h)->dim();
        for (size_t i = 0; i < v.size(); ++i) {
            ids[i] = v[i].first;
            std::memcpy(vecs + i * dim, v[i].second.data(), dim * sizeof(float));
        }
    }
    return v.size();
}

// dump_pool text; returns required length (incl. NUL)
uint64_t ref_dump_pool(void* h, char* buf, uint64_t cap) {
    std::ostringstream os;
    I(h)->dump_pool(os);
    const std::string s = os.str();
    if (buf && cap > 0) {
        const size_t n = std::min<size_t>(cap - 1, s.size());
        std::memcpy(buf, s.data(), n);
        buf[n] = 0;
    }
    return s.size() + 1;
}

int ref_kmeans(const float* pts, uint64_t n, uint64_t dim, uint64_t k, uint64_t iters,
               uint64_t seed, float* centroids, uint32_t* assignment, uint64_t* iters_run) {
    REF_GUARD({
        auto r = kmeans(std::span<const float>(pts, n * dim), n, dim, k, iters, seed);
        std::memcpy(centroids, r.centroids.data(), r.centroids.size() * sizeof(float));
        std::memcpy(assignment, r.assignment.data(), r.assignment.size() * sizeof(uint32_t));
        *iters_run = r.iters_run;
    })
}

int ref_synthetic_dataset(uint64_t n, uint64_t dim, uint64_t comps, uint64_t seed, float* out) {
    REF_GUARD({
        auto ds = synthetic_dataset(n, dim, comps, seed);
        std::memcpy(out, ds.data.data(), ds.data.size() * sizeof(float));
    })
}

int ref_exact_knn(const float* base, uint64_t n, uint64_t dim, const float* q, uint64_t k,
                  int64_t* ids, float* d, uint64_t* count) {
    REF_GUARD({
        auto r = exact_knn(std::span<const float>(base, n * dim), n, dim,
                           std::span<const float>(q, dim), k);
        *count = r.ids.size();
        for (size_t i = 0; i < r.ids.size(); ++i) {
            ids[i] = r.ids[i];
            d[i] = r.distances[i];
        }
    })
}

// CPU baseline: `threads` workers each run ClusterIndex::search over a
// strided share of `nq` queries (the reference's per-query search path,
// src/ivf_index.cpp:262-298), repeating the sample `reps` times.  Results of
// the first pass land in ids/d (nq*k).  Returns wall seconds in *secs.
int ref_search_threads(void* h, const float* q, uint64_t nq, uint64_t k, uint64_t nprobe,
                       uint32_t threads, uint32_t reps, int64_t* ids, float* d, double* secs) {
    REF_GUARD({
        const size_t dim = I(h)->dim();
        std::atomic<int> err{0};
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (uint32_t t = 0; t < threads; ++t) {
            pool.emplace_back([&, t] {
                try {
                    for (uint32_t r = 0; r < reps; ++r) {
                        for (uint64_t i = t; i < nq; i += threads) {
                            auto res = I(h)->search(std::span<const float>(q + i * dim, dim), k,
                                                    nprobe);
                            if (r == 0 && ids) {
                                for (size_t j = 0; j < k; ++j) {
                                    ids[i * k + j] = j < res.ids.size() ? res.ids[j] : -1;
                                    d[i * k + j] = j < res.ids.size() ? res.distances[j] : 0.0f;
                                }
                            }
                        }
                    }
                } catch (...) {
                    err = 1;
                }
            });
        }
        for (auto& th : pool) th.join();
        *secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (err) throw std::runtime_error("search worker failed");
    })
}

// Parallel bulk insert through the reference's thread-safe insert
// (src/ivf_index.cpp:122-164): `threads` callers each insert contiguous
// chunks of `chunk` vectors with auto ids.  Used only to build the CPU
// baseline's index quickly; layout is nondeterministic (as in the reference).
int ref_insert_threads(void* h, const float* x, uint64_t n, uint32_t threads, uint64_t chunk) {
    REF_GUARD({
        const size_t dim = I(h)->dim();
        std::atomic<uint64_t> next{0};
        std::atomic<int> err{0};
        std::vector<std::thread> pool;
        for (uint32_t t = 0; t < threads; ++t) {
            pool.emplace_back([&] {
                try {
                    for (;;) {
                        const uint64_t s = next.fetch_add(chunk);
                        if (s >= n) break;
                        const uint64_t m = std::min<uint64_t>(chunk, n - s);
                        I(h)->insert(std::span<const float>(x + s * dim, m * dim), m);
                    }
                } catch (...) {
                    err = 1;
                }
            });
        }
        for (auto& th : pool) th.join();
        if (err) throw std::runtime_error("insert worker failed");
    })
}

// --- reference Executor (multi-lane pool), for the CPU latency baseline ---
void* ref_exec_create(void* h, uint64_t lanes, uint32_t serialized) {
    ExecutorConfig cfg;
    cfg.num_lanes = lanes;
    cfg.mode = serialized ? ExecutionMode::Serialized : ExecutionMode::Parallel;
    return new Executor(*I(h), cfg);
}
void ref_exec_destroy(void* e) {
    auto* ex = static_cast<Executor*>(e);
    ex->shutdown();
    delete ex;
}

// Open-loop replay of search requests (nq queries each, `dim` floats per
// query) at `qps` through the reference Executor, with an optional concurrent
// insert stream at `insert_rate` vectors/s submitted as 128-vector requests
// (the batcher's multiple, executor.hpp:31).  Per-ticket latency_us
// (executor.cpp:53) lands in lat_us[nreq] (-1 for rejected tickets).
int ref_exec_replay_dim(void* e, uint64_t dim, const float* q, uint64_t nreq, uint64_t nq,
                        uint64_t k, uint64_t nprobe, double qps, const float* ins, uint64_t n_ins,
                        double insert_rate, double* lat_us, uint64_t* rejected) {
    REF_GUARD({
        auto* ex = static_cast<Executor*>(e);
        std::atomic<bool> stop{false};
        std::thread inserter;
        if (insert_rate > 0 && n_ins >= 128) {
            inserter = std::thread([&] {
                const uint64_t per = 128;
                const auto period = std::chrono::duration_cast<std::chrono::steady_clock::duration>(
                    std::chrono::duration<double>(static_cast<double>(per) / insert_rate));
                auto next = std::chrono::steady_clock::now();
                uint64_t pos = 0;
                std::vector<Ticket> its;
                while (!stop.load()) {
                    if (pos + per > n_ins) pos = 0;
                    its.push_back(
                        ex->submit_insert(std::span<const float>(ins + pos * dim, per * dim), per));
                    pos += per;
                    next += period;
                    std::this_thread::sleep_until(next);
                }
                ex->flush_insertions();
                for (auto& t : its) t.wait();
            });
        }
        std::vector<Ticket> tickets;
        tickets.reserve(nreq);
        const auto period = std::chrono::duration_cast<std::chrono::steady_clock::duration>(
            std::chrono::duration<double>(1.0 / qps));
        auto next = std::chrono::steady_clock::now();
        for (uint64_t r = 0; r < nreq; ++r) {
            tickets.push_back(
                ex->submit_search(std::span<const float>(q + r * nq * dim, nq * dim), nq, k, nprobe));
            next += period;
            std::this_thread::sleep_until(next);
        }
        uint64_t rej = 0;
        for (uint64_t r = 0; r < nreq; ++r) {
            const auto& res = tickets[r].get();
            if (res.status == TicketStatus::Rejected) {
                ++rej;
                lat_us[r] = -1.0;
            } else {
                lat_us[r] = res.latency_us;
            }
        }
        stop = true;
        if (inserter.joinable()) inserter.join();
        *rejected = rej;
    })
}

}  // extern "C"
