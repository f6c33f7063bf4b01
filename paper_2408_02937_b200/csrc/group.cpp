// Vector-sharded groups of indexes (north star (5)), C++ only.
//
// Shard g of a G-shard group owns the vectors whose id satisfies id mod G == g;
// every shard holds all centroids, so the probe set of a query is the same on
// every shard and the merged top-k equals the single index's bit for bit.
//
// One search, every step device-resident on the shards' lease streams:
//   1. every shard receives the whole query batch (H2D);
//   2. shard g runs the coarse quantizer for query slice g only (1/G of the
//      batch) and the probe rows are all-gathered, so the quantizer is not
//      replicated;
//   3. every shard scans its own lists for the whole batch (local exact top-k);
//   4. the local top-k lists are all-gathered and merged on device (K8).
// Two transports carry steps 2 and 4:
//   * in-process: G shard handles in one process (any devices, one device
//     repeated included), peer copies between their lease streams ordered by
//     events (cudaMemcpyPeerAsync: NVLink P2P between GPUs);
//   * NCCL: one shard per process, ncclAllGather / ncclAllReduce on the lease
//     stream.  libnccl is loaded at run time (dlopen), so the library has no
//     link-time dependency on it.  `channels` communicators are split from the
//     root one at creation (ncclCommSplit); a call names its channel, and calls
//     on one channel must be issued in the same order on every rank (the usual
//     NCCL contract) — concurrent callers use different channels.  Channel 0
//     also carries the all-reduces of inserts and deletes.
// Inserts: every rank passes the same global batch; auto ids are the group's
// contiguous next_id range (ivf_index.cpp:133-141); each shard inserts its own
// rows with those explicit ids; outcomes are all-reduced so every rank returns
// the whole batch's result.  Deletes are routed by id mod G the same way.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/bivf.h"
#include "index.h"
#include "maint.cuh"

namespace bivf {

namespace {

// ---- libnccl, resolved at run time ---------------------------------------
struct Nccl {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
    std::string why;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        // a libnccl already loaded in the process (e.g. the one torch ships) wins
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            n.why = std::string("libnccl not loadable: ") + (e ? e : "?");
            return;
        }
        auto sym = [&](const char* name) { return dlsym(h, name); };
        n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
        n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
        n.CommSplit = reinterpret_cast<decltype(n.CommSplit)>(sym("ncclCommSplit"));
        n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
        n.AllGather = reinterpret_cast<decltype(n.AllGather)>(sym("ncclAllGather"));
        n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(sym("ncclAllReduce"));
        n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
        n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
        n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
        n.ok = n.GetUniqueId && n.CommInitRank && n.CommSplit && n.CommDestroy && n.AllGather &&
               n.AllReduce && n.GroupStart && n.GroupEnd && n.GetErrorString;
        if (!n.ok) n.why = "libnccl lacks a required symbol";
    });
    return n;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw Error(BIVF_ECUDA, std::string("NCCL error in ") + what + ": " + nccl().GetErrorString(r));
}
#define BIVF_NCCL(x) ::bivf::nccl_check((x), #x)

const Nccl& need_nccl() {
    const Nccl& n = nccl();
    if (!n.ok) throw Error(BIVF_ECUDA, n.why);
    return n;
}

uint32_t owner_of(int64_t id, uint32_t G) { return (uint32_t)((uint64_t)id % G); }

}  // namespace

class Group {
public:
    // in-process: every shard local
    explicit Group(std::vector<GpuIndex*> shards) : shards_(std::move(shards)) {
        G_ = (uint32_t)shards_.size();
        validate_shards();
        rank_ = 0;
        next_id_ = 0;
        for (auto* s : shards_) next_id_ = std::max<int64_t>(next_id_, s->next_id());
        // NVLink peer access between distinct devices (the peer copies work without it)
        for (auto* a : shards_)
            for (auto* b : shards_)
                if (a->device() != b->device()) {
                    int can = 0;
                    cudaDeviceCanAccessPeer(&can, a->device(), b->device());
                    if (can) {
                        cudaSetDevice(a->device());
                        if (cudaDeviceEnablePeerAccess(b->device(), 0) != cudaSuccess) cudaGetLastError();
                    }
                }
    }
    // NCCL: this process's shard is rank `rank` of `nranks`
    Group(GpuIndex* shard, const ncclUniqueId& uid, int nranks, int rank, uint32_t channels)
        : shards_{shard}, G_((uint32_t)nranks), rank_((uint32_t)rank) {
        const Nccl& n = need_nccl();
        if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(BIVF_EINVAL, "group: bad rank / nranks");
        BIVF_CUDA(cudaSetDevice(shard->device()));
        ncclComm_t root = nullptr;
        BIVF_NCCL(n.CommInitRank(&root, nranks, uid, rank));
        comms_.push_back(root);
        // one communicator per channel (concurrent callers), split from the root
        for (uint32_t c = 1; c < std::max<uint32_t>(1, channels); ++c) {
            ncclComm_t sub = nullptr;
            BIVF_NCCL(n.CommSplit(root, 0, rank, &sub, nullptr));
            comms_.push_back(sub);
        }
        chan_mu_ = std::vector<std::mutex>(comms_.size());
        for (size_t c = 0; c < comms_.size(); ++c) bufs_.push_back(std::make_unique<Bufs>());
        // next_id agreed on: the max over ranks
        int64_t mine = shard->next_id();
        DevBuf t;
        t.alloc(8);
        BIVF_CUDA(cudaMemcpy(t.p, &mine, 8, cudaMemcpyHostToDevice));
        BIVF_NCCL(n.AllReduce(t.p, t.p, 1, ncclInt64, ncclMax, root, nullptr));
        BIVF_CUDA(cudaMemcpy(&next_id_, t.p, 8, cudaMemcpyDeviceToHost));
    }
    ~Group() {
        if (!comms_.empty()) {
            const Nccl& n = nccl();
            for (auto it = comms_.rbegin(); it != comms_.rend(); ++it) n.CommDestroy(*it);
        }
    }

    bool nccl_mode() const { return !comms_.empty(); }
    uint32_t size() const { return G_; }

    // host buffers in and out (every rank: the same queries; every rank: all results)
    void search(const float* q, uint64_t nq, uint64_t k, uint64_t P, int64_t* ids, float* d,
                uint32_t* cnt, uint32_t channel) {
        if (nccl_mode()) search_nccl(q, nullptr, nq, k, P, ids, d, cnt, nullptr, channel);
        else search_local(q, nq, k, P, ids, d, cnt);
    }
    // device buffers on this rank's device, ordered after / before `stream` (NCCL mode)
    void search_device(const float* q_dev, uint64_t nq, uint64_t k, uint64_t P, int64_t* ids_dev,
                       float* d_dev, uint32_t* cnt_dev, cudaStream_t stream, uint32_t channel) {
        if (!nccl_mode()) throw Error(BIVF_EINVAL, "group_search_device: NCCL groups only");
        search_nccl(nullptr, q_dev, nq, k, P, ids_dev, d_dev, cnt_dev, stream, channel);
    }

    uint64_t insert(const float* x, uint64_t n, const int64_t* ids, int64_t* out) {
        if (n == 0) return 0;
        const uint32_t D = shards_[0]->D();
        std::vector<int64_t> gid(n);
        {
            std::lock_guard<std::mutex> lk(id_mu_);
            if (!ids) {
                for (uint64_t i = 0; i < n; ++i) gid[i] = next_id_ + (int64_t)i;
                next_id_ += (int64_t)n;
            } else {
                for (uint64_t i = 0; i < n; ++i) {
                    gid[i] = ids[i];
                    if (ids[i] >= 0) next_id_ = std::max<int64_t>(next_id_, ids[i] + 1);
                }
            }
        }
        std::vector<int64_t> res(n, -1);
        uint64_t inserted = 0;
        bool exhausted = false;
        for (uint32_t li = 0; li < shards_.size(); ++li) {
            const uint32_t g = nccl_mode() ? rank_ : li;
            std::vector<uint64_t> rows;
            for (uint64_t i = 0; i < n; ++i)
                if (gid[i] >= 0 && owner_of(gid[i], G_) == g) rows.push_back(i);
            if (rows.empty()) continue;
            std::vector<float> xs(rows.size() * D);
            std::vector<int64_t> is(rows.size()), os(rows.size(), -1);
            for (size_t r = 0; r < rows.size(); ++r) {
                std::memcpy(xs.data() + r * D, x + rows[r] * D, (size_t)D * 4);
                is[r] = gid[rows[r]];
            }
            try {
                shards_[li]->insert(xs.data(), rows.size(), is.data(), os.data());
            } catch (const Error& e) {
                if (e.code != BIVF_EPOOL) throw;
                exhausted = true;
            }
            for (size_t r = 0; r < rows.size(); ++r) res[rows[r]] = os[r];
        }
        if (nccl_mode()) all_reduce_max_i64(res.data(), n);
        for (uint64_t i = 0; i < n; ++i) {
            out[i] = res[i];
            inserted += res[i] >= 0;
        }
        if (nccl_mode()) {
            int64_t ex = exhausted ? 1 : 0;
            all_reduce_max_i64(&ex, 1);
            exhausted = ex != 0;
        }
        if (exhausted) {
            Error e(BIVF_EPOOL, "central memory pool exhausted on a shard after inserting " +
                                    std::to_string(inserted) + " vectors of the batch");
            e.inserted = inserted;
            throw e;
        }
        return inserted;
    }

    uint64_t remove(const int64_t* ids, uint64_t n, uint8_t* found) {
        std::vector<int64_t> f(n, 0);
        for (uint32_t li = 0; li < shards_.size(); ++li) {
            const uint32_t g = nccl_mode() ? rank_ : li;
            std::vector<int64_t> mine;
            std::vector<uint64_t> at;
            for (uint64_t i = 0; i < n; ++i)
                if (ids[i] >= 0 && owner_of(ids[i], G_) == g) {
                    mine.push_back(ids[i]);
                    at.push_back(i);
                }
            if (mine.empty()) continue;
            std::vector<uint8_t> fl(mine.size(), 0);
            shards_[li]->remove(mine.data(), mine.size(), fl.data());
            for (size_t j = 0; j < mine.size(); ++j) f[at[j]] = fl[j];
        }
        if (nccl_mode()) all_reduce_max_i64(f.data(), n);
        uint64_t removed = 0;
        for (uint64_t i = 0; i < n; ++i) {
            if (found) found[i] = (uint8_t)f[i];
            removed += f[i] != 0;
        }
        return removed;
    }

private:
    struct Bufs {  // per channel: gathered top-k lists + merged results (device)
        DevBuf gd, gi, md, mi, mc, q;
        PinBuf pin;
    };

    void validate_shards() {
        if (G_ == 0) throw Error(BIVF_EINVAL, "group: no shards");
        for (auto* s : shards_) {
            if (!s) throw Error(BIVF_EINVAL, "group: null shard");
            if (s->D() != shards_[0]->D() || s->C() != shards_[0]->C())
                throw Error(BIVF_EINVAL, "group: shards differ in dim / num_clusters");
        }
    }

    void all_reduce_max_i64(int64_t* v, uint64_t n) {
        const Nccl& nc = need_nccl();
        std::lock_guard<std::mutex> lk(chan_mu_[0]);
        BIVF_CUDA(cudaSetDevice(shards_[0]->device()));
        DevBuf t;
        t.alloc(n * 8);
        BIVF_CUDA(cudaMemcpy(t.p, v, n * 8, cudaMemcpyHostToDevice));
        BIVF_NCCL(nc.AllReduce(t.p, t.p, n, ncclInt64, ncclMax, comms_[0], nullptr));
        BIVF_CUDA(cudaMemcpy(v, t.p, n * 8, cudaMemcpyDeviceToHost));
    }

    // ---- in-process transport: peer copies ordered by events
    void search_local(const float* q, uint64_t nq, uint64_t k, uint64_t P, int64_t* ids, float* d,
                      uint32_t* cnt) {
        if (nq == 0) return;
        std::lock_guard<std::mutex> lk(local_mu_);
        const uint32_t G = G_, D = shards_[0]->D();
        std::vector<GpuIndex::ShardCtx> cx(G);
        struct Close {
            std::vector<GpuIndex*>& sh;
            std::vector<GpuIndex::ShardCtx>& cx;
            ~Close() {
                for (size_t g = 0; g < cx.size(); ++g) {
                    try {
                        sh[g]->shard_close(cx[g]);
                    } catch (...) {
                    }
                }
            }
        } closer{shards_, cx};
        std::vector<cudaEvent_t> ev(2 * G, nullptr);
        struct Evs {
            std::vector<cudaEvent_t>& e;
            ~Evs() {
                for (auto x : e)
                    if (x) cudaEventDestroy(x);
            }
        } evg{ev};
        for (uint32_t g = 0; g < G; ++g) {
            shards_[g]->shard_open(cx[g], nq, k, P, G);
            BIVF_CUDA(cudaSetDevice(shards_[g]->device()));
            BIVF_CUDA(cudaEventCreateWithFlags(&ev[g], cudaEventDisableTiming));
            BIVF_CUDA(cudaEventCreateWithFlags(&ev[G + g], cudaEventDisableTiming));
            BIVF_CUDA(cudaMemcpyAsync(cx[g].w.qraw, q, nq * D * 4, cudaMemcpyHostToDevice,
                                      cx[g].lease->stream));
            shards_[g]->shard_quantize(cx[g], g);
            BIVF_CUDA(cudaEventRecord(ev[g], cx[g].lease->stream));
        }
        const uint32_t slice = cx[0].slice;
        if (P != shards_[0]->C())
            for (uint32_t g = 0; g < G; ++g) {
                BIVF_CUDA(cudaSetDevice(shards_[g]->device()));
                for (uint32_t h = 0; h < G; ++h) {
                    if (h == g || (uint64_t)h * slice >= nq) continue;
                    const uint64_t rows = std::min<uint64_t>(slice, nq - (uint64_t)h * slice);
                    BIVF_CUDA(cudaStreamWaitEvent(cx[g].lease->stream, ev[h], 0));
                    BIVF_CUDA(cudaMemcpyPeerAsync(cx[g].w.probes + (size_t)h * slice * P, shards_[g]->device(),
                                                  cx[h].w.probes + (size_t)h * slice * P, shards_[h]->device(),
                                                  rows * P * 8, cx[g].lease->stream));
                }
            }
        for (uint32_t g = 0; g < G; ++g) {
            shards_[g]->shard_scan(cx[g]);
            BIVF_CUDA(cudaEventRecord(ev[G + g], cx[g].lease->stream));
        }
        // gather the local top-k lists on shard 0's device, merge, copy out
        const int dev0 = shards_[0]->device();
        BIVF_CUDA(cudaSetDevice(dev0));
        cudaStream_t s0 = cx[0].lease->stream;
        Bufs& b = local_bufs_;
        b.gd.ensure((size_t)G * nq * k * 4);
        b.gi.ensure((size_t)G * nq * k * 8);
        b.md.ensure((size_t)nq * k * 4);
        b.mi.ensure((size_t)nq * k * 8);
        b.mc.ensure((size_t)nq * 4);
        for (uint32_t g = 0; g < G; ++g) {
            BIVF_CUDA(cudaStreamWaitEvent(s0, ev[G + g], 0));
            BIVF_CUDA(cudaMemcpyPeerAsync(b.gd.as<float>() + (size_t)g * nq * k, dev0, cx[g].w.out_d,
                                          shards_[g]->device(), nq * k * 4, s0));
            BIVF_CUDA(cudaMemcpyPeerAsync(b.gi.as<long long>() + (size_t)g * nq * k, dev0, cx[g].w.out_i,
                                          shards_[g]->device(), nq * k * 8, s0));
        }
        BIVF_CUDA(launch_merge_shards(b.gd.as<float>(), b.gi.as<long long>(), G, (uint32_t)nq, (uint32_t)k,
                                      b.md.as<float>(), b.mi.as<long long>(), b.mc.as<uint32_t>(), s0));
        BIVF_CUDA(cudaMemcpyAsync(d, b.md.p, nq * k * 4, cudaMemcpyDeviceToHost, s0));
        BIVF_CUDA(cudaMemcpyAsync(ids, b.mi.p, nq * k * 8, cudaMemcpyDeviceToHost, s0));
        if (cnt) BIVF_CUDA(cudaMemcpyAsync(cnt, b.mc.p, nq * 4, cudaMemcpyDeviceToHost, s0));
        // every shard's lease is released only after the merge consumed its results
        for (uint32_t g = 1; g < G; ++g) {
            BIVF_CUDA(cudaEventRecord(ev[G + g], s0));
            BIVF_CUDA(cudaSetDevice(shards_[g]->device()));
            BIVF_CUDA(cudaStreamWaitEvent(cx[g].lease->stream, ev[G + g], 0));
            BIVF_CUDA(cudaSetDevice(dev0));
        }
        BIVF_CUDA(cudaStreamSynchronize(s0));
    }

    // ---- NCCL transport: one shard per process
    void search_nccl(const float* q_host, const float* q_dev, uint64_t nq, uint64_t k, uint64_t P,
                     int64_t* ids, float* d, uint32_t* cnt, cudaStream_t user, uint32_t channel) {
        if (nq == 0) return;
        if (channel >= comms_.size()) throw Error(BIVF_EINVAL, "group: channel out of range");
        const Nccl& nc = need_nccl();
        std::lock_guard<std::mutex> lk(chan_mu_[channel]);
        ncclComm_t comm = comms_[channel];
        GpuIndex* sh = shards_[0];
        const uint32_t D = sh->D();
        GpuIndex::ShardCtx cx;
        struct Close {
            GpuIndex* s;
            GpuIndex::ShardCtx& c;
            ~Close() {
                try {
                    s->shard_close(c);
                } catch (...) {
                }
            }
        } closer{sh, cx};
        sh->shard_open(cx, nq, k, P, G_);
        BIVF_CUDA(cudaSetDevice(sh->device()));
        cudaStream_t st = cx.lease->stream;
        cudaEvent_t ue = nullptr;
        if (user) {
            BIVF_CUDA(cudaEventCreateWithFlags(&ue, cudaEventDisableTiming));
            BIVF_CUDA(cudaEventRecord(ue, user));
            BIVF_CUDA(cudaStreamWaitEvent(st, ue, 0));
        }
        BIVF_CUDA(cudaMemcpyAsync(cx.w.qraw, q_host ? (const void*)q_host : (const void*)q_dev, nq * D * 4,
                                  q_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
        sh->shard_quantize(cx, rank_);
        if (P != sh->C())  // in-place all-gather of the probe rows (slice per rank)
            BIVF_NCCL(nc.AllGather(cx.w.probes + (size_t)rank_ * cx.slice * P, cx.w.probes,
                                   (size_t)cx.slice * P, ncclInt64, comm, st));
        sh->shard_scan(cx);
        Bufs& b = *bufs_[channel];
        b.gd.ensure((size_t)G_ * nq * k * 4);
        b.gi.ensure((size_t)G_ * nq * k * 8);
        BIVF_NCCL(nc.GroupStart());
        BIVF_NCCL(nc.AllGather(cx.w.out_d, b.gd.p, nq * k, ncclFloat32, comm, st));
        BIVF_NCCL(nc.AllGather(cx.w.out_i, b.gi.p, nq * k, ncclInt64, comm, st));
        BIVF_NCCL(nc.GroupEnd());
        float* od = d;
        long long* oi = reinterpret_cast<long long*>(ids);
        uint32_t* oc = cnt;
        if (q_host) {  // host outputs: merge into device scratch, then D2H
            b.md.ensure((size_t)nq * k * 4);
            b.mi.ensure((size_t)nq * k * 8);
            b.mc.ensure((size_t)nq * 4);
            od = b.md.as<float>();
            oi = b.mi.as<long long>();
            oc = b.mc.as<uint32_t>();
        }
        BIVF_CUDA(launch_merge_shards(b.gd.as<float>(), b.gi.as<long long>(), G_, (uint32_t)nq, (uint32_t)k, od,
                                      oi, oc, st));
        if (q_host) {
            BIVF_CUDA(cudaMemcpyAsync(d, od, nq * k * 4, cudaMemcpyDeviceToHost, st));
            BIVF_CUDA(cudaMemcpyAsync(ids, oi, nq * k * 8, cudaMemcpyDeviceToHost, st));
            if (cnt) BIVF_CUDA(cudaMemcpyAsync(cnt, oc, nq * 4, cudaMemcpyDeviceToHost, st));
            BIVF_CUDA(cudaStreamSynchronize(st));
        } else {
            BIVF_CUDA(cudaEventRecord(ue, st));
            BIVF_CUDA(cudaStreamWaitEvent(user, ue, 0));
        }
        if (ue) cudaEventDestroy(ue);
    }

    std::vector<GpuIndex*> shards_;
    uint32_t G_ = 1, rank_ = 0;
    int64_t next_id_ = 0;
    std::mutex id_mu_, local_mu_;
    std::vector<ncclComm_t> comms_;
    std::vector<std::mutex> chan_mu_;
    std::vector<std::unique_ptr<Bufs>> bufs_;
    Bufs local_bufs_;
};

}  // namespace bivf

// ---- C-ABI (include/bivf.h) -------------------------------------------------
struct bivf_group {
    std::unique_ptr<bivf::Group> impl;
};

namespace bivf {
GpuIndex& index_of(bivf_index* h);  // capi.cpp
bivf_status run_guarded(const std::function<void()>& f);
}  // namespace bivf

using bivf::Error;

namespace {
bivf::Group& G(bivf_group* g) {
    if (!g || !g->impl) throw Error(BIVF_EINVAL, "null group handle");
    return *g->impl;
}
}  // namespace

extern "C" {

bivf_status bivf_nccl_unique_id(void* out128) {
    return bivf::run_guarded([&] {
        if (!out128) throw Error(BIVF_EINVAL, "out must not be NULL");
        ncclUniqueId id;
        BIVF_NCCL(bivf::need_nccl().GetUniqueId(&id));
        std::memcpy(out128, &id, sizeof(id));
    });
}

bivf_status bivf_group_create_local(bivf_index* const* shards, uint32_t nshards, bivf_group** out) {
    return bivf::run_guarded([&] {
        if (!out || !shards) throw Error(BIVF_EINVAL, "NULL argument");
        *out = nullptr;
        std::vector<bivf::GpuIndex*> v;
        for (uint32_t i = 0; i < nshards; ++i) v.push_back(&bivf::index_of(shards[i]));
        auto g = std::make_unique<bivf_group>();
        g->impl = std::make_unique<bivf::Group>(std::move(v));
        *out = g.release();
    });
}

bivf_status bivf_group_create_nccl(bivf_index* shard, const void* uid128, int32_t nranks, int32_t rank,
                                   uint32_t channels, bivf_group** out) {
    return bivf::run_guarded([&] {
        if (!out || !uid128) throw Error(BIVF_EINVAL, "NULL argument");
        *out = nullptr;
        ncclUniqueId id;
        std::memcpy(&id, uid128, sizeof(id));
        auto g = std::make_unique<bivf_group>();
        g->impl = std::make_unique<bivf::Group>(&bivf::index_of(shard), id, nranks, rank, channels);
        *out = g.release();
    });
}

void bivf_group_destroy(bivf_group* g) {
    try {
        delete g;
    } catch (...) {
    }
}

bivf_status bivf_group_search(bivf_group* g, const float* q, uint64_t nq, uint64_t k, uint64_t nprobe,
                              int64_t* out_ids, float* out_d, uint32_t* out_counts, uint32_t channel) {
    return bivf::run_guarded([&] {
        if (nq && (!q || !out_ids || !out_d)) throw Error(BIVF_EINVAL, "NULL argument");
        G(g).search(q, nq, k, nprobe, out_ids, out_d, out_counts, channel);
    });
}

bivf_status bivf_group_search_device(bivf_group* g, const float* q_dev, uint64_t nq, uint64_t k,
                                     uint64_t nprobe, int64_t* ids_dev, float* d_dev, uint32_t* counts_dev,
                                     void* stream, uint32_t channel) {
    return bivf::run_guarded([&] {
        G(g).search_device(q_dev, nq, k, nprobe, ids_dev, d_dev, counts_dev, static_cast<cudaStream_t>(stream),
                           channel);
    });
}

bivf_status bivf_group_insert(bivf_group* g, const float* x, uint64_t n, const int64_t* ids, int64_t* out_ids,
                              uint64_t* inserted) {
    uint64_t done = 0;
    const bivf_status st = bivf::run_guarded([&] {
        if (n && (!x || !out_ids)) throw Error(BIVF_EINVAL, "NULL argument");
        try {
            done = G(g).insert(x, n, ids, out_ids);
        } catch (const Error& e) {
            done = e.inserted;
            throw;
        }
    });
    if (inserted) *inserted = done;
    return st;
}

bivf_status bivf_group_remove(bivf_group* g, const int64_t* ids, uint64_t n, uint64_t* removed, uint8_t* found) {
    return bivf::run_guarded([&] {
        if (n && !ids) throw Error(BIVF_EINVAL, "NULL argument");
        const uint64_t r = G(g).remove(ids, n, found);
        if (removed) *removed = r;
    });
}

bivf_status bivf_group_size(const bivf_group* g, uint32_t* out) {
    return bivf::run_guarded([&] {
        if (!g || !g->impl || !out) throw Error(BIVF_EINVAL, "NULL argument");
        *out = g->impl->size();
    });
}

}  // extern "C"
