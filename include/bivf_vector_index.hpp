// bivf_vector_index.hpp — drop-in adapter: the B200 index as a
// blockivf::VectorIndex (/root/reference/proj/include/blockivf/vector_index.hpp:19-44).
//
// Header-only, over the C-ABI in bivf.h.  Include it in a build that has the
// reference's headers on the include path and link libbivf_gpu.so; the
// reference's own Executor (executor.hpp:82) and replay (workload.hpp:85-87)
// then run on the GPU index unchanged.  Error codes are rethrown as the
// reference's exception types so its CHECK_THROWS_AS tests keep passing.
#pragma once

#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "blockivf/types.hpp"
#include "blockivf/vector_index.hpp"
#include "bivf.h"

namespace bivf_adapter {

[[noreturn]] inline void rethrow(bivf_status s, uint64_t inserted = 0) {
    const std::string m = bivf_last_error();
    switch (s) {
        case BIVF_EINVAL: throw std::invalid_argument(m);
        case BIVF_EPOOL: throw blockivf::PoolExhaustedError(inserted);
        case BIVF_ECORRUPT: throw blockivf::CorruptListError(m);
        case BIVF_ERANGE: throw std::out_of_range(m);
        case BIVF_ELOGIC: throw std::logic_error(m);
        default: throw std::runtime_error(m);
    }
}
inline void ok(bivf_status s) {
    if (s != BIVF_OK) rethrow(s);
}

class GpuClusterIndex final : public blockivf::VectorIndex {
public:
    // ClusterIndex(offline, n, IndexConfig) equivalent: train + bulk load.
    GpuClusterIndex(std::span<const float> offline, std::size_t n, const bivf_config& cfg) {
        ok(bivf_create(&cfg, &h_));
        ok(bivf_train(h_, offline.data(), n));
        ok(bivf_get_config(h_, &cfg_));
    }
    explicit GpuClusterIndex(const std::string& snapshot_path) {
        ok(bivf_load_snapshot(snapshot_path.c_str(), nullptr, &h_));
        ok(bivf_get_config(h_, &cfg_));
    }
    ~GpuClusterIndex() override {
        if (h_) bivf_destroy(h_);
    }
    GpuClusterIndex(const GpuClusterIndex&) = delete;
    GpuClusterIndex& operator=(const GpuClusterIndex&) = delete;

    std::vector<blockivf::vector_id> insert(std::span<const float> vectors, std::size_t n,
                                            std::span<const blockivf::vector_id> ids = {}) override {
        std::vector<blockivf::vector_id> out(n, -1);
        if (n == 0) return out;  // before the extent checks, as ivf_index.cpp:124-129
        if (vectors.size() != n * dim())
            throw std::invalid_argument("insert: vectors extent does not match n * dim");
        if (!ids.empty() && ids.size() != n)
            throw std::invalid_argument("insert: ids size does not match n");
        uint64_t inserted = 0;
        const bivf_status s = bivf_add(h_, vectors.data(), n, ids.empty() ? nullptr : ids.data(),
                                       out.data(), &inserted);
        if (s != BIVF_OK) rethrow(s, inserted);
        return out;
    }

    blockivf::SearchResult search(std::span<const float> query, std::size_t k,
                                  std::size_t nprobe) const override {
        if (query.size() != dim()) throw std::invalid_argument("search: dimension mismatch");
        std::vector<int64_t> ids(k);
        std::vector<float> d(k);
        uint32_t cnt = 0;
        ok(bivf_search(h_, query.data(), 1, k, nprobe, ids.data(), d.data(), &cnt));
        blockivf::SearchResult r;
        r.ids.assign(ids.begin(), ids.begin() + cnt);
        r.distances.assign(d.begin(), d.begin() + cnt);
        return r;
    }

    blockivf::cluster_id assign(std::span<const float> y) const override {
        if (y.size() != dim()) throw std::invalid_argument("assign: dimension mismatch");
        uint32_t c = 0;
        ok(bivf_assign(h_, y.data(), 1, &c));
        return c;
    }

    void post_insert_maintenance() override { ok(bivf_rearrange_sweep(h_)); }

    std::size_t dim() const override { return cfg_.dim; }
    std::size_t num_clusters() const override { return cfg_.num_clusters; }
    std::size_t size() const override {
        uint64_t v = 0;
        ok(bivf_size(h_, &v));
        return v;
    }
    std::uint64_t scalars_copied() const override {
        uint64_t v = 0;
        ok(bivf_scalars_copied(h_, &v));
        return v;
    }
    std::uint64_t reallocations() const override { return 0; }

    bivf_index* handle() const { return h_; }

private:
    bivf_index* h_ = nullptr;
    bivf_config cfg_{};
};

}  // namespace bivf_adapter
