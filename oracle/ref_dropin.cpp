// TEST INFRASTRUCTURE — drop-in proof: the reference's own Executor + replay
// harness (src/executor.cpp, src/workload.cpp, unmodified) driving the B200
// index through include/bivf_vector_index.hpp, checked against the reference
// ClusterIndex loaded from the same BIVFSNAP snapshot.
// Built by `make -C oracle ref` into oracle/_ref/ref_dropin; run by
// tests/test_gpu_dropin.py on a GPU box.
#include <cstdio>
#include <cstring>
#include <memory>

#include "bivf_vector_index.hpp"
#include "blockivf/dataset.hpp"
#include "blockivf/executor.hpp"
#include "blockivf/ivf_index.hpp"
#include "blockivf/workload.hpp"

using namespace blockivf;

int main(int argc, char** argv) {
    const char* snap = argc > 1 ? argv[1] : "/tmp/bivf_dropin.bivf";
    auto base = synthetic_dataset(4000, 32, 24, 7);
    bivf_config cfg{};
    cfg.num_clusters = 24;
    cfg.dim = 32;
    cfg.block_capacity = 16;
    cfg.num_blocks = 2000;
    cfg.rearrange_threshold = 64;
    cfg.kmeans_iters = 10;
    cfg.nprobe_default = 8;
    bivf_adapter::GpuClusterIndex gpu(base.all(), base.size(), cfg);

    // 1. the reference Executor + replay over the GPU index (VectorIndex&)
    auto queries = synthetic_dataset(200, 32, 24, 8);
    auto inserts = synthetic_dataset(3000, 32, 24, 9);
    ExecutorConfig ecfg;
    ecfg.num_lanes = 8;
    WorkloadReport rep;
    {
        Executor ex(gpu, ecfg);
        WorkloadSpec spec;
        spec.qps_search = 400;
        spec.qps_insert = 50;
        spec.insert_batch = 16;
        spec.search_batch = 4;
        spec.duration_s = 1.0;
        spec.k = 10;
        spec.nprobe = 8;
        spec.timeout_ms = 1000;
        rep = replay(spec, ex, gpu, queries, inserts);
        ex.shutdown();
    }
    std::printf("replay: searches=%zu inserts=%zu rejected=%zu errors=%zu p50=%.3fms p99=%.3fms\n",
                rep.search.count, rep.insertion.count, rep.rejected, rep.errors, rep.search.p50_ms,
                rep.search.p99_ms);
    if (rep.search.count == 0 || rep.errors != 0) return 2;

    // 2. same state in the reference: snapshot -> ClusterIndex::load
    if (bivf_save_snapshot(gpu.handle(), snap) != BIVF_OK) return 3;
    auto ref = ClusterIndex::load(snap);
    std::size_t bad = 0;
    for (std::size_t q = 0; q < queries.size(); ++q) {
        for (std::size_t nprobe : {1, 4, 24}) {
            const auto a = gpu.search(queries.row(q), 10, nprobe);
            const auto b = ref->search(queries.row(q), 10, nprobe);
            if (a.ids != b.ids || std::memcmp(a.distances.data(), b.distances.data(),
                                              a.distances.size() * 4) != 0)
                ++bad;
        }
        if (gpu.assign(queries.row(q)) != ref->assign(queries.row(q))) ++bad;
    }
    std::printf("dropin: size gpu=%zu ref=%zu mismatches=%zu\n", gpu.size(), ref->size(), bad);
    std::remove(snap);
    return (bad == 0 && gpu.size() == ref->size()) ? 0 : 1;
}
