// GpuIndex implementation (see index.h for the ownership / concurrency model).
#include "index.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <fstream>
#include <sstream>
#include <set>
#include <unordered_map>

#include "launches.h"
#include "maint.cuh"

namespace bivf {

std::atomic<uint64_t> g_launches{0};

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw Error(BIVF_ECUDA, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
    }
}

DevBuf::~DevBuf() {
    if (p) cudaFree(p);
}
void DevBuf::alloc(size_t n) {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    if (n == 0) n = 16;
    cudaError_t e = cudaMalloc(&p, n);
    if (e != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
        throw Error(BIVF_ENOMEM, "device allocation of " + std::to_string(n) + " bytes failed: " +
                                     cudaGetErrorString(e));
    }
    bytes = n;
}
void DevBuf::ensure(size_t n) {
    if (n <= bytes && p) return;
    size_t grow = std::max(n, bytes + bytes / 2);
    alloc(grow);
}
PinBuf::~PinBuf() {
    if (p) cudaFreeHost(p);
}
void PinBuf::ensure(size_t n) {
    if (n <= bytes && p) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    size_t grow = std::max<size_t>(std::max(n, bytes + bytes / 2), 4096);
    BIVF_CUDA(cudaHostAlloc(&p, grow, cudaHostAllocDefault));
    bytes = grow;
}

// True for page-locked host memory (cudaHostAlloc / cudaHostRegister): the
// search path DMAs such buffers directly instead of staging them.
static bool is_pinned(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// Host staging copies of the search path (user buffers <-> pinned lease
// buffers) on the OpenMP pool: one thread moves ~6-10 GB/s, the copy of a
// 10K x 128 query batch would otherwise be a sizeable part of the call.
static void par_memcpy(void* dst, const void* src, size_t n) {
    constexpr size_t kChunk = 128 * 1024;
    if (n < 2 * kChunk) {
        std::memcpy(dst, src, n);
        return;
    }
    const long nch = (long)((n + kChunk - 1) / kChunk);
#pragma omp parallel for num_threads(8) schedule(static)
    for (long i = 0; i < nch; ++i) {
        const size_t o = (size_t)i * kChunk;
        std::memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o,
                    std::min(kChunk, n - o));
    }
}

cudaError_t GpuIndex::h2d(void* dst, const void* src, size_t n) const {
    if (!n) return cudaSuccess;
    cudaError_t e = cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, data_stream_);
    return e != cudaSuccess ? e : cudaStreamSynchronize(data_stream_);
}
cudaError_t GpuIndex::d2h(void* dst, const void* src, size_t n) const {
    if (!n) return cudaSuccess;
    cudaError_t e = cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, data_stream_);
    return e != cudaSuccess ? e : cudaStreamSynchronize(data_stream_);
}
cudaError_t GpuIndex::dset(void* p, int v, size_t n) const {
    if (!n) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(p, v, n, data_stream_);
    return e != cudaSuccess ? e : cudaStreamSynchronize(data_stream_);
}

namespace {

int log_level() {
    const char* v = std::getenv("BIVF_LOG");
    if (!v) v = std::getenv("BLOCKIVF_LOG");  // log.hpp:9-20
    if (!v) return 1;
    std::string s(v);
    if (s == "quiet") return 0;
    if (s == "info") return 2;
    if (s == "debug") return 3;
    return 1;
}

void log_warn(const std::string& m) {
    if (log_level() >= 1) std::fprintf(stderr, "[bivf] %s\n", m.c_str());
}

// Slow-event trace (BIVF_TRACE=<microseconds>): searches and maintenance
// operations slower than the threshold print their phase breakdown.
double trace_threshold_us() {
    static const double t = [] {
        const char* v = std::getenv("BIVF_TRACE");
        return v ? std::max(1.0, atof(v)) : -1.0;
    }();
    return t;
}
using TClock = std::chrono::steady_clock;
double us_since(TClock::time_point t) {
    return std::chrono::duration<double, std::micro>(TClock::now() - t).count();
}
void trace(const char* what, double total_us, const std::string& detail) {
    const double thr = trace_threshold_us();
    if (thr > 0 && total_us >= thr)
        std::fprintf(stderr, "[bivf-trace] %.3f %s %.0f us: %s\n",
                     std::chrono::duration<double>(TClock::now().time_since_epoch()).count(), what, total_us,
                     detail.c_str());
}

size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

uint32_t ceil_div(uint64_t a, uint64_t b) { return (uint32_t)((a + b - 1) / b); }

bivf_config normalized(bivf_config c) {
    if (c.num_clusters == 0) c.num_clusters = 100;
    if (c.nprobe_default == 0) c.nprobe_default = std::min<uint64_t>(8, c.num_clusters);
    if (c.rearrange_threshold == 0) c.rearrange_threshold = 256;
    if (c.kmeans_iters == 0) c.kmeans_iters = 25;
    if (c.kmeans_seed == 0 && !c.kmeans_seed_set) c.kmeans_seed = 42;
    if (c.num_blocks == 0) c.num_blocks = 1024;
    if (c.block_capacity == 0) c.block_capacity = 64;
    if (c.alert_watermark == 0.0) c.alert_watermark = 0.9;
    if (c.num_leases == 0) c.num_leases = 32;
    if (c.max_list_blocks == 0) c.max_list_blocks = (uint32_t)c.num_blocks;
    return c;
}

// IndexConfig::validate + PoolConfig::validate (ivf_index.cpp:28-35, block_store.cpp:9-17)
void validate(const bivf_config& c) {
    if (c.dim < 1) throw Error(BIVF_EINVAL, "PoolConfig: dim must be >= 1");
    if (c.num_clusters < 1) throw Error(BIVF_EINVAL, "IndexConfig: num_clusters must be >= 1");
    if (c.nprobe_default < 1 || c.nprobe_default > c.num_clusters)
        throw Error(BIVF_EINVAL, "IndexConfig: nprobe_default out of [1, num_clusters]");
    if (c.alert_watermark <= 0.0 || c.alert_watermark > 1.0)
        throw Error(BIVF_EINVAL, "PoolConfig: alert_watermark must be in (0, 1]");
    if (c.metric != BIVF_METRIC_L2 && c.metric != BIVF_METRIC_IP)
        throw Error(BIVF_EINVAL, "metric must be BIVF_METRIC_L2 or BIVF_METRIC_IP");
    if (c.num_blocks > 0x7fffffffull) throw Error(BIVF_EINVAL, "num_blocks exceeds int32 block ids");
    if (c.dim > 65536) throw Error(BIVF_EINVAL, "dim above 65536 is not supported");
}

}  // namespace

// ========================================================================
// construction
// ========================================================================

GpuIndex::GpuIndex(const bivf_config& in) : cfg_(normalized(in)) {
    validate(cfg_);
    C_ = (uint32_t)cfg_.num_clusters;
    D_ = (uint32_t)cfg_.dim;
    Dp_ = pad4(D_);
    T_ = (uint32_t)cfg_.block_capacity;
    gpb_ = ceil_div(T_, 32);
    PS_ = (uint64_t)gpb_ * 32u * D_;
    NB_ = (uint32_t)cfg_.num_blocks;
    // block-table rows start small and grow on demand (grow_rows) up to the
    // configured cap (default: the pool size, i.e. never an insert failure)
    MLB_cap_ = std::max<uint32_t>(1, std::min<uint32_t>(cfg_.max_list_blocks, NB_));
    // (64 entries per list: 2 x 256 B per list, so a Zipf-hot list's chain rarely
    // forces a table reallocation while searches run)
    MLB_ = std::min<uint32_t>(MLB_cap_, std::max<uint32_t>(64, 4 * ceil_div(NB_, C_)));
    {
        const char* v = std::getenv("BIVF_COW");
        cow_on_ = !(v && std::string(v) == "0");
        NS_ = cow_on_ ? std::min<uint32_t>(256, std::max<uint32_t>(16, NB_ / 8)) : 0;
    }
    device_ = cfg_.device;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        throw Error(BIVF_ECUDA, "no CUDA device visible: the B200 path has no CPU fallback");
    }
    if (device_ < 0 || device_ >= ndev) throw Error(BIVF_EINVAL, "device ordinal out of range");
    BIVF_CUDA(cudaSetDevice(device_));
    BIVF_CUDA(cudaDeviceGetAttribute(&num_sms_, cudaDevAttrMultiProcessorCount, device_));
    // every host<->device copy/memset of the index goes through data_stream_
    // (h2d/d2h/dset): the legacy stream does not order against the index's
    // non-blocking streams, and a pageable cudaMemcpy may return before its DMA lands.
    {
        // searches run on high-priority lease streams, the data lane (inserts,
        // maintenance) on the lowest priority: pending search blocks are
        // dispatched first when both contend for SMs
        int lo = 0, hi = 0;
        BIVF_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        prio_hi_ = hi;
        BIVF_CUDA(cudaStreamCreateWithPriority(&data_stream_, cudaStreamNonBlocking, lo));
        data_lease_.stream = data_stream_;
    }
    h_sel_.assign(C_, 0);
    alloc_device();
    BIVF_CUDA(cudaEventCreateWithFlags(&maint_evt_, cudaEventDisableTiming));
    for (uint32_t i = 0; i < cfg_.num_leases; ++i) {
        auto l = std::make_unique<Lease>();
        l->id = (int)i;
        leases_.push_back(std::move(l));
    }
    h_len_.assign(C_, 0);
    h_off_count_.assign(C_, 0);
    h_nblocks_.assign(C_, 0);
    h_off_start_.assign(C_, 0);
    h_head_.assign(C_, -1);
    h_tail_.assign(C_, -1);
    h_blocks_.assign(C_, {});
    h_prev_.assign(NB_, -1);
    h_next_.assign(NB_, -1);
    h_owner_.assign(NB_, -1);
    h_mid_.assign(NB_, -1);
    h_merged_.assign(NB_, 0);
}

GpuIndex::~GpuIndex() {
    cudaSetDevice(device_);
    cudaDeviceSynchronize();
    for (auto& l : leases_) {
        for (auto& g : l->graphs) cudaGraphExecDestroy(g.exec);
        if (l->stream) cudaStreamDestroy(l->stream);
        for (cudaEvent_t e : {l->done, l->t0, l->t1, l->t2, l->t3, l->t4})
            if (e) cudaEventDestroy(e);
    }
    if (data_stream_) cudaStreamDestroy(data_stream_);
    if (maint_evt_) cudaEventDestroy(maint_evt_);
}

void GpuIndex::alloc_device() {
    // block_store.cpp:19-29: whole arena reserved and zero-filled up front,
    // ids -1; here in HBM.
    d_cent_.alloc((size_t)C_ * D_ * 4);
    d_cent_il_.alloc((size_t)ceil_div(C_, 32) * 32 * D_ * 4);
    BIVF_CUDA(dset(d_cent_.p, 0, d_cent_.bytes));
    BIVF_CUDA(dset(d_cent_il_.p, 0, d_cent_il_.bytes));
    d_off_start_.alloc((size_t)C_ * 8);
    d_off_count_.alloc((size_t)C_ * 4);
    BIVF_CUDA(dset(d_off_start_.p, 0, d_off_start_.bytes));
    BIVF_CUDA(dset(d_off_count_.p, 0, d_off_count_.bytes));
    // the scan mirror exists iff the tensor-core scan can serve this index
    // (L2, 8 <= D <= 128) and it was not disabled (BIVF_SCAN=cuda)
    {
        const char* m = std::getenv("BIVF_SCAN");
        mir_on_ = tc_supported(D_, 1, cfg_.metric) && !(m && std::string(m) == "cuda");
        GF_ = cfg_.metric == BIVF_METRIC_IP ? mirror_group_floats_wide(D_) : mirror_group_floats(D_);
        MPS_ = (uint64_t)gpb_ * GF_;
        tc_ok_ = mir_on_;
    }
    ensure_offline_capacity(32);
    // the pool's blocks, then NS_ scratch blocks (copy-on-write maintenance)
    const uint64_t NBS = (uint64_t)NB_ + NS_;
    d_arena_.alloc((size_t)NBS * PS_ * 4);
    BIVF_CUDA(dset(d_arena_.p, 0, d_arena_.bytes));
    if (mir_on_) {
        d_arena_mir_.alloc((size_t)NBS * MPS_ * 4);
        BIVF_CUDA(dset(d_arena_mir_.p, 0, d_arena_mir_.bytes));
        d_arena_nrm_.alloc((size_t)NBS * gpb_ * kNormFloats * 4);
        BIVF_CUDA(dset(d_arena_nrm_.p, 0, d_arena_nrm_.bytes));
        // the slot-major row copy feeds the L2 refine's gathers; the inner-product
        // (wide, D <= 768) refine reads the interleaved payload instead: at D = 768
        // a second copy of the payload would not fit next to it in HBM
        if (cfg_.metric != BIVF_METRIC_IP) {
            d_arena_rows_.alloc((size_t)NBS * PS_ * 4);
            BIVF_CUDA(dset(d_arena_rows_.p, 0, d_arena_rows_.bytes));
        }
        tc_ok_ = make_mirror_map(d_arena_mir_.as<float>(), NBS * gpb_, D_, cfg_.metric == BIVF_METRIC_IP,
                                 &map_arena_) ==
                 cudaSuccess;
        maps_h_ok_ = cfg_.metric != BIVF_METRIC_IP &&
                     make_vm_maps(d_arena_mir_.as<float>(), d_arena_nrm_.as<float>(), NBS * gpb_, D_, &maps_h_[3]) ==
                         cudaSuccess;
    }
    mirror_ = mirror_view();
    d_bids_.alloc((size_t)NBS * T_ * 8);
    BIVF_CUDA(dset(d_bids_.p, 0xff, d_bids_.bytes));
    d_owner_.alloc((size_t)NB_ * 4);
    BIVF_CUDA(dset(d_owner_.p, 0xff, d_owner_.bytes));
    d_cursor_.alloc(16);
    BIVF_CUDA(dset(d_cursor_.p, 0, 16));
    d_len_.alloc((size_t)C_ * 4);
    d_nblocks_.alloc((size_t)C_ * 4);
    d_fail_.alloc((size_t)C_);
    BIVF_CUDA(dset(d_len_.p, 0, d_len_.bytes));
    BIVF_CUDA(dset(d_nblocks_.p, 0, d_nblocks_.bytes));
    BIVF_CUDA(dset(d_fail_.p, 0, d_fail_.bytes));
    d_rows_.alloc((size_t)2 * C_ * MLB_ * 4);
    BIVF_CUDA(dset(d_rows_.p, 0xff, d_rows_.bytes));
    d_ver_.alloc((size_t)C_ * 4);
    BIVF_CUDA(dset(d_ver_.p, 0, d_ver_.bytes));
    d_rowptr_.alloc((size_t)C_ * 8);
    {
        std::vector<uint64_t> rp(C_);
        for (uint32_t c = 0; c < C_; ++c) rp[c] = row_addr(c, 0);
        BIVF_CUDA(h2d(d_rowptr_.p, rp.data(), rp.size() * 8));
    }
    if (const char* m = std::getenv("BIVF_SCAN")) {
        if (std::string(m) == "cuda") scan_mode_ = 1;
        if (std::string(m) == "tc") scan_mode_ = 2;
    }
    d_run_.alloc((size_t)C_ * 4);
    d_failfrom_.alloc((size_t)C_ * 4);
    d_newlen_.alloc((size_t)C_ * 4);
    d_ctr_.alloc(16);
    BIVF_CUDA(cudaDeviceSynchronize());
}

void GpuIndex::ensure_offline_capacity(uint64_t slots) {
    slots = std::max<uint64_t>(32, (slots + 31) / 32 * 32);
    if (slots <= off_slots_cap_) return;
    ++gen_;  // cached search graphs embed the old buffers and TMA extents
    d_off_pay_.alloc((size_t)slots * D_ * 4);
    d_off_ids_.alloc((size_t)slots * 8);
    BIVF_CUDA(dset(d_off_pay_.p, 0, d_off_pay_.bytes));
    BIVF_CUDA(dset(d_off_ids_.p, 0xff, d_off_ids_.bytes));
    off_slots_cap_ = slots;
    if (mir_on_) {
        d_off_mir_.alloc((size_t)(slots / 32) * GF_ * 4);
        BIVF_CUDA(dset(d_off_mir_.p, 0, d_off_mir_.bytes));
        d_off_nrm_.alloc((size_t)(slots / 32) * kNormFloats * 4);
        BIVF_CUDA(dset(d_off_nrm_.p, 0, d_off_nrm_.bytes));
        if (cfg_.metric != BIVF_METRIC_IP) {  // see alloc_device: no row copy for the IP mirror
            d_off_rows_.alloc((size_t)slots * D_ * 4);
            BIVF_CUDA(dset(d_off_rows_.p, 0, d_off_rows_.bytes));
        }
        if (make_mirror_map(d_off_mir_.as<float>(), slots / 32, D_, cfg_.metric == BIVF_METRIC_IP, &map_off_) !=
            cudaSuccess)
            tc_ok_ = false;
        if (cfg_.metric != BIVF_METRIC_IP &&
            make_vm_maps(d_off_mir_.as<float>(), d_off_nrm_.as<float>(), slots / 32, D_, &maps_h_[0]) != cudaSuccess)
            maps_h_ok_ = false;
    }
    mirror_ = mirror_view();
}

MirrorView GpuIndex::mirror_view() const {
    MirrorView M{};
    M.off_mir = d_off_mir_.as<float>();
    M.arena_mir = d_arena_mir_.as<float>();
    M.off_nrm = d_off_nrm_.as<float>();
    M.arena_nrm = d_arena_nrm_.as<float>();
    M.off_rows = d_off_rows_.as<float>();
    M.arena_rows = d_arena_rows_.as<float>();
    M.cent = d_cent_.as<float>();
    M.D = D_;
    M.wide = cfg_.metric == BIVF_METRIC_IP ? 1u : 0u;
    M.K = M.wide ? mirror_k_wide(D_) : mirror_k(D_);
    M.T = T_;
    M.gpb = gpb_;
    M.GF = GF_;
    M.MPS = MPS_;
    return M;
}

// Recompute the whole mirror from the payload (centroids changed under data).
// Caller holds data_mu_.
void GpuIndex::rebuild_mirror() {
    if (!mir_on_) return;
    std::vector<uint64_t> g;
    std::vector<uint32_t> cl;
    for (uint32_t c = 0; c < C_; ++c)
        for (uint64_t j = 0; j < (h_off_count_[c] + 31ull) / 32; ++j) {
            g.push_back(h_off_start_[c] / 32 + j);
            cl.push_back(c);
        }
    std::vector<uint64_t> ga;
    std::vector<uint32_t> cla;
    for (uint32_t b = 0; b < h_cursor_; ++b)
        if (h_owner_[b] >= 0)
            for (uint32_t j = 0; j < gpb_; ++j) {
                ga.push_back((uint64_t)b * gpb_ + j);
                cla.push_back((uint32_t)h_owner_[b]);
            }
    DevBuf dg, dc;
    for (int pass = 0; pass < 2; ++pass) {
        auto& G = pass ? ga : g;
        auto& CL = pass ? cla : cl;
        if (G.empty()) continue;
        dg.ensure(G.size() * 8);
        dc.ensure(CL.size() * 4);
        BIVF_CUDA(h2d(dg.p, G.data(), G.size() * 8));
        BIVF_CUDA(h2d(dc.p, CL.data(), CL.size() * 4));
        BIVF_CUDA(launch_mirror_groups(mirror_, pass ? d_arena_.as<float>() : d_off_pay_.as<float>(),
                                       pass == 1, PS_, dg.as<uint64_t>(), dc.as<uint32_t>(),
                                       (uint32_t)G.size(), data_stream_));
        BIVF_CUDA(cudaStreamSynchronize(data_stream_));
    }
}

// The coarse quantizer as a tensor-core search: ONE list holding every
// centroid (offline segment = the interleaved centroids, ids = cluster ids),
// centred at the centroid mean.  TC filter + exact refine returns exactly the
// CUDA-core quantizer's (dist, cluster) top-P (ivf_index.cpp:271-276).
void GpuIndex::build_quantizer_mirror(const float* c) {
    q_tc_ok_ = false;
    if (!mir_on_ || C_ < 64) return;
    // L2: 3xBF16 over centroids centred at their mean (dense mode + selection);
    // inner product: the wide 1xFP16 mirror of the raw centroids (filter + refine)
    const bool wide = cfg_.metric == BIVF_METRIC_IP;
    const uint32_t ngq = ceil_div(C_, 32);
    std::vector<float> mu(D_, 0.f);
    for (uint32_t k = 0; k < C_; ++k)
        for (uint32_t d = 0; d < D_; ++d) mu[d] += c[(size_t)k * D_ + d];
    for (uint32_t d = 0; d < D_; ++d) mu[d] /= (float)C_;
    d_q_mu_.alloc((size_t)D_ * 4);
    BIVF_CUDA(h2d(d_q_mu_.p, mu.data(), (size_t)D_ * 4));
    d_q_mir_.alloc((size_t)ngq * GF_ * 4);
    BIVF_CUDA(dset(d_q_mir_.p, 0, d_q_mir_.bytes));
    d_q_nrm_.alloc((size_t)ngq * kNormFloats * 4);
    std::vector<long long> ids((size_t)ngq * 32);
    for (size_t i = 0; i < ids.size(); ++i) ids[i] = i < C_ ? (long long)i : -1;
    d_q_ids_.alloc(ids.size() * 8);
    BIVF_CUDA(h2d(d_q_ids_.p, ids.data(), ids.size() * 8));
    // meta: off_start u64 = 0 | off_count u32 = C | len u32 = 0 | rowptr u64 = 0 | ver u32 = 0
    struct {
        uint64_t off_start;
        uint32_t off_count, len;
        uint64_t rowptr;
        uint32_t ver, pad;
    } meta{0, C_, 0, 0, 0, 0};
    d_q_meta_.alloc(sizeof(meta));
    BIVF_CUDA(h2d(d_q_meta_.p, &meta, sizeof(meta)));
    d_q_zero_.alloc((size_t)65536 * 8);
    BIVF_CUDA(dset(d_q_zero_.p, 0, d_q_zero_.bytes));
    MirrorView M{};
    M.off_mir = d_q_mir_.as<float>();
    M.off_nrm = d_q_nrm_.as<float>();
    M.cent = d_q_mu_.as<float>();
    M.D = D_;
    M.wide = wide ? 1u : 0u;
    M.K = wide ? mirror_k_wide(D_) : mirror_k(D_);
    M.T = 32;
    M.gpb = 1;
    M.GF = GF_;
    M.MPS = GF_;
    std::vector<uint64_t> g(ngq);
    std::vector<uint32_t> cl(ngq, 0);
    for (uint32_t i = 0; i < ngq; ++i) g[i] = i;
    DevBuf dg, dc;
    dg.alloc(g.size() * 8);
    dc.alloc(cl.size() * 4);
    BIVF_CUDA(h2d(dg.p, g.data(), g.size() * 8));
    BIVF_CUDA(h2d(dc.p, cl.data(), cl.size() * 4));
    BIVF_CUDA(launch_mirror_groups(M, d_cent_il_.as<float>(), false, (uint64_t)32 * D_,
                                   dg.as<uint64_t>(), dc.as<uint32_t>(), ngq, data_stream_));
    BIVF_CUDA(cudaStreamSynchronize(data_stream_));
    q_tc_ok_ = make_mirror_map(d_q_mir_.as<float>(), ngq, D_, wide, &map_q_) == cudaSuccess;
    // the vector-major scan's maps over the same mirror (L2 quantizer through scan_vm_kernel)
    q_vm_ok_ = !wide && D_ <= 128 && make_vm_maps(d_q_mir_.as<float>(), d_q_nrm_.as<float>(), ngq, D_, &q_vm_maps_[0]) ==
                                         cudaSuccess;
    for (int i = 0; i < 3; ++i) q_vm_maps_[3 + i] = q_vm_maps_[i];  // no arena part
}

bool GpuIndex::use_tc_quantizer(uint32_t P) const {
    // inner product: filter mode (k = P <= 32); L2: dense mode up to 256
    return q_tc_ok_ && scan_mode_ != 1 && P <= (cfg_.metric == BIVF_METRIC_IP ? 32u : 256u) && P < C_;
}

uint32_t GpuIndex::quantizer_slice() const {
    const uint64_t ld = (uint64_t)ceil_div(C_, 32) * 32;
    return (uint32_t)std::max<uint64_t>(128, std::min<uint64_t>(65536, (1ull << 27) / ld));
}

uint32_t GpuIndex::quantizer_maxch(uint32_t nq) const {
    static const uint32_t min_ch = [] {  // tuning aid: at least this many centroid chunks
        const char* v = std::getenv("BIVF_QMAXCH");
        return v ? (uint32_t)atoi(v) : 1u;
    }();
    const uint32_t tiles = ceil_div(nq, 128u), ngq = ceil_div(C_, 32u);
    const uint32_t want = std::max(min_ch, ceil_div((uint32_t)num_sms_, std::max(1u, tiles)));
    return std::max(1u, std::min(want, std::max(1u, ngq / 4)));
}

DevLists GpuIndex::quantizer_lists() const {
    DevLists L;
    L.C = 1;
    L.D = D_;
    L.T = 32;
    L.gpb = 1;
    L.PS = (uint64_t)32 * D_;
    char* m = d_q_meta_.as<char>();
    L.off_payload = d_cent_il_.as<float>();
    L.off_ids = d_q_ids_.as<long long>();
    L.off_start = reinterpret_cast<const uint64_t*>(m);
    L.off_count = reinterpret_cast<const uint32_t*>(m + 8);
    L.len = reinterpret_cast<const uint32_t*>(m + 12);
    L.rowptr = reinterpret_cast<const int32_t* const*>(m + 16);
    L.ver = reinterpret_cast<const uint32_t*>(m + 24);
    L.arena = nullptr;
    L.bids = nullptr;
    return L;
}

// w.queries -> w.probes (P lowest (key, cluster)) + w.pdist, on stream s.
void GpuIndex::enqueue_quantizer(cudaStream_t s, uint32_t nq, uint32_t P, uint32_t fnch,
                                 Workspace& w, uint32_t qbase) {
    static const uint32_t tcq_min = [] {  // smallest batch for the TC quantizer (tuning knob)
        const char* v = std::getenv("BIVF_TCQ_MIN");
        return v ? (uint32_t)atoi(v) : 0u;
    }();
    static const bool vm_quant = [] {  // 1: the L2 quantizer through scan_vm_kernel (measured slower at the
        const char* v = std::getenv("BIVF_VM_QUANT");  // north star: 0.37 vs 0.22 ms per 10K; kept for comparison)
        return v && v[0] == '1';
    }();
    if (vm_quant && q_vm_ok_ && use_tc_quantizer(P) && P <= 32 && nq <= 65536 && nq >= tcq_min) {
        // L2, nprobe <= 32: the centroid set as one list through the vector-major scan
        // (tcgen05 filter over the centroid mirror's bf16 hi plane, exact top-nprobe by
        // the refine over the row-major centroids: the reference's distance bits)
        const uint32_t qsl = quantizer_slice();
        for (uint32_t q0 = 0; q0 < nq; q0 += qsl) {
            const uint32_t m = std::min(qsl, nq - q0);
            SearchShape qs;
            qs.nq = m;
            qs.k = P;
            qs.P = 1;
            qs.maxch = quantizer_maxch(m);  // carve reserved nq x quantizer_maxch(nq) x 2 runs
            qs.gcmin = 4;
            qs.QT = 32;
            qs.metric = cfg_.metric;
            const size_t g0 = (size_t)qbase + q0;
            BIVF_CUDA(launch_ivf_search_tc(quantizer_lists(), w.plan, d_q_zero_.as<long long>(),
                                           w.queries + g0 * Dp_, d_q_mu_.as<float>(), qs, map_q_, map_q_,
                                           d_q_nrm_.as<float>(), nullptr, d_cent_.as<float>(), nullptr, w.tc,
                                           nullptr, w.pdist + g0 * P, w.probes + g0 * P, nullptr, num_sms_, s,
                                           nullptr, nullptr, 1 << 30, q_vm_maps_));
        }
        return;
    }
    if (use_tc_quantizer(P) && nq <= 65536 && nq >= tcq_min) {
        // dense mode: approximate distances of every (query, centroid) on the
        // tensor cores, then a per-query selection + exact recompute of the few
        // centroids whose lower bound can reach the P-th upper bound
        const uint32_t ld = ceil_div(C_, 32) * 32, qsl = quantizer_slice();
        for (uint32_t q0 = 0; q0 < nq; q0 += qsl) {
            const uint32_t m = std::min(qsl, nq - q0);
            SearchShape qs;
            qs.nq = m;
            qs.k = P;
            qs.P = 1;
            qs.maxch = quantizer_maxch(m);
            qs.gcmin = 2;
            qs.QT = 128;
            qs.metric = cfg_.metric;
            // per-(query, group) bound minima: the selection opens only the groups
            // whose minimum can reach its thresholds
            // (written only when selective: several groups per wanted probe, as the
            // selection requires)
            TcDense dn{w.qdense, w.qdense_nq, ld, C_, nullptr,
                       ceil_div(C_, 32) >= 4 * P ? w.qgsum : nullptr};
            // both metrics: dense keys + exact selection (measured: L2 filter mode 0.39 vs
            // 0.18 ms dense; inner product, D = 768, filter + refine vs dense: see DESIGN 6)
            static const bool ip_filter = [] {  // comparison aid: the round-1 IP filter mode
                const char* v = std::getenv("BIVF_IPQ_FILTER");
                return v && v[0] == '1';
            }();
            const bool ip = cfg_.metric == BIVF_METRIC_IP && ip_filter;
            const size_t g0 = (size_t)qbase + q0;
            // work items = tiles x chunks (the centroid list has no online part)
            const uint32_t ngq = ceil_div(C_, 32);
            const uint32_t gcq = std::max(2u, ceil_div(ngq, qs.maxch));
            const int items = (int)(ceil_div(m, 128) * ceil_div(ngq, gcq));
            BIVF_CUDA(launch_ivf_search_tc(quantizer_lists(), w.plan, d_q_zero_.as<long long>(),
                                           w.queries + g0 * Dp_, d_q_mu_.as<float>(), qs,
                                           map_q_, map_q_, d_q_nrm_.as<float>(), nullptr,
                                           d_cent_.as<float>(), nullptr, w.tc, ip ? nullptr : &dn,
                                           w.pdist + g0 * P, w.probes + g0 * P,
                                           nullptr, num_sms_, s, nullptr, nullptr, items));
        }
    } else {
        BIVF_CUDA(launch_flat_topk(d_cent_il_.as<float>(), C_, D_, w.queries + (size_t)qbase * Dp_,
                                   nq, P, cfg_.metric, fnch, w.fcand_d, w.fcand_i,
                                   w.pdist + (size_t)qbase * P, w.probes + (size_t)qbase * P,
                                   nullptr, w.ctr, num_sms_, s));
    }
}

DevLists GpuIndex::dev_lists() const {
    DevLists L;
    L.C = C_;
    L.D = D_;
    L.T = T_;
    L.gpb = gpb_;
    L.PS = PS_;
    L.off_payload = d_off_pay_.as<float>();
    L.off_ids = d_off_ids_.as<long long>();
    L.off_start = d_off_start_.as<uint64_t>();
    L.off_count = d_off_count_.as<uint32_t>();
    L.arena = d_arena_.as<float>();
    L.bids = d_bids_.as<long long>();
    L.rowptr = d_rowptr_.as<const int32_t* const>();
    L.len = d_len_.as<uint32_t>();
    L.ver = d_ver_.as<uint32_t>();
    return L;
}

InsertState GpuIndex::insert_state() {
    InsertState S;
    S.C = C_;
    S.D = D_;
    S.T = T_;
    S.MLB = MLB_;
    S.num_blocks = NB_;
    S.PS = PS_;
    S.arena = d_arena_.as<float>();
    S.bids = d_bids_.as<long long>();
    S.owner = d_owner_.as<int32_t>();
    S.cursor = d_cursor_.as<uint32_t>();
    S.len = d_len_.as<uint32_t>();
    S.nblocks = d_nblocks_.as<uint32_t>();
    S.fail = d_fail_.as<uint8_t>();
    S.rowptr = d_rowptr_.as<int32_t* const>();
    S.run = d_run_.as<uint32_t>();
    S.fail_from = d_failfrom_.as<uint32_t>();
    S.newlen = d_newlen_.as<uint32_t>();
    return S;
}

// ========================================================================
// centroids, training, bulk load
// ========================================================================

void GpuIndex::upload_centroids() {
    // row-major copy (interchange) + interleaved copy (quantizer scan source)
    BIVF_CUDA(launch_interleave(d_cent_.as<float>(), C_, D_, d_cent_il_.as<float>(), data_stream_));
    BIVF_CUDA(cudaStreamSynchronize(data_stream_));
}

void GpuIndex::set_centroids(const float* c) {
    std::lock_guard<std::mutex> lk(data_mu_);
    BIVF_CUDA(cudaSetDevice(device_));
    // centroids, the quantizer mirror and the residual mirror change under the
    // data: searches are quiesced
    std::unique_lock<std::shared_mutex> gx(gate_);
    begin_maintenance();
    BIVF_CUDA(cudaStreamSynchronize(data_stream_));
    struct End {
        GpuIndex* g;
        ~End() { g->end_maintenance(); }
    } end_guard{this};
    ++gen_;
    BIVF_CUDA(h2d(d_cent_.p, c, (size_t)C_ * D_ * 4));
    upload_centroids();
    build_quantizer_mirror(c);
    trained_ = true;
    bool any = false;
    for (uint32_t k = 0; k < C_ && !any; ++k) any = h_off_count_[k] > 0 || h_len_[k] > 0;
    if (any) rebuild_mirror();
}

void GpuIndex::get_centroids(float* out) const {
    BIVF_CUDA(cudaSetDevice(device_));
    BIVF_CUDA(d2h(out, d_cent_.p, (size_t)C_ * D_ * 4));
}

void GpuIndex::train(const float* x, uint64_t n) {
    // ivf_index.cpp:47-59
    if (n < C_) throw Error(BIVF_EINVAL, "train: need at least num_clusters offline vectors");
    std::vector<float> cent((size_t)C_ * D_);
    std::vector<uint32_t> asg(n);
    kmeans_gpu(x, n, D_, C_, cfg_.kmeans_iters, cfg_.kmeans_seed, device_, cent.data(),
               asg.data());
    set_centroids(cent.data());
    bulk_load(x, n, asg.data(), nullptr);
}

void GpuIndex::bulk_load(const float* x, uint64_t n, const uint32_t* assignment,
                         const int64_t* ids) {
    std::vector<uint32_t> asg_local;
    if (!assignment) {
        if (!trained_) throw Error(BIVF_ELOGIC, "bulk_load: index has no centroids");
        asg_local.resize(n);
        assign(x, n, asg_local.data());
        assignment = asg_local.data();
    }
    std::lock_guard<std::mutex> lk(data_mu_);
    BIVF_CUDA(cudaSetDevice(device_));
    // a bulk load rewrites the offline area in place: searches are quiesced
    std::unique_lock<std::shared_mutex> gx(gate_);
    begin_maintenance();
    BIVF_CUDA(cudaStreamSynchronize(data_stream_));
    struct End {
        GpuIndex* g;
        ~End() { g->end_maintenance(); }
    } end_guard{this};
    // ivf_index.cpp:61-82: per-cluster counts; rows appended in ascending row
    // order; each segment padded to whole groups.
    std::vector<uint64_t> counts(C_, 0);
    for (uint64_t i = 0; i < n; ++i) {
        if (assignment[i] >= C_) throw Error(BIVF_EINVAL, "bulk_load: assignment out of range");
        counts[assignment[i]]++;
    }
    for (uint32_t c = 0; c < C_; ++c)
        if (counts[c] > 0xffffffffull) throw Error(BIVF_EINVAL, "bulk_load: list too long");
    uint64_t total = 0, maxseg = 0;
    for (uint32_t c = 0; c < C_; ++c) {
        h_off_start_[c] = total;
        total += (counts[c] + 31) / 32 * 32;
        maxseg = std::max<uint64_t>(maxseg, (counts[c] + 31) / 32 * 32);
    }
    // free space beside the segments: a delete writes a segment's new version
    // there and frees the old one after a grace period (copy-on-write)
    const uint64_t slack = cow_on_ ? std::max<uint64_t>(total / 4, 64 * maxseg) : 0;
    ensure_offline_capacity(total + slack);
    BIVF_CUDA(dset(d_off_ids_.p, 0xff, d_off_ids_.bytes));
    off_region_.clear();
    off_free_.clear();
    off_pending_.clear();
    for (uint32_t c = 0; c < C_; ++c)
        if (counts[c]) off_region_[h_off_start_[c]] = {c, (counts[c] + 31) / 32 * 32};
    off_free_add(total, off_slots_cap_ - total);
    copy_backend_ = false;
    std::vector<uint64_t> fill(C_, 0);
    const uint64_t chunk = 1ull << 20;
    DevBuf dx, ddest, dids, dasg;
    PinBuf pin;
    std::vector<uint64_t> dest;
    std::vector<long long> idv;
    for (uint64_t s = 0; s < n; s += chunk) {
        const uint64_t m = std::min(chunk, n - s);
        dest.resize(m);
        idv.resize(m);
        for (uint64_t i = 0; i < m; ++i) {
            const uint32_t c = assignment[s + i];
            dest[i] = h_off_start_[c] + fill[c]++;
            idv[i] = ids ? ids[s + i] : (long long)(s + i);
        }
        dx.ensure(m * D_ * 4);
        ddest.ensure(m * 8);
        dids.ensure(m * 8);
        BIVF_CUDA(h2d(dx.p, x + s * D_, m * D_ * 4));
        BIVF_CUDA(h2d(ddest.p, dest.data(), m * 8));
        BIVF_CUDA(h2d(dids.p, idv.data(), m * 8));
        BIVF_CUDA(launch_scatter_rows(dx.as<float>(), (uint32_t)m, D_, ddest.as<uint64_t>(),
                                      dids.as<long long>(), d_off_pay_.as<float>(),
                                      d_off_ids_.as<long long>(), data_stream_));
        if (mir_on_) {
            dasg.ensure(m * 4);
            BIVF_CUDA(h2d(dasg.p, assignment + s, m * 4));
            BIVF_CUDA(launch_mirror_offline(mirror_, (uint32_t)m, dx.as<float>(),
                                            ddest.as<uint64_t>(), dasg.as<uint32_t>(),
                                            data_stream_));
        }
        BIVF_CUDA(cudaStreamSynchronize(data_stream_));
    }
    for (uint32_t c = 0; c < C_; ++c) h_off_count_[c] = (uint32_t)counts[c];
    BIVF_CUDA(h2d(d_off_start_.p, h_off_start_.data(), (size_t)C_ * 8));
    BIVF_CUDA(h2d(d_off_count_.p, h_off_count_.data(), (size_t)C_ * 4));
    // seed samples of the vector-major scan: central offline vectors per list
    if (cfg_.metric != BIVF_METRIC_IP && D_ <= 128) {
        d_samp_rows_.ensure((size_t)C_ * D_ * kSampS * 4);
        d_samp_ids_.ensure((size_t)C_ * kSampS * 8);
        BIVF_CUDA(launch_sample_build(d_off_pay_.as<float>(), d_off_ids_.as<long long>(), d_off_start_.as<uint64_t>(),
                                      d_off_count_.as<uint32_t>(), d_cent_.as<float>(), C_, D_,
                                      d_samp_rows_.as<float>(), d_samp_ids_.as<long long>(), data_stream_));
        BIVF_CUDA(cudaStreamSynchronize(data_stream_));
        samp_on_ = true;
    }
    if (ids) {
        int64_t mx = -1;
        for (uint64_t i = 0; i < n; ++i) {
            supplied_.insert(ids[i]);
            mx = std::max<int64_t>(mx, ids[i]);
        }
        next_id_ = std::max<int64_t>(next_id_, mx + 1);
    } else {
        next_id_ = (int64_t)n;
        offline_end_ = (int64_t)n;
    }
    refresh_size();
}

// ========================================================================
// copy-based baseline backend (baseline_index.cpp:51-103)
// ========================================================================

// Grow the offline-segment area to `slots`, keeping every byte (the block-based
// path never needs this: its area is sized once by bulk_load).
void GpuIndex::grow_offline_preserving(uint64_t slots) {
    if (trace_threshold_us() > 0)
        trace("grow_offline", trace_threshold_us(), "slots " + std::to_string(off_slots_cap_) + " -> " + std::to_string(slots));
    slots = (slots + 31) / 32 * 32;
    if (slots <= off_slots_cap_) return;
    const uint64_t cap = std::max<uint64_t>(slots, off_slots_cap_ * 2);
    BIVF_CUDA(cudaDeviceSynchronize());  // in-flight searches read the old buffers
    auto regrow = [&](DevBuf& b, size_t new_bytes, int fill) {
        DevBuf nb;
        nb.alloc(new_bytes);
        BIVF_CUDA(dset(nb.p, fill, nb.bytes));
        if (b.p && b.bytes) BIVF_CUDA(cudaMemcpy(nb.p, b.p, std::min(b.bytes, new_bytes), cudaMemcpyDeviceToDevice));
        std::swap(b.p, nb.p);
        std::swap(b.bytes, nb.bytes);
    };
    ++gen_;
    regrow(d_off_pay_, (size_t)cap * D_ * 4, 0);
    regrow(d_off_ids_, (size_t)cap * 8, 0xff);
    if (mir_on_) {
        regrow(d_off_mir_, (size_t)(cap / 32) * GF_ * 4, 0);
        regrow(d_off_nrm_, (size_t)(cap / 32) * kNormFloats * 4, 0);
        if (d_off_rows_.p) regrow(d_off_rows_, (size_t)cap * D_ * 4, 0);
        if (make_mirror_map(d_off_mir_.as<float>(), cap / 32, D_, cfg_.metric == BIVF_METRIC_IP, &map_off_) !=
            cudaSuccess)
            tc_ok_ = false;
        if (cfg_.metric != BIVF_METRIC_IP &&
            make_vm_maps(d_off_mir_.as<float>(), d_off_nrm_.as<float>(), cap / 32, D_, &maps_h_[0]) != cudaSuccess)
            maps_h_ok_ = false;
    }
    off_slots_cap_ = cap;
    mirror_ = mirror_view();
}

uint64_t GpuIndex::extend_copy(const float* x, uint64_t n, const int64_t* ids, int64_t* out_ids) {
    if (n == 0) return 0;
    if (!trained_) throw Error(BIVF_ELOGIC, "insert: index has no centroids");
    std::vector<uint32_t> asg(n);
    assign(x, n, asg.data());  // ivf assign, lowest cluster id on ties (ivf_index.cpp:93-105)
    // the baseline's extend excludes searches (baseline_index.cpp:66, :113 share one mutex)
    std::lock_guard<std::mutex> lk(data_mu_);  // lock order: data_mu_, then gate_
    std::unique_lock<std::shared_mutex> gx(gate_);
    BIVF_CUDA(cudaSetDevice(device_));
    begin_maintenance();
    BIVF_CUDA(cudaStreamSynchronize(data_stream_));
    struct End {
        GpuIndex* g;
        ~End() { g->end_maintenance(); }
    } end_guard{this};
    // the copy-based backend owns the offline area from here on (no free-space
    // bookkeeping; deletes take the quiescent path)
    copy_backend_ = true;
    off_free_.clear();
    // bucket the batch per cluster, batch order inside a bucket
    std::vector<std::vector<uint64_t>> buckets(C_);
    for (uint64_t i = 0; i < n; ++i) buckets[asg[i]].push_back(i);
    int64_t base = -1;
    if (!ids) {
        base = next_id_;
        next_id_ += (int64_t)n;
    }
    uint64_t top = 0;
    for (uint32_t c = 0; c < C_; ++c) top = std::max<uint64_t>(top, h_off_start_[c] + (h_off_count_[c] + 31ull) / 32 * 32);
    uint64_t need = top;
    for (uint32_t c = 0; c < C_; ++c)
        if (!buckets[c].empty()) need += (h_off_count_[c] + buckets[c].size() + 31ull) / 32 * 32;
    grow_offline_preserving(need);
    // the batch on device once; per list: copy old groups to a fresh region, append
    DevBuf dx, ddest, dids, dasg;
    dx.alloc(n * D_ * 4);
    BIVF_CUDA(h2d(dx.p, x, n * D_ * 4));
    std::vector<uint64_t> dest(n);
    std::vector<long long> idv(n);
    const uint64_t gfl = mir_on_ ? GF_ : 0;
    for (uint32_t c = 0; c < C_; ++c) {
        if (buckets[c].empty()) continue;
        const uint64_t old_n = h_off_count_[c], add_n = buckets[c].size();
        const uint64_t from = h_off_start_[c], to = top;
        top += (old_n + add_n + 31) / 32 * 32;
        const uint64_t og = (old_n + 31) / 32;  // whole groups of the old list
        if (og) {
            cudaStream_t st = data_stream_;
            BIVF_CUDA(cudaMemcpyAsync(d_off_pay_.as<float>() + to * D_, d_off_pay_.as<float>() + from * D_,
                                      og * 32 * D_ * 4, cudaMemcpyDeviceToDevice, st));
            BIVF_CUDA(cudaMemcpyAsync(d_off_ids_.as<long long>() + to, d_off_ids_.as<long long>() + from,
                                      og * 32 * 8, cudaMemcpyDeviceToDevice, st));
            if (mir_on_) {
                BIVF_CUDA(cudaMemcpyAsync(d_off_mir_.as<float>() + (to / 32) * gfl,
                                          d_off_mir_.as<float>() + (from / 32) * gfl, og * gfl * 4,
                                          cudaMemcpyDeviceToDevice, st));
                BIVF_CUDA(cudaMemcpyAsync(d_off_nrm_.as<float>() + (to / 32) * kNormFloats,
                                          d_off_nrm_.as<float>() + (from / 32) * kNormFloats,
                                          og * kNormFloats * 4, cudaMemcpyDeviceToDevice, st));
                if (d_off_rows_.p)
                    BIVF_CUDA(cudaMemcpyAsync(d_off_rows_.as<float>() + to * D_,
                                              d_off_rows_.as<float>() + from * D_, og * 32 * D_ * 4,
                                              cudaMemcpyDeviceToDevice, st));
            }
        }
        for (uint64_t j = 0; j < add_n; ++j) {
            const uint64_t i = buckets[c][j];
            dest[i] = to + old_n + j;
            idv[i] = ids ? (long long)ids[i] : (long long)(base + (int64_t)i);
            if (out_ids) out_ids[i] = idv[i];
        }
        reallocations_ += 1;
        scalars_copied_ += (old_n + add_n) * D_;
        // the abandoned region keeps no live ids (delete's locate scans the area)
        if (og) {
            BIVF_CUDA(cudaMemsetAsync(d_off_ids_.as<long long>() + from, 0xff, og * 32 * 8, data_stream_));
            off_region_.erase(from);
        }
        off_region_[to] = {c, (old_n + add_n + 31) / 32 * 32};
        h_off_start_[c] = to;
        h_off_count_[c] = (uint32_t)(old_n + add_n);
    }
    ddest.alloc(n * 8);
    dids.alloc(n * 8);
    BIVF_CUDA(h2d(ddest.p, dest.data(), n * 8));
    BIVF_CUDA(h2d(dids.p, idv.data(), n * 8));
    BIVF_CUDA(launch_scatter_rows(dx.as<float>(), (uint32_t)n, D_, ddest.as<uint64_t>(), dids.as<long long>(),
                                  d_off_pay_.as<float>(), d_off_ids_.as<long long>(), data_stream_));
    if (mir_on_) {
        dasg.alloc(n * 4);
        BIVF_CUDA(h2d(dasg.p, asg.data(), n * 4));
        BIVF_CUDA(launch_mirror_offline(mirror_, (uint32_t)n, dx.as<float>(), ddest.as<uint64_t>(),
                                        dasg.as<uint32_t>(), data_stream_));
    }
    BIVF_CUDA(cudaStreamSynchronize(data_stream_));
    BIVF_CUDA(h2d(d_off_start_.p, h_off_start_.data(), (size_t)C_ * 8));
    BIVF_CUDA(h2d(d_off_count_.p, h_off_count_.data(), (size_t)C_ * 4));
    refresh_size();
    return n;  // supplied ids do not move next_id (baseline_index.cpp:68-69)
}

// ========================================================================
// leases
// ========================================================================

Lease* GpuIndex::acquire_lease() {
    std::unique_lock<std::mutex> lk(lease_mu_);
    for (;;) {
        for (auto& l : leases_) {
            if (!l->busy) {
                l->busy = true;
                if (!l->stream) {
                    BIVF_CUDA(cudaSetDevice(device_));
                    BIVF_CUDA(cudaStreamCreateWithPriority(&l->stream, cudaStreamNonBlocking,
                                                           prio_hi_));
                    BIVF_CUDA(cudaEventCreateWithFlags(&l->done, cudaEventDisableTiming));
                    for (cudaEvent_t* e : {&l->t0, &l->t1, &l->t2, &l->t3, &l->t4})
                        BIVF_CUDA(cudaEventCreate(e));
                }
                return l.get();
            }
        }
        lease_cv_.wait(lk);
    }
}

void GpuIndex::release_lease(Lease* l) {
    {
        std::lock_guard<std::mutex> lk(lease_mu_);
        l->busy = false;
    }
    lease_cv_.notify_one();
}

Workspace GpuIndex::carve(Lease& l, uint32_t nq, uint32_t k, uint32_t P, uint32_t maxch,
                          uint32_t fnch) {
    const uint64_t npairs = (uint64_t)nq * P;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += align_up(bytes);
        return o;
    };
    const size_t o_qraw = take((size_t)nq * D_ * 4);
    const size_t o_q = take((size_t)nq * Dp_ * 4);
    const size_t o_probes = take(npairs * 8);
    const size_t o_pdist = take(npairs * 4);
    const size_t ncf = (size_t)nq * fnch * P;
    const size_t o_fcd = take(ncf * 4);
    const size_t o_fci = take(ncf * 8);
    const size_t ncand = npairs * maxch * k;
    const size_t o_cd = take(ncand * 4);
    const size_t o_ci = take(ncand * 8);
    const size_t o_od = take((size_t)nq * k * 4);
    const size_t o_oi = take((size_t)nq * k * 8);
    const size_t o_oc = take((size_t)nq * 4);
    const size_t o_ctr = take(16);
    const size_t o_plan = take((size_t)C_ * 4 * 5 + (size_t)(C_ + 1) * 4 * 2 + 16);
    const size_t o_snap = take((size_t)C_ * 8 * 2);  // snap_start, snap_row
    // TC scan: one run per (pair, chunk, warpgroup); the TC quantizer reuses the
    // same buffers (nq pairs, quantizer_maxch chunks, P upper bounds per run)
    const size_t qruns = (size_t)nq * quantizer_maxch(nq) * 2;
    const size_t runs = std::max<size_t>(npairs * maxch * 2, qruns);
    const size_t o_ub = take(std::max<size_t>(npairs * maxch * 2 * k, qruns * P) * 4);
    const size_t o_cc = take(runs * 4);
    const size_t o_clb = take(runs * kKC * 4);
    const size_t o_clo = take(runs * kKC * 4);
    const size_t o_qthr = take((size_t)nq * 4);
    const size_t o_qdense = take(q_tc_ok_ ? (size_t)std::min<uint32_t>(nq, quantizer_slice()) *
                                                ceil_div(C_, 32) * 32 * 4 : 16);
    const size_t o_qdnq = take((size_t)nq * 4);
    const size_t o_qgsum = take(q_tc_ok_ ? (size_t)std::min<uint32_t>(nq, quantizer_slice()) *
                                               ceil_div(C_, 32) * 8 : 16);
    const size_t o_ppos = take(npairs * 4);
    const size_t o_plist = take(npairs * 4);
    if (off > l.ws.bytes && l.stream) {
        // work already queued on this lease may still use the old workspace
        BIVF_CUDA(cudaStreamSynchronize(l.stream));
    }
    l.ws.ensure(off);
    char* b = static_cast<char*>(l.ws.p);
    Workspace w;
    w.qraw = reinterpret_cast<float*>(b + o_qraw);
    w.queries = reinterpret_cast<float*>(b + o_q);
    w.probes = reinterpret_cast<long long*>(b + o_probes);
    w.pdist = reinterpret_cast<float*>(b + o_pdist);
    w.fcand_d = reinterpret_cast<float*>(b + o_fcd);
    w.fcand_i = reinterpret_cast<long long*>(b + o_fci);
    w.cand_d = reinterpret_cast<float*>(b + o_cd);
    w.cand_i = reinterpret_cast<long long*>(b + o_ci);
    w.out_d = reinterpret_cast<float*>(b + o_od);
    w.out_i = reinterpret_cast<long long*>(b + o_oi);
    w.out_cnt = reinterpret_cast<uint32_t*>(b + o_oc);
    w.ctr = reinterpret_cast<uint32_t*>(b + o_ctr);
    uint32_t* pl = reinterpret_cast<uint32_t*>(b + o_plan);
    w.plan.snap_off = pl;
    w.plan.snap_len = pl + C_;
    w.plan.gc = pl + 2 * C_;
    w.plan.nch = pl + 3 * C_;
    w.plan.cnt = pl + 4 * C_;
    w.plan.qoff = pl + 5 * C_;
    w.plan.item_off = pl + 6 * C_ + 1;
    w.plan.n_items = pl + 7 * C_ + 2;
    w.plan.item_ctr = pl + 7 * C_ + 3;
    w.plan.snap_start = reinterpret_cast<uint64_t*>(b + o_snap);
    w.plan.snap_row = w.plan.snap_start + C_;
    w.tc.ub = reinterpret_cast<float*>(b + o_ub);
    w.tc.ccount = reinterpret_cast<uint32_t*>(b + o_cc);
    w.tc.clb = reinterpret_cast<float*>(b + o_clb);
    w.tc.cloc = reinterpret_cast<uint32_t*>(b + o_clo);
    w.tc.qthr = reinterpret_cast<float*>(b + o_qthr);
    w.qdense = reinterpret_cast<float*>(b + o_qdense);
    w.qdense_nq = reinterpret_cast<float*>(b + o_qdnq);
    w.qgsum = reinterpret_cast<float2*>(b + o_qgsum);
    w.plan.ppos = reinterpret_cast<uint32_t*>(b + o_ppos);
    w.plan.plist = reinterpret_cast<uint32_t*>(b + o_plist);
    return w;
}

namespace {
struct LaunchShape {
    uint32_t maxch, gcmin, fnch;
};
LaunchShape pick_shape(uint32_t nq, uint32_t k, uint32_t P, uint32_t C, int sms) {
    LaunchShape s;
    const uint64_t target = (uint64_t)sms * 8;
    const uint64_t npairs = (uint64_t)nq * P;
    s.maxch = (uint32_t)std::min<uint64_t>(32, std::max<uint64_t>(1, (target + npairs - 1) / npairs));
    s.gcmin = 2;
    if (P > 256) {  // nprobe == num_clusters: no quantizer pass
        s.fnch = 1;
        return s;
    }
    const uint32_t qtq = qt_for(P, 0);
    const uint64_t tiles = (nq + qtq - 1) / qtq;
    const uint32_t ng = (C + 31) / 32;
    s.fnch = (uint32_t)std::min<uint64_t>(ng, std::max<uint64_t>(1, (target + tiles - 1) / tiles));
    (void)k;
    return s;
}
}  // namespace

bool GpuIndex::use_tc(uint32_t k) const {
    if (scan_mode_ == 1 || !tc_ok_) return false;
    return tc_supported(D_, k, cfg_.metric);
}

bool GpuIndex::use_tc_dense(uint32_t k) const {
    if (scan_mode_ == 1 || !tc_ok_) return false;
    return tc_dense_supported(D_, k, cfg_.metric);
}

void GpuIndex::validate_search(uint64_t k, uint64_t nprobe) const {
    // ivf_index.cpp:266-269
    if (k < 1) throw Error(BIVF_EINVAL, "search: k must be >= 1");
    if (nprobe < 1 || nprobe > C_) throw Error(BIVF_EINVAL, "search: nprobe out of [1, num_clusters]");
    if (k > 256) throw Error(BIVF_EINVAL, "search: k above the device top-k capacity (256)");
    if (nprobe > 256 && nprobe != C_)
        throw Error(BIVF_EINVAL, "search: nprobe must be <= 256 or == num_clusters");
    if (!trained_) throw Error(BIVF_ELOGIC, "search: index has no centroids");
}

// Enqueue one search slice on the lease stream: pad -> quantizer -> plan ->
// scan -> merge.  Caller holds gate_ shared.
// pad + coarse quantizer for queries [q0, q0 + m) of the slice (raw rows at
// q_dev_raw_piece), on the lease stream; probes land at their slice offsets.
// fnch: the slice's quantizer chunking (carve sized the CUDA-core quantizer's
// candidate scratch with it).
void GpuIndex::enqueue_probes(Lease& l, const float* q_dev_raw_piece, uint32_t q0, uint32_t m,
                              uint32_t P, uint32_t fnch, Workspace& w) {
    BIVF_CUDA(launch_pad_rows(q_dev_raw_piece, m, D_, Dp_, w.queries + (size_t)q0 * Dp_, l.stream));
    if (P == C_) {
        BIVF_CUDA(launch_all_probes(w.probes + (size_t)q0 * P, m, C_, l.stream));
    } else {
        enqueue_quantizer(l.stream, m, P, fnch, w, q0);
    }
}

// Small-batch searches (the latency path: executor requests of <= 10 queries,
// up to 256) are launch-bound: ~10 dependent kernels and memsets of a few us each.
// Their device work is captured once per (shape, workspace, device-buffer
// signature) into a CUDA graph on the lease and replayed with one launch.  Every
// kernel argument is a function of that key: buffer pointers (the signature),
// the batch shape, and device-side state read at run time (list lengths, the
// plan).  Not for timed runs (event records) or the k > 32 dense path (it reads
// a size back to the host mid-search).
uint64_t GpuIndex::graph_sig() const {
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](uint64_t v) { h = (h ^ v) * 1099511628211ull; };
    for (const DevBuf* b : {&d_off_pay_, &d_off_ids_, &d_off_mir_, &d_off_nrm_, &d_off_rows_, &d_q_mir_,
                            &d_q_nrm_, &d_q_mu_, &d_q_ids_, &d_q_meta_, &d_q_zero_, &d_cent_, &d_cent_il_,
                            &d_arena_, &d_arena_mir_})
        mix(reinterpret_cast<uintptr_t>(b->p));
    mix((uint64_t)scan_mode_);
    mix((uint64_t)tc_ok_ | (uint64_t)q_tc_ok_ << 1 | (uint64_t)mir_on_ << 2);
    mix(gen_.load());  // reallocations and centroid changes (buffer addresses can repeat)
    return h;
}

bool GpuIndex::graph_search(Lease& l, uint32_t m, uint32_t k, uint32_t P, Workspace& w) {
    static const bool env_on = [] {
        const char* v = std::getenv("BIVF_GRAPHS");
        return !(v && std::string(v) == "0");
    }();
    if (!env_on || !graphs_on_.load() || m > 256 || timing_ || use_tc_dense(k)) return false;
    const uint64_t sig = graph_sig();
    for (auto& g : l.graphs)
        if (g.m == m && g.k == k && g.P == P && g.ws == l.ws.p && g.sig == sig) {
            BIVF_CUDA(cudaGraphLaunch(g.exec, l.stream));
            count_launch(g.launches);
            return true;
        }
    const uint64_t t0 = t_launches;
    if (cudaStreamBeginCapture(l.stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cudaGetLastError();
        graphs_on_ = false;
        return false;
    }
    bool threw = false;
    try {
        enqueue_search(l, w.qraw, m, k, P, w);
    } catch (...) {
        threw = true;
    }
    cudaGraph_t g = nullptr;
    const cudaError_t ee = cudaStreamEndCapture(l.stream, &g);
    cudaGraphExec_t ge = nullptr;
    if (threw || ee != cudaSuccess || !g || cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        graphs_on_ = false;  // fall back to direct launches from now on
        return false;
    }
    cudaGraphDestroy(g);
    if (l.graphs.size() >= 8) {
        cudaGraphExecDestroy(l.graphs.front().exec);
        l.graphs.erase(l.graphs.begin());
    }
    l.graphs.push_back({m, k, P, l.ws.p, sig, ge, t_launches - t0});
    BIVF_CUDA(cudaGraphLaunch(ge, l.stream));  // its launches were counted while recording
    return true;
}

void GpuIndex::enqueue_search(Lease& l, const float* q_dev_raw, uint32_t nq, uint32_t k,
                              uint32_t P, Workspace& w) {
    if (timing_) BIVF_CUDA(cudaEventRecord(l.t0, l.stream));
    enqueue_probes(l, q_dev_raw, 0, nq, P, pick_shape(nq, k, P, C_, num_sms_).fnch, w);
    enqueue_scan(l, nq, k, P, w);
}

// plan + list scan + merge/refine over the slice's probes (after enqueue_probes).
void GpuIndex::enqueue_scan(Lease& l, uint32_t nq, uint32_t k, uint32_t P, Workspace& w) {
    const LaunchShape sh = pick_shape(nq, k, P, C_, num_sms_);
    if (timing_) BIVF_CUDA(cudaEventRecord(l.t1, l.stream));
    SearchShape ss;
    ss.nq = nq;
    ss.k = k;
    ss.P = P;
    ss.maxch = sh.maxch;
    if (use_tc(k)) {
        // TC filter: a chunk is cheap to scan but every (pair, chunk) run is merged by
        // the refine's one warp per query, so keep ~2 work items per SM, not 8
        static const uint64_t ipsm = [] {  // work items per SM target (tuning knob)
            const char* v = std::getenv("BIVF_TC_ITEMS_PER_SM");
            return v ? std::max<uint64_t>(1, (uint64_t)atoi(v)) : 2ull;
        }();
        const uint64_t npairs = (uint64_t)nq * P;
        ss.maxch = (uint32_t)std::min<uint64_t>(
            ss.maxch, std::max<uint64_t>(1, (ipsm * num_sms_ + npairs - 1) / npairs));
    }
    ss.gcmin = sh.gcmin;
    ss.QT = qt_for(k, D_);
    ss.metric = cfg_.metric;
    if (use_tc(k)) {
        static const bool stats = std::getenv("BIVF_TC_STATS") != nullptr;  // debugging aid
        const uint64_t runs = (uint64_t)nq * P * ss.maxch * 2;
        if (stats) BIVF_CUDA(cudaMemsetAsync(w.tc.ccount, 0, runs * 4, l.stream));
        BIVF_CUDA(launch_ivf_search_tc(dev_lists(), w.plan, w.probes, w.queries,
                                       d_cent_.as<float>(), ss, map_off_, map_arena_,
                                       d_off_nrm_.as<float>(), d_arena_nrm_.as<float>(),
                                       d_off_rows_.as<float>(), d_arena_rows_.as<float>(), w.tc,
                                       nullptr, w.out_d,
                                       w.out_i, w.out_cnt, num_sms_, l.stream,
                                       timing_ ? l.t2 : nullptr, timing_ ? l.t3 : nullptr, 1 << 30,
                                       maps_h_ok_ && d_arena_rows_.p ? maps_h_ : nullptr,
                                       samp_on_ ? d_samp_rows_.as<float>() : nullptr,
                                       samp_on_ ? d_samp_ids_.as<long long>() : nullptr,
                                       scan_mode_ == 3 ? 1 : scan_mode_ == 4 ? 0 : -1));
        if (stats) {
            std::vector<uint32_t> cc(runs);
            BIVF_CUDA(cudaMemcpyAsync(cc.data(), w.tc.ccount, runs * 4, cudaMemcpyDeviceToHost,
                                      l.stream));
            BIVF_CUDA(cudaStreamSynchronize(l.stream));
            uint64_t ovf = 0, cand = 0, nz = 0;
            for (uint32_t c : cc) {
                if (c == kOverflow) ++ovf;
                else { cand += c; nz += c > 0; }
            }
            std::fprintf(stderr, "[tc-stats] nq=%u P=%u maxch=%u runs=%llu overflow=%llu cand=%llu "
                         "(%.2f/query) nonempty=%llu\n", nq, P, ss.maxch, (unsigned long long)runs,
                         (unsigned long long)ovf, (unsigned long long)cand, (double)cand / nq,
                         (unsigned long long)nz);
        }
    } else if (use_tc_dense(k)) {
        // k > 32: the tensor cores write the approximate distance of every
        // (query, probed vector) pair, a per-query selection takes the exact
        // top-k (scan_tc.cu dense_ivf_select_kernel).  The rows' total size is
        // read back once (one stream sync) to size the lease's dense buffer.
        const uint32_t npairs = nq * P;
        const size_t tmpb = dense_plan_tmp_bytes(C_);
        const size_t o_len = 0, o_off = align_up((size_t)C_ * 8),
                     o_nq = o_off + align_up((size_t)C_ * 8),
                     o_tot = o_nq + align_up((size_t)npairs * 4), o_tmp = o_tot + 256;
        if (o_tmp + tmpb > l.dense_aux.bytes) BIVF_CUDA(cudaStreamSynchronize(l.stream));
        l.dense_aux.ensure(o_tmp + tmpb);
        char* ab = l.dense_aux.as<char>();
        uint64_t* plen = reinterpret_cast<uint64_t*>(ab + o_len);
        uint64_t* poff = reinterpret_cast<uint64_t*>(ab + o_off);
        float* pnq = reinterpret_cast<float*>(ab + o_nq);
        uint64_t* ptot = reinterpret_cast<uint64_t*>(ab + o_tot);
        BIVF_CUDA(launch_dense_plan(dev_lists(), w.plan, w.probes, ss, plen, poff, ab + o_tmp, tmpb,
                                    ptot, l.stream));
        l.dpin.ensure(64);
        BIVF_CUDA(cudaMemcpyAsync(l.dpin.p, ptot, 8, cudaMemcpyDeviceToHost, l.stream));
        BIVF_CUDA(cudaStreamSynchronize(l.stream));
        const uint64_t total = *l.dpin.as<uint64_t>();
        const size_t rows_b = align_up(std::max<size_t>(total, 1) * 4);
        l.dense.ensure(rows_b + std::max<size_t>(total / 32, 1) * 8);
        TcDense dn{l.dense.as<float>(), pnq, 0, 0, poff,
                   reinterpret_cast<float2*>(l.dense.as<char>() + rows_b)};
        BIVF_CUDA(launch_ivf_search_tc(dev_lists(), w.plan, w.probes, w.queries,
                                       d_cent_.as<float>(), ss, map_off_, map_arena_,
                                       d_off_nrm_.as<float>(), d_arena_nrm_.as<float>(),
                                       d_off_rows_.as<float>(), d_arena_rows_.as<float>(), w.tc,
                                       &dn, w.out_d, w.out_i, w.out_cnt, num_sms_, l.stream,
                                       timing_ ? l.t2 : nullptr, timing_ ? l.t3 : nullptr));
    } else {
        BIVF_CUDA(launch_ivf_search(dev_lists(), w.plan, w.probes, w.queries, ss, w.cand_d,
                                    w.cand_i, w.out_d, w.out_i, w.out_cnt, num_sms_, l.stream,
                                    timing_ ? l.t2 : nullptr, timing_ ? l.t3 : nullptr));
    }
    if (timing_) BIVF_CUDA(cudaEventRecord(l.t4, l.stream));
}

void GpuIndex::search(const float* q, uint64_t nq, uint64_t k, uint64_t nprobe, int64_t* out_ids,
                      float* out_d, uint32_t* out_cnt) {
    validate_search(k, nprobe);
    if (nq == 0) return;
    const auto t_in = TClock::now();
    BIVF_CUDA(cudaSetDevice(device_));
    Lease* l = acquire_lease();
    const double us_lease = us_since(t_in);
    struct Rel {
        GpuIndex* g;
        Lease* l;
        ~Rel() { g->release_lease(l); }
    } rel{this, l};
    search_on(l, q, nq, k, nprobe, out_ids, out_d, out_cnt, us_lease);
}

// Serving start-up: one search of `nq` zero queries on EVERY lease (all held at
// once), so each lease's stream, events, workspace, pinned staging and CUDA graph
// for that request shape exist before traffic arrives.  Without it a lease is
// set up by the first request that finds the lower-numbered leases busy, and
// that request (plus every lane waiting behind the device-wide cudaFree of a
// workspace regrowth) pays milliseconds.
void GpuIndex::prewarm(uint64_t nq, uint64_t k, uint64_t nprobe) {
    validate_search(k, nprobe);
    if (nq == 0) return;
    BIVF_CUDA(cudaSetDevice(device_));
    std::vector<float> q((size_t)nq * D_, 0.f);
    std::vector<int64_t> ids((size_t)nq * k);
    std::vector<float> d((size_t)nq * k);
    std::vector<uint32_t> cnt(nq);
    std::vector<Lease*> held;
    struct RelAll {
        GpuIndex* g;
        std::vector<Lease*>& v;
        ~RelAll() {
            for (Lease* l : v) g->release_lease(l);
        }
    } rel{this, held};
    for (size_t i = 0; i < leases_.size(); ++i) held.push_back(acquire_lease());
    for (Lease* l : held) search_on(l, q.data(), nq, k, nprobe, ids.data(), d.data(), cnt.data(), 0.0);
}

void GpuIndex::search_on(Lease* l, const float* q, uint64_t nq, uint64_t k, uint64_t nprobe, int64_t* out_ids,
                         float* out_d, uint32_t* out_cnt, double us_lease) {
    const auto t_in = TClock::now();
    double us_gate = 0, us_enq = 0, us_sync = 0, us_prep = 0;
    const uint64_t slice = 32768;
    for (uint64_t s = 0; s < nq; s += slice) {
        const uint32_t m = (uint32_t)std::min(slice, nq - s);
        const auto t_p = TClock::now();
        const LaunchShape sh = pick_shape(m, (uint32_t)k, (uint32_t)nprobe, C_, num_sms_);
        Workspace w = carve(*l, m, (uint32_t)k, (uint32_t)nprobe, sh.maxch, sh.fnch);
        const size_t in_b = (size_t)m * D_ * 4;
        const size_t out_b = (size_t)m * k * 12 + (size_t)m * 4;
        // page-locked user buffers are DMA'd directly (no host staging copy)
        const bool q_pin = is_pinned(q + s * D_);
        const bool o_pin = is_pinned(out_d + s * k) && is_pinned(out_ids + s * k) &&
                           (!out_cnt || is_pinned(out_cnt + s));
        l->pin.ensure(in_b + out_b + 256);
        us_prep += us_since(t_p);
        char* pin = l->pin.as<char>();
        float* pd = reinterpret_cast<float*>(pin + align_up(in_b, 64));
        long long* pi = reinterpret_cast<long long*>(pd + (size_t)m * k + ((m * k) & 1));
        uint32_t* pc = reinterpret_cast<uint32_t*>(pi + (size_t)m * k);
        {
            const auto t_g = TClock::now();
            std::shared_lock<std::shared_mutex> g(gate_);
            us_gate += us_since(t_g);
            const auto t_e = TClock::now();
            const uint64_t gen = maint_gen_.load();
            if (l->seen_maint != gen) {
                BIVF_CUDA(cudaStreamWaitEvent(l->stream, maint_evt_, 0));
                l->seen_maint = gen;
            }
            // stage the queries in ~1 MB pieces: the DMA of piece i overlaps the
            // host copy of piece i+1 (a per-piece quantizer was measured slower:
            // smaller quantizer launches cost more than the DMA they hide)
            if (q_pin) {
                BIVF_CUDA(cudaMemcpyAsync(w.qraw, q + s * D_, in_b, cudaMemcpyHostToDevice, l->stream));
            } else {
                const size_t piece = std::max<size_t>(1u << 20, (size_t)D_ * 4 * 256);
                for (size_t o = 0; o < in_b; o += piece) {
                    const size_t nb = std::min(piece, in_b - o);
                    par_memcpy(pin + o, reinterpret_cast<const char*>(q + s * D_) + o, nb);
                    BIVF_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(w.qraw) + o, pin + o, nb,
                                              cudaMemcpyHostToDevice, l->stream));
                }
            }
            if (!graph_search(*l, m, (uint32_t)k, (uint32_t)nprobe, w))
                enqueue_search(*l, w.qraw, m, (uint32_t)k, (uint32_t)nprobe, w);
            float* hd = o_pin ? out_d + s * k : pd;
            long long* hi = o_pin ? reinterpret_cast<long long*>(out_ids + s * k) : pi;
            uint32_t* hc = o_pin && out_cnt ? out_cnt + s : pc;
            BIVF_CUDA(cudaMemcpyAsync(hd, w.out_d, (size_t)m * k * 4, cudaMemcpyDeviceToHost, l->stream));
            BIVF_CUDA(cudaMemcpyAsync(hi, w.out_i, (size_t)m * k * 8, cudaMemcpyDeviceToHost, l->stream));
            BIVF_CUDA(cudaMemcpyAsync(hc, w.out_cnt, (size_t)m * 4, cudaMemcpyDeviceToHost, l->stream));
            BIVF_CUDA(cudaEventRecord(l->done, l->stream));
            us_enq += us_since(t_e);
        }
        const auto t_s = TClock::now();
        BIVF_CUDA(cudaEventSynchronize(l->done));
        us_sync += us_since(t_s);
        if (!o_pin) {
            par_memcpy(out_d + s * k, pd, (size_t)m * k * 4);
            par_memcpy(out_ids + s * k, pi, (size_t)m * k * 8);
            if (out_cnt) std::memcpy(out_cnt + s, pc, (size_t)m * 4);
        }
        if (timing_) record_timings(*l);
    }
    if (trace_threshold_us() > 0)
        trace("search", us_since(t_in),
              "nq=" + std::to_string(nq) + " lease=" + std::to_string((int)us_lease) + " prep=" +
                  std::to_string((int)us_prep) + " gate=" +
                  std::to_string((int)us_gate) + " enqueue=" + std::to_string((int)us_enq) + " device_wait=" +
                  std::to_string((int)us_sync));
}

void GpuIndex::shard_open(ShardCtx& s, uint64_t nq, uint64_t k, uint64_t nprobe, uint32_t G) {
    validate_search(k, nprobe);
    if (nq == 0 || G == 0) throw Error(BIVF_EINVAL, "sharded search: empty batch or group");
    if (nq > 0xffffffffull / std::max<uint64_t>(1, nprobe) / G)
        throw Error(BIVF_EINVAL, "sharded search: nq * nprobe too large for one call");
    BIVF_CUDA(cudaSetDevice(device_));
    s.nq = (uint32_t)nq;
    s.k = (uint32_t)k;
    s.P = (uint32_t)nprobe;
    s.slice = ceil_div(nq, G);
    s.nq_pad = s.slice * G;
    s.lease = acquire_lease();
    const LaunchShape sh = pick_shape(s.nq_pad, s.k, s.P, C_, num_sms_);
    s.w = carve(*s.lease, s.nq_pad, s.k, s.P, sh.maxch, sh.fnch);
    s.gate = std::shared_lock<std::shared_mutex>(gate_);
    const uint64_t gen = maint_gen_.load();
    if (s.lease->seen_maint != gen) {
        BIVF_CUDA(cudaStreamWaitEvent(s.lease->stream, maint_evt_, 0));
        s.lease->seen_maint = gen;
    }
}

void GpuIndex::shard_quantize(ShardCtx& s, uint32_t g) {
    BIVF_CUDA(cudaSetDevice(device_));
    cudaStream_t st = s.lease->stream;
    BIVF_CUDA(launch_pad_rows(s.w.qraw, s.nq, D_, Dp_, s.w.queries, st));
    if (s.P == C_) {  // every list probed: every shard fills all rows (no all-gather)
        BIVF_CUDA(launch_all_probes(s.w.probes, s.nq, C_, st));
        return;
    }
    const uint32_t q0 = g * s.slice;
    if (q0 >= s.nq) return;
    const uint32_t m = std::min(s.slice, s.nq - q0);
    enqueue_quantizer(st, m, s.P, pick_shape(s.nq_pad, s.k, s.P, C_, num_sms_).fnch, s.w, q0);
}

void GpuIndex::shard_scan(ShardCtx& s) {
    BIVF_CUDA(cudaSetDevice(device_));
    enqueue_scan(*s.lease, s.nq, s.k, s.P, s.w);
}

void GpuIndex::shard_close(ShardCtx& s) {
    if (!s.lease) return;
    BIVF_CUDA(cudaSetDevice(device_));
    BIVF_CUDA(cudaEventRecord(s.lease->done, s.lease->stream));
    if (s.gate.owns_lock()) s.gate.unlock();
    release_lease(s.lease);
    s.lease = nullptr;
}

void GpuIndex::search_device(const float* q_dev, uint64_t nq, uint64_t k, uint64_t nprobe,
                             int64_t* ids_dev, float* d_dev, uint32_t* cnt_dev,
                             cudaStream_t user) {
    validate_search(k, nprobe);
    if (nq == 0) return;
    if (nq > 0xffffffffull / std::max<uint64_t>(1, nprobe))
        throw Error(BIVF_EINVAL, "search_device: nq * nprobe too large for one call");
    BIVF_CUDA(cudaSetDevice(device_));
    Lease* l = acquire_lease();
    struct Rel {
        GpuIndex* g;
        Lease* l;
        ~Rel() { g->release_lease(l); }
    } rel{this, l};
    const uint32_t m = (uint32_t)nq;
    const LaunchShape sh = pick_shape(m, (uint32_t)k, (uint32_t)nprobe, C_, num_sms_);
    Workspace w = carve(*l, m, (uint32_t)k, (uint32_t)nprobe, sh.maxch, sh.fnch);
    cudaEvent_t ue;
    BIVF_CUDA(cudaEventCreateWithFlags(&ue, cudaEventDisableTiming));
    BIVF_CUDA(cudaEventRecord(ue, user));
    {
        std::shared_lock<std::shared_mutex> g(gate_);
        const uint64_t gen = maint_gen_.load();
        if (l->seen_maint != gen) {
            BIVF_CUDA(cudaStreamWaitEvent(l->stream, maint_evt_, 0));
            l->seen_maint = gen;
        }
        BIVF_CUDA(cudaStreamWaitEvent(l->stream, ue, 0));
        w.out_d = d_dev;
        w.out_i = reinterpret_cast<long long*>(ids_dev);
        w.out_cnt = cnt_dev;
        enqueue_search(*l, q_dev, m, (uint32_t)k, (uint32_t)nprobe, w);
        BIVF_CUDA(cudaEventRecord(l->done, l->stream));
    }
    BIVF_CUDA(cudaStreamWaitEvent(user, l->done, 0));
    cudaEventDestroy(ue);
    // No host sync: the lease's workspace is only ever used on the lease's own
    // stream, so the next search on this lease is stream-ordered after this one.
    if (timing_) {
        BIVF_CUDA(cudaEventSynchronize(l->done));
        record_timings(*l);
    }
}

void GpuIndex::record_timings(Lease& l) {
    cudaEventElapsedTime(&last_ms_[0], l.t0, l.t1);
    cudaEventElapsedTime(&last_ms_[1], l.t1, l.t2);
    cudaEventElapsedTime(&last_ms_[2], l.t2, l.t3);
    cudaEventElapsedTime(&last_ms_[3], l.t3, l.t4);
}

void GpuIndex::last_timings(float* out4) const {
    for (int i = 0; i < 4; ++i) out4[i] = last_ms_[i];
}

void GpuIndex::assign(const float* y, uint64_t n, uint32_t* out) {
    if (!trained_) throw Error(BIVF_ELOGIC, "assign: index has no centroids");
    if (n == 0) return;
    probes(y, n, 1, out);
}

void GpuIndex::probes(const float* q, uint64_t nq, uint64_t nprobe, uint32_t* out) {
    if (nprobe < 1 || nprobe > C_) throw Error(BIVF_EINVAL, "probes: nprobe out of [1, num_clusters]");
    if (nprobe > 256 && nprobe != C_) throw Error(BIVF_EINVAL, "probes: nprobe must be <= 256 or == num_clusters");
    if (!trained_) throw Error(BIVF_ELOGIC, "probes: index has no centroids");
    if (nq == 0) return;
    BIVF_CUDA(cudaSetDevice(device_));
    Lease* l = acquire_lease();
    struct Rel {
        GpuIndex* g;
        Lease* l;
        ~Rel() { g->release_lease(l); }
    } rel{this, l};
    const uint64_t slice = 65536;
    std::vector<long long> tmp;
    for (uint64_t s = 0; s < nq; s += slice) {
        const uint32_t m = (uint32_t)std::min(slice, nq - s);
        const LaunchShape sh = pick_shape(m, 1, (uint32_t)nprobe, C_, num_sms_);
        Workspace w = carve(*l, m, 1, (uint32_t)nprobe, 1, sh.fnch);
        tmp.resize((size_t)m * nprobe);
        BIVF_CUDA(cudaMemcpyAsync(w.qraw, q + s * D_, (size_t)m * D_ * 4, cudaMemcpyHostToDevice,
                                  l->stream));
        BIVF_CUDA(launch_pad_rows(w.qraw, m, D_, Dp_, w.queries, l->stream));
        if (nprobe > 256) {  // == C_: every cluster (cluster-id order)
            BIVF_CUDA(launch_all_probes(w.probes, m, C_, l->stream));
        } else {
            enqueue_quantizer(l->stream, m, (uint32_t)nprobe, sh.fnch, w);
        }
        BIVF_CUDA(cudaMemcpyAsync(tmp.data(), w.probes, tmp.size() * 8, cudaMemcpyDeviceToHost,
                                  l->stream));
        BIVF_CUDA(cudaStreamSynchronize(l->stream));
        for (size_t i = 0; i < tmp.size(); ++i) out[s * nprobe + i] = (uint32_t)tmp[i];
    }
}

// ========================================================================
// insert (ivf_index.cpp:107-164)
// ========================================================================

bool GpuIndex::is_duplicate_id(int64_t id) {
    if (id < 0) return true;
    if (id < offline_end_) return true;
    for (const auto& r : auto_ranges_)
        if (id >= r.first && id < r.second) return true;
    if (!supplied_.insert(id).second) return true;
    if (id >= next_id_) next_id_ = id + 1;
    return false;
}

void GpuIndex::absorb_new_blocks(uint32_t cursor_old, uint32_t cursor_new) {
    if (cursor_new <= cursor_old) return;
    std::vector<int32_t> own(cursor_new - cursor_old);
    BIVF_CUDA(d2h(own.data(), d_owner_.as<int32_t>() + cursor_old, own.size() * 4));
    // Blocks are handed out in batch order, which is each list's logical
    // order: append = link after the tail (block_store.cpp:55-65).
    for (uint32_t b = cursor_old; b < cursor_new; ++b) {
        const int32_t c = own[b - cursor_old];
        if (c < 0 || (uint32_t)c >= C_) throw Error(BIVF_ECORRUPT, "insert: new block without owner");
        h_owner_[b] = c;
        h_mid_[b] = (int32_t)h_blocks_[c].size();
        const int32_t t = h_tail_[c];
        h_prev_[b] = t;
        h_next_[b] = -1;
        h_merged_[b] = 0;
        if (t >= 0) h_next_[t] = (int32_t)b;
        else h_head_[c] = (int32_t)b;
        h_tail_[c] = (int32_t)b;
        h_blocks_[c].push_back((int32_t)b);
        h_nblocks_[c] = (uint32_t)h_blocks_[c].size();
    }
    h_cursor_ = cursor_new;
    // one-shot utilization alert (block_store.cpp:41-46): the first allocation
    // whose used/total strictly exceeds the watermark, reported once
    for (uint64_t used = (uint64_t)cursor_old + 1; !alert_fired_ && used <= cursor_new; ++used)
        if ((double)used / (double)NB_ > cfg_.alert_watermark) {
            alert_fired_ = true;
            alert_used_ = used;
            log_warn("central pool utilization " + std::to_string(used) + "/" + std::to_string(NB_) +
                     " exceeds watermark");
        }
}

void GpuIndex::alert_state(int32_t* fired, uint64_t* used_at) const {
    std::lock_guard<std::mutex> lk(data_mu_);
    if (fired) *fired = alert_fired_ ? 1 : 0;
    if (used_at) *used_at = alert_used_;
}

void GpuIndex::block_set_next(int32_t b, int32_t next) {
    std::lock_guard<std::mutex> lk(data_mu_);
    check_block(b);
    if (next >= 0) check_block(next);
    h_next_[b] = next;
}

void GpuIndex::refresh_lengths() {
    BIVF_CUDA(d2h(h_len_.data(), d_len_.p, (size_t)C_ * 4));
}

uint64_t GpuIndex::insert(const float* x, uint64_t n, const int64_t* ids, int64_t* out_ids) {
    for (uint64_t i = 0; i < n; ++i) out_ids[i] = -1;
    if (n == 0) return 0;
    if (!trained_) throw Error(BIVF_ELOGIC, "insert: index has no centroids");
    const auto t_in = TClock::now();
    std::lock_guard<std::mutex> lk(data_mu_);
    struct Tr {
        TClock::time_point t;
        double lock;
        uint64_t n;
        double ph[5] = {0, 0, 0, 0, 0};  // stage+quantizer enqueue, grow_rows, insert enqueue, sync, absorb
        ~Tr() {
            if (trace_threshold_us() > 0)
                trace("insert", us_since(t), "n=" + std::to_string(n) + " data_mu=" + std::to_string((int)lock) +
                                                 " enqueue=" + std::to_string((int)ph[0]) + " grow_rows=" +
                                                 std::to_string((int)ph[1]) + " insert=" + std::to_string((int)ph[2]) +
                                                 " sync=" + std::to_string((int)ph[3]) + " absorb=" +
                                                 std::to_string((int)ph[4]));
        }
    } tr{t_in, us_since(t_in), n};
    TClock::time_point tp0 = TClock::now();
    auto lap = [&](int i) {
        const auto now = TClock::now();
        tr.ph[i] += std::chrono::duration<double, std::micro>(now - tp0).count();
        tp0 = now;
    };
    BIVF_CUDA(cudaSetDevice(device_));
    // ids: contiguous auto range, or supplied ids checked in batch order
    std::vector<long long> idv(n);
    if (!ids) {
        const int64_t base = next_id_;
        next_id_ += (int64_t)n;
        if (!auto_ranges_.empty() && auto_ranges_.back().second == base)
            auto_ranges_.back().second = base + (int64_t)n;
        else
            auto_ranges_.emplace_back(base, base + (int64_t)n);
        for (uint64_t i = 0; i < n; ++i) idv[i] = base + (int64_t)i;
    } else {
        for (uint64_t i = 0; i < n; ++i) idv[i] = is_duplicate_id(ids[i]) ? -1 : ids[i];
    }
    uint64_t inserted = 0;
    bool exhausted = false;
    const uint64_t chunk = 1ull << 18;
    std::vector<int32_t> blk;
    for (uint64_t s = 0; s < n; s += chunk) {
        const uint32_t m = (uint32_t)std::min(chunk, n - s);
        // staging sized for at least the executor's largest batch (1024) on first
        // use: a buffer regrowth mid-stream (cudaFree / cudaFreeHost synchronise)
        // stalled an insert for ~0.4 s under live search traffic
        const uint32_t mc = std::max<uint32_t>(m, 1024u);
        d_x_.ensure((size_t)mc * D_ * 4);
        d_qtmp_.ensure((size_t)mc * Dp_ * 4);
        d_ids_.ensure((size_t)mc * 8);
        d_asg_.ensure((size_t)mc * 4);
        d_blk_.ensure((size_t)mc * 4);
        d_did_.ensure((size_t)mc * 4);
        const LaunchShape sh = pick_shape(m, 1, 1, C_, num_sms_);
        const LaunchShape shc = pick_shape(mc, 1, 1, C_, num_sms_);
        const size_t fc = std::max((size_t)m * sh.fnch, (size_t)mc * shc.fnch);
        d_fc_d_.ensure(fc * 4);
        d_fc_i_.ensure(fc * 8);
        d_fo_i_.ensure((size_t)mc * 8);
        d_fo_d_.ensure((size_t)mc * 4);
        h_stage_.ensure((size_t)mc * D_ * 4 + (size_t)mc * 8 + 64);
        float* px = h_stage_.as<float>();
        std::memcpy(px, x + s * D_, (size_t)m * D_ * 4);
        long long* pid = reinterpret_cast<long long*>(h_stage_.as<char>() + align_up((size_t)m * D_ * 4, 64));
        std::memcpy(pid, idv.data() + s, (size_t)m * 8);
        cudaStream_t st = data_stream_;
        BIVF_CUDA(cudaMemcpyAsync(d_x_.p, px, (size_t)m * D_ * 4, cudaMemcpyHostToDevice, st));
        BIVF_CUDA(cudaMemcpyAsync(d_ids_.p, pid, (size_t)m * 8, cudaMemcpyHostToDevice, st));
        // assign (ivf_index.cpp:93-105) = quantizer top-1 on device; the TC
        // quantizer sizes its grid to its few work items, so an insert beside
        // live searches occupies a handful of SMs, not the whole GPU
        const long long* nearest = d_fo_i_.as<long long>();
        if (use_tc_quantizer(1) && m <= 65536) {
            // carved for mc queries (the lease workspace keeps its largest size), used for m
            Workspace dw = carve(data_lease_, mc, 1, 1, 1, std::max(sh.fnch, shc.fnch));
            BIVF_CUDA(launch_pad_rows(d_x_.as<float>(), m, D_, Dp_, dw.queries, st));
            enqueue_quantizer(st, m, 1, sh.fnch, dw);
            nearest = dw.probes;
        } else {
            BIVF_CUDA(launch_pad_rows(d_x_.as<float>(), m, D_, Dp_, d_qtmp_.as<float>(), st));
            BIVF_CUDA(launch_flat_topk(d_cent_il_.as<float>(), C_, D_, d_qtmp_.as<float>(), m, 1,
                                       cfg_.metric, sh.fnch, d_fc_d_.as<float>(),
                                       d_fc_i_.as<long long>(), d_fo_d_.as<float>(),
                                       d_fo_i_.as<long long>(), nullptr, d_ctr_.as<uint32_t>(),
                                       num_sms_, st));
        }
        BIVF_CUDA(launch_make_asg(nearest, d_ids_.as<long long>(), m, d_asg_.as<uint32_t>(), st));
        lap(0);
        // block-table rows with room for every block this chunk can open in one list
        uint32_t mxb = 0;
        for (uint32_t c = 0; c < C_; ++c) mxb = std::max(mxb, h_nblocks_[c]);
        grow_rows(mxb + ceil_div(m, T_) + 1);
        lap(1);
        const uint32_t cursor_old = h_cursor_;
        BIVF_CUDA(launch_insert(insert_state(), m, d_x_.as<float>(), d_ids_.as<long long>(),
                                d_asg_.as<uint32_t>(), d_blk_.as<int32_t>(),
                                d_did_.as<uint32_t>(), mirror_ptr(), st));
        blk.resize(m);
        uint32_t cursor_new = 0;
        BIVF_CUDA(cudaMemcpyAsync(blk.data(), d_blk_.p, (size_t)m * 4, cudaMemcpyDeviceToHost, st));
        BIVF_CUDA(cudaMemcpyAsync(h_len_.data(), d_len_.p, (size_t)C_ * 4, cudaMemcpyDeviceToHost, st));
        BIVF_CUDA(cudaMemcpyAsync(&cursor_new, d_cursor_.p, 4, cudaMemcpyDeviceToHost, st));
        lap(2);
        BIVF_CUDA(cudaStreamSynchronize(st));
        lap(3);
        absorb_new_blocks(cursor_old, cursor_new);
        lap(4);
        for (uint32_t i = 0; i < m; ++i) {
            if (idv[s + i] < 0) continue;  // rejected duplicate
            if (blk[i] >= 0) {
                out_ids[s + i] = idv[s + i];
                ++inserted;
            } else {
                exhausted = true;
            }
        }
    }
    scalars_copied_ += inserted * D_;
    refresh_size();
    if (exhausted) {
        Error e(BIVF_EPOOL, "central memory pool exhausted after inserting " +
                                std::to_string(inserted) + " vectors of the batch");
        e.inserted = inserted;
        throw e;
    }
    return inserted;
}

// ========================================================================
// maintenance fencing
// ========================================================================

void GpuIndex::begin_maintenance() {
    // caller holds data_mu_ and gate_ exclusively (see rearrange/remove)
    std::lock_guard<std::mutex> lk(lease_mu_);
    for (auto& l : leases_)
        if (l->done) BIVF_CUDA(cudaStreamWaitEvent(data_stream_, l->done, 0));
}

void GpuIndex::end_maintenance() {
    BIVF_CUDA(cudaEventRecord(maint_evt_, data_stream_));
    maint_gen_.fetch_add(1);
}

// ========================================================================
// read-copy-update maintenance (see index.h)
// ========================================================================

// Grace period.  (1) Everything enqueued on the data stream so far (the
// publishes) has landed on the device.  (2) With gate_ held exclusively no
// search is mid-enqueue, so every search either recorded its lease's `done`
// event already — the data stream waits on it, on the device — or will be
// enqueued after the publishes landed and so plans against the new state.
// Work enqueued on the data stream after this call may reuse whatever the
// old state referenced.  The host never waits for searches.
void GpuIndex::grace() {
    const auto t0 = TClock::now();
    BIVF_CUDA(cudaStreamSynchronize(data_stream_));
    const double us_sync = us_since(t0);
    const auto t1 = TClock::now();
    {
        std::unique_lock<std::shared_mutex> g(gate_);
        std::lock_guard<std::mutex> lk(lease_mu_);
        for (auto& l : leases_)
            if (l->done) BIVF_CUDA(cudaStreamWaitEvent(data_stream_, l->done, 0));
    }
    // offline regions retired before the grace: clear their ids (locate must
    // not find stale copies), then they are free (data-stream order)
    for (auto& r : off_pending_) {
        BIVF_CUDA(cudaMemsetAsync(d_off_ids_.as<long long>() + r.first, 0xff, r.second * 8,
                                  data_stream_));
        off_free_add(r.first, r.second);
    }
    off_pending_.clear();
    grace_pending_ = false;
    if (trace_threshold_us() > 0)
        trace("grace", us_since(t0),
              "data_stream_sync=" + std::to_string((int)us_sync) + " gate+waits=" + std::to_string((int)us_since(t1)));
}

uint64_t GpuIndex::row_addr(uint32_t c, uint32_t sel) const {
    return reinterpret_cast<uint64_t>(d_rows_.as<int32_t>() + ((size_t)sel * C_ + c) * MLB_);
}

GpuIndex::ListPub GpuIndex::current_pub(uint32_t c) const {
    return ListPub{c, h_off_start_[c], h_off_count_[c], row_addr(c, h_sel_[c]), h_len_[c]};
}

// One seqlocked publish of whole list states on the data stream (maint.cu).
void GpuIndex::publish(const std::vector<ListPub>& pubs) {
    const size_t n = pubs.size();
    if (!n) return;
    const size_t o_idx = 0, o_start = align_up(n * 4, 16), o_count = o_start + align_up(n * 8, 16),
                 o_row = o_count + align_up(n * 4, 16), o_len = o_row + align_up(n * 8, 16),
                 total = o_len + align_up(n * 4, 16);
    // sized for every list at once on first use: pinned regrowth (cudaFreeHost +
    // cudaHostAlloc) would stall the lease threads' CUDA calls mid-window
    const size_t full = 48 * (size_t)C_ + 256;
    h_pub_.ensure(std::max(total, full));
    s_pub_.ensure(std::max(total, full));
    char* h = h_pub_.as<char>();
    for (size_t i = 0; i < n; ++i) {
        reinterpret_cast<uint32_t*>(h + o_idx)[i] = pubs[i].c;
        reinterpret_cast<uint64_t*>(h + o_start)[i] = pubs[i].start;
        reinterpret_cast<uint32_t*>(h + o_count)[i] = pubs[i].count;
        reinterpret_cast<uint64_t*>(h + o_row)[i] = pubs[i].row;
        reinterpret_cast<uint32_t*>(h + o_len)[i] = pubs[i].len;
    }
    char* d = s_pub_.as<char>();
    BIVF_CUDA(h2d(d, h, total));
    BIVF_CUDA(launch_publish_lists((uint32_t)n, reinterpret_cast<uint32_t*>(d + o_idx),
                                   reinterpret_cast<uint64_t*>(d + o_start),
                                   reinterpret_cast<uint32_t*>(d + o_count),
                                   reinterpret_cast<uint64_t*>(d + o_row),
                                   reinterpret_cast<uint32_t*>(d + o_len), d_off_start_.as<uint64_t>(),
                                   d_off_count_.as<uint32_t>(), d_rowptr_.as<uint64_t>(),
                                   d_len_.as<uint32_t>(), d_ver_.as<uint32_t>(), data_stream_));
}

// rows[i] (-1 padded to MLB_) -> copy sel[i] of list lists[i]'s row.
void GpuIndex::write_rows(const std::vector<uint32_t>& lists,
                          const std::vector<std::vector<int32_t>>& rows,
                          const std::vector<uint8_t>& sel) {
    if (lists.empty()) return;
    std::vector<int32_t> flat((size_t)lists.size() * MLB_, -1);
    for (size_t i = 0; i < lists.size(); ++i) {
        if (rows[i].size() > MLB_) throw Error(BIVF_ECORRUPT, "block-table row above capacity");
        std::copy(rows[i].begin(), rows[i].end(), flat.begin() + i * MLB_);
    }
    DevBuf& tmp = s_rows_;
    tmp.ensure(flat.size() * 4);
    BIVF_CUDA(h2d(tmp.p, flat.data(), flat.size() * 4));
    for (size_t i = 0; i < lists.size(); ++i)
        BIVF_CUDA(cudaMemcpyAsync(reinterpret_cast<void*>(row_addr(lists[i], sel[i])),
                                  tmp.as<int32_t>() + i * MLB_, (size_t)MLB_ * 4,
                                  cudaMemcpyDeviceToDevice, data_stream_));
    BIVF_CUDA(cudaStreamSynchronize(data_stream_));
}

// Row capacity >= need (<= MLB_cap_): a new double-buffered row array filled
// from the host mirror, every list republished on copy 0; searches that
// snapshotted the old array keep reading it (retired, never written again).
void GpuIndex::grow_rows(uint32_t need) {
    need = std::min(need, MLB_cap_);
    if (need <= MLB_) return;
    const auto t_gr = TClock::now();
    struct Tr {
        TClock::time_point t;
        uint32_t from, to;
        ~Tr() {
            if (trace_threshold_us() > 0) trace("grow_rows", us_since(t), "MLB " + std::to_string(from) + " -> " + std::to_string(to));
        }
    } tr{t_gr, MLB_, std::min(MLB_cap_, std::max(need, 2 * MLB_))};
    const uint32_t nm = std::min(MLB_cap_, std::max(need, 2 * MLB_));
    auto nb = std::make_unique<DevBuf>();
    nb->alloc((size_t)2 * C_ * nm * 4);
    std::vector<int32_t> flat((size_t)C_ * nm, -1);
    for (uint32_t c = 0; c < C_; ++c)
        std::copy(h_blocks_[c].begin(), h_blocks_[c].end(), flat.begin() + (size_t)c * nm);
    BIVF_CUDA(h2d(nb->p, flat.data(), flat.size() * 4));
    BIVF_CUDA(dset(static_cast<int32_t*>(nb->p) + (size_t)C_ * nm, 0xff, (size_t)C_ * nm * 4));
    auto old = std::make_unique<DevBuf>();
    std::swap(old->p, d_rows_.p);
    std::swap(old->bytes, d_rows_.bytes);
    std::swap(d_rows_.p, nb->p);
    std::swap(d_rows_.bytes, nb->bytes);
    retired_.push_back(std::move(old));
    MLB_ = nm;
    std::vector<ListPub> pubs;
    pubs.reserve(C_);
    for (uint32_t c = 0; c < C_; ++c) {
        h_sel_[c] = 0;
        pubs.push_back(current_pub(c));
    }
    publish(pubs);
    BIVF_CUDA(cudaStreamSynchronize(data_stream_));
}

// Whole-block copies src[i] -> dst[i] of every per-block array (payload, ids,
// scan mirror planes, norms, row copy).
void GpuIndex::copy_block_set(const std::vector<int32_t>& src, const std::vector<int32_t>& dst) {
    const uint32_t n = (uint32_t)src.size();
    if (!n) return;
    DevBuf &ds = s_rr_src_, &dd = s_rr_dst_;
    ds.ensure((size_t)n * 4);
    dd.ensure((size_t)n * 4);
    BIVF_CUDA(cudaMemcpyAsync(ds.p, src.data(), (size_t)n * 4, cudaMemcpyHostToDevice, data_stream_));
    BIVF_CUDA(cudaMemcpyAsync(dd.p, dst.data(), (size_t)n * 4, cudaMemcpyHostToDevice, data_stream_));
    cudaStream_t st = data_stream_;
    BIVF_CUDA(launch_copy_blocks(d_arena_.p, PS_ * 4, ds.as<int32_t>(), dd.as<int32_t>(), n, st));
    BIVF_CUDA(launch_copy_blocks(d_bids_.p, (uint64_t)T_ * 8, ds.as<int32_t>(), dd.as<int32_t>(), n, st));
    if (mir_on_) {
        BIVF_CUDA(launch_copy_blocks(d_arena_mir_.p, MPS_ * 4, ds.as<int32_t>(), dd.as<int32_t>(), n, st));
        BIVF_CUDA(launch_copy_blocks(d_arena_nrm_.p, (uint64_t)gpb_ * kNormFloats * 4, ds.as<int32_t>(),
                                     dd.as<int32_t>(), n, st));
        if (d_arena_rows_.p)
            BIVF_CUDA(launch_copy_blocks(d_arena_rows_.p, PS_ * 4, ds.as<int32_t>(), dd.as<int32_t>(), n, st));
    }
    BIVF_CUDA(cudaStreamSynchronize(st));  // the pageable src/dst vectors
}

uint64_t GpuIndex::off_alloc(uint64_t slots) {
    // best fit: a delete's new segment version usually takes a hole left by an
    // earlier version of similar size, so holes are not whittled into slivers
    // (first fit fragmented the free space until most copy-on-write deletes fell
    // back to the quiescent path under a sustained delete stream)
    slots = std::max<uint64_t>(32, (slots + 31) / 32 * 32);
    auto best = off_free_.end();
    for (auto it = off_free_.begin(); it != off_free_.end(); ++it)
        if (it->second >= slots && (best == off_free_.end() || it->second < best->second)) {
            best = it;
            if (it->second == slots) break;
        }
    if (best == off_free_.end()) return ~0ull;
    const uint64_t st = best->first, len = best->second;
    off_free_.erase(best);
    if (len > slots) off_free_[st + slots] = len - slots;
    return st;
}

void GpuIndex::off_free_add(uint64_t start, uint64_t slots) {
    if (!slots) return;
    auto it = off_free_.emplace(start, slots).first;
    auto nx = std::next(it);
    if (nx != off_free_.end() && it->first + it->second == nx->first) {
        it->second += nx->second;
        off_free_.erase(nx);
    }
    if (it != off_free_.begin()) {
        auto pv = std::prev(it);
        if (pv->first + pv->second == it->first) {
            pv->second += it->second;
            off_free_.erase(it);
        }
    }
}

uint32_t GpuIndex::off_owner(uint64_t slot) const {
    auto it = off_region_.upper_bound(slot);
    if (it == off_region_.begin()) throw Error(BIVF_ECORRUPT, "delete: offline slot outside every segment");
    --it;
    if (slot >= it->first + it->second.second)
        throw Error(BIVF_ECORRUPT, "delete: offline slot outside every segment");
    return it->second.first;
}

// ========================================================================
// delete (extension)
// ========================================================================

uint64_t GpuIndex::remove(const int64_t* ids, uint64_t n, uint8_t* found) {
    if (found)
        for (uint64_t i = 0; i < n; ++i) found[i] = 0;
    if (n == 0) return 0;
    const auto t_in = TClock::now();
    std::lock_guard<std::mutex> lk(data_mu_);
    struct Tr {
        TClock::time_point t;
        double lock;
        uint64_t n;
        ~Tr() {
            if (trace_threshold_us() > 0)
                trace("remove", us_since(t), "n=" + std::to_string(n) + " data_mu=" + std::to_string((int)lock));
        }
    } tr{t_in, us_since(t_in), n};
    BIVF_CUDA(cudaSetDevice(device_));
    cudaStream_t st = data_stream_;
    reclaim();  // retired offline regions: ids cleared before the locate below
    // request hash (first occurrence of each id)
    uint32_t hcap = 64;
    while (hcap < 2 * n) hcap <<= 1;
    std::vector<long long> hk(hcap, -1);
    std::vector<uint32_t> hv(hcap, 0);
    auto mix = [](uint64_t x) {
        x ^= x >> 33;
        x *= 0xff51afd7ed558ccdULL;
        x ^= x >> 33;
        x *= 0xc4ceb9fe1a85ec53ULL;
        x ^= x >> 33;
        return x;
    };
    for (uint64_t r = 0; r < n; ++r) {
        if (ids[r] < 0) continue;
        uint32_t h = (uint32_t)mix((uint64_t)ids[r]) & (hcap - 1);
        while (hk[h] >= 0 && hk[h] != ids[r]) h = (h + 1) & (hcap - 1);
        if (hk[h] < 0) {
            hk[h] = ids[r];
            hv[h] = (uint32_t)r;
        }
    }
    DevBuf &dk = s_rm_[0], &dv = s_rm_[1], &dloc = s_rm_[2];
    dk.ensure(hcap * 8);
    dv.ensure(hcap * 4);
    dloc.ensure(n * 8);
    BIVF_CUDA(cudaMemcpyAsync(dk.p, hk.data(), hcap * 8, cudaMemcpyHostToDevice, st));
    BIVF_CUDA(cudaMemcpyAsync(dv.p, hv.data(), hcap * 4, cudaMemcpyHostToDevice, st));
    BIVF_CUDA(cudaMemsetAsync(dloc.p, 0xff, n * 8, st));
    // every offline slot outside a live segment holds id -1 (bulk_load, grace)
    BIVF_CUDA(launch_locate(d_off_ids_.as<long long>(), off_slots_cap_, false, dk.as<long long>(),
                            dv.as<uint32_t>(), hcap - 1, dloc.as<uint64_t>(), st));
    BIVF_CUDA(launch_locate(d_bids_.as<long long>(), (uint64_t)h_cursor_ * T_, true,
                            dk.as<long long>(), dv.as<uint32_t>(), hcap - 1, dloc.as<uint64_t>(), st));
    std::vector<uint64_t> loc(n);
    BIVF_CUDA(cudaMemcpyAsync(loc.data(), dloc.p, n * 8, cudaMemcpyDeviceToHost, st));
    BIVF_CUDA(cudaStreamSynchronize(st));

    // Plan on the host, part by part, in request order: the hole takes the
    // part's last vector.  Part key: 2c (offline) or
    // 2c+1 (online); positions are offline slot index / list position `did`.
    struct Part {
        uint32_t count;                       // live count while planning
        std::unordered_map<uint64_t, uint64_t> content;  // pos -> original pos
        std::unordered_map<uint64_t, uint64_t> where;    // original pos -> current pos
    };
    std::map<uint64_t, Part> parts;  // ordered: deterministic scratch / region assignment
    auto part_of = [&](uint64_t a, uint64_t& key, uint64_t& pos) {
        if (a & kArenaBit) {
            const uint64_t g = a & ~kArenaBit;
            const uint32_t b = (uint32_t)(g / T_), slot = (uint32_t)(g % T_);
            const int32_t c = h_owner_[b];
            key = 2ull * (uint32_t)c + 1;
            pos = (uint64_t)h_mid_[b] * T_ + slot;
        } else {
            const uint32_t c = off_owner(a);
            key = 2ull * c;
            pos = a - h_off_start_[c];
        }
    };
    uint64_t removed = 0;
    std::vector<long long> gone;
    for (uint64_t r = 0; r < n; ++r) {
        if (loc[r] == ~0ull) continue;
        uint64_t key, pos0;
        part_of(loc[r], key, pos0);
        const uint32_t c = (uint32_t)(key / 2);
        auto ins = parts.try_emplace(key);
        Part& P = ins.first->second;
        if (ins.second) P.count = (key & 1) ? h_len_[c] : h_off_count_[c];
        // current position of this request's vector
        auto w = P.where.find(pos0);
        const uint64_t pos = w == P.where.end() ? pos0 : w->second;
        if (pos == ~0ull || pos >= P.count) continue;  // already gone
        const uint64_t last = P.count - 1;
        auto content_at = [&](uint64_t p) {
            auto it = P.content.find(p);
            return it == P.content.end() ? p : it->second;
        };
        const uint64_t moved_orig = content_at(last);
        const uint64_t gone_orig = content_at(pos);
        if (pos != last) {
            P.content[pos] = moved_orig;
            P.where[moved_orig] = pos;
        }
        P.content[last] = ~0ull;
        P.where[gone_orig] = ~0ull;
        P.count = (uint32_t)last;
        if (found) found[r] = 1;
        gone.push_back(ids[r]);
        ++removed;
    }
    if (removed == 0) return 0;
    // the seed samples drop the deleted ids before any list is republished: a
    // search that plans against the new versions never seeds with them
    if (samp_on_) {
        std::sort(gone.begin(), gone.end());
        DevBuf& dg = s_rm_[11];
        dg.ensure(gone.size() * 8);
        BIVF_CUDA(cudaMemcpyAsync(dg.p, gone.data(), gone.size() * 8, cudaMemcpyHostToDevice, st));
        BIVF_CUDA(launch_sample_invalidate(d_samp_ids_.as<long long>(), (uint64_t)C_ * kSampS, dg.as<long long>(),
                                           (uint32_t)gone.size(), st));
        BIVF_CUDA(cudaStreamSynchronize(st));  // the host copy of `gone` is a pageable source
    }
    // slot addresses (maint.cuh): payload float offset / id index, arena bit 63
    auto pay_at = [&](bool arena, uint64_t blk_or_start, uint64_t slot) -> uint64_t {
        if (arena)
            return kArenaBit | (blk_or_start * PS_ + (slot / 32) * 32 * D_ + slot % 32);
        const uint64_t s = blk_or_start + slot;
        return (s / 32) * 32 * D_ + s % 32;
    };
    auto id_at = [&](bool arena, uint64_t blk_or_start, uint64_t slot) -> uint64_t {
        return arena ? kArenaBit | (blk_or_start * T_ + slot) : blk_or_start + slot;
    };
    std::vector<uint64_t> msrc_p, mdst_p, msrc_i, mdst_i, clear, pa, ia;
    // stream-ordered on the data stream; the address vectors outlive the copies
    auto apply_moves = [&]() {
        const uint32_t nm = (uint32_t)msrc_p.size();
        pa = msrc_p;
        ia = msrc_i;
        pa.insert(pa.end(), mdst_p.begin(), mdst_p.end());
        ia.insert(ia.end(), mdst_i.begin(), mdst_i.end());
        DevBuf &dpa = s_rm_[3], &dia = s_rm_[4], &dscr_p = s_rm_[5], &dscr_i = s_rm_[6],
               &dclr = s_rm_[7];
        dpa.ensure(std::max<size_t>(pa.size(), 1) * 8);
        dia.ensure(std::max<size_t>(ia.size(), 1) * 8);
        dscr_p.ensure(std::max<size_t>((size_t)nm * (mir_on_ ? 2 * mirror_k(D_) + 2 + D_ : D_), 1) * 4);
        dscr_i.ensure(std::max<size_t>(nm, 1) * 8);
        dclr.ensure(std::max<size_t>(clear.size(), 1) * 8);
        if (!pa.empty()) {
            BIVF_CUDA(cudaMemcpyAsync(dpa.p, pa.data(), pa.size() * 8, cudaMemcpyHostToDevice, st));
            BIVF_CUDA(cudaMemcpyAsync(dia.p, ia.data(), ia.size() * 8, cudaMemcpyHostToDevice, st));
        }
        if (!clear.empty())
            BIVF_CUDA(cudaMemcpyAsync(dclr.p, clear.data(), clear.size() * 8, cudaMemcpyHostToDevice, st));
        BIVF_CUDA(launch_slot_moves(d_off_pay_.as<float>(), d_off_ids_.as<long long>(),
                                    d_arena_.as<float>(), d_bids_.as<long long>(), D_,
                                    dpa.as<uint64_t>(), dia.as<uint64_t>(), nm,
                                    dscr_p.as<float>(), dscr_i.as<long long>(), st));
        if (mir_on_)
            BIVF_CUDA(launch_mirror_slot_moves(mirror_, dia.as<uint64_t>(), nm, dscr_p.as<float>(), st));
        BIVF_CUDA(launch_clear_ids(d_off_ids_.as<long long>(), d_bids_.as<long long>(),
                                   dclr.as<uint64_t>(), (uint32_t)clear.size(), st));
    };

    // ---- read-copy-update: new versions beside the published ones
    uint32_t need_blocks = 0;
    for (auto& kv : parts) {
        if (!(kv.first & 1)) continue;
        std::set<uint64_t> mids;
        for (auto& pc : kv.second.content) mids.insert(pc.first / T_);
        need_blocks += (uint32_t)mids.size();
    }
    std::map<uint32_t, uint64_t> new_region;  // offline part -> new segment start
    bool cow = cow_on_ && !copy_backend_ && need_blocks <= NS_;
    if (cow) {
        for (auto& kv : parts) {
            if (kv.first & 1) continue;
            const uint32_t c = (uint32_t)(kv.first / 2);
            const uint64_t slots = (kv.second.count + 31ull) / 32 * 32;
            uint64_t r = 0;
            if (slots && (r = off_alloc(slots)) == ~0ull) {
                cow = false;
                break;
            }
            new_region[c] = slots ? r : ~0ull;
        }
        if (!cow)  // give back what was taken
            for (auto& nr : new_region)
                if (nr.second != ~0ull)
                    off_free_add(nr.second, (parts[2ull * nr.first].count + 31ull) / 32 * 32);
    }
    if (cow) {
        ++cow_ops_;
        std::map<uint32_t, ListPub> pubs;
        auto pub_of = [&](uint32_t c) -> ListPub& {
            auto it = pubs.find(c);
            if (it == pubs.end()) it = pubs.emplace(c, current_pub(c)).first;
            return it->second;
        };
        std::vector<int32_t> cp_src, cp_dst;                  // original block -> scratch
        std::vector<uint32_t> row_lists;
        std::vector<std::vector<int32_t>> rows1;
        std::vector<uint8_t> sel1;
        uint32_t next_sc = NB_;
        for (auto& kv : parts) {
            const uint32_t c = (uint32_t)(kv.first / 2);
            Part& P = kv.second;
            if (kv.first & 1) {
                // online: every logical block the plan writes gets a scratch copy
                std::map<uint32_t, int32_t> sc_of;
                for (auto& pc : P.content) {
                    const uint32_t m = (uint32_t)(pc.first / T_);
                    if (!sc_of.count(m)) {
                        sc_of[m] = (int32_t)next_sc++;
                        cp_src.push_back(h_blocks_[c][m]);
                        cp_dst.push_back(sc_of[m]);
                    }
                }
                for (auto& pc : P.content) {
                    const uint64_t pos = pc.first, orig = pc.second;
                    const int32_t sb = sc_of[(uint32_t)(pos / T_)];
                    if (pos >= P.count) {
                        clear.push_back(id_at(true, (uint64_t)sb, pos % T_));
                    } else if (orig != pos) {
                        const int32_t ob = h_blocks_[c][orig / T_];
                        msrc_p.push_back(pay_at(true, (uint64_t)ob, orig % T_));
                        msrc_i.push_back(id_at(true, (uint64_t)ob, orig % T_));
                        mdst_p.push_back(pay_at(true, (uint64_t)sb, pos % T_));
                        mdst_i.push_back(id_at(true, (uint64_t)sb, pos % T_));
                    }
                }
                std::vector<int32_t> r1 = h_blocks_[c];
                for (auto& so : sc_of) r1[so.first] = so.second;
                row_lists.push_back(c);
                rows1.push_back(std::move(r1));
                sel1.push_back((uint8_t)(1 - h_sel_[c]));
                ListPub& pb = pub_of(c);
                pb.row = row_addr(c, 1 - h_sel_[c]);
                pb.len = P.count;
            } else {
                // offline: the segment's new version in a free region (live groups copied,
                // then the tail-into-hole moves read from the old version)
                const uint64_t r = new_region[c], old = h_off_start_[c];
                const uint64_t groups = (P.count + 31ull) / 32;
                if (groups) {
                    auto cpy = [&](void* base, size_t per_slot_bytes) {
                        BIVF_CUDA(cudaMemcpyAsync(static_cast<char*>(base) + r * per_slot_bytes,
                                                  static_cast<char*>(base) + old * per_slot_bytes,
                                                  groups * 32 * per_slot_bytes, cudaMemcpyDeviceToDevice, st));
                    };
                    cpy(d_off_pay_.p, (size_t)D_ * 4);
                    cpy(d_off_ids_.p, 8);
                    if (mir_on_) {
                        BIVF_CUDA(cudaMemcpyAsync(d_off_mir_.as<float>() + (r / 32) * GF_,
                                                  d_off_mir_.as<float>() + (old / 32) * GF_,
                                                  groups * GF_ * 4, cudaMemcpyDeviceToDevice, st));
                        BIVF_CUDA(cudaMemcpyAsync(d_off_nrm_.as<float>() + (r / 32) * kNormFloats,
                                                  d_off_nrm_.as<float>() + (old / 32) * kNormFloats,
                                                  groups * kNormFloats * 4, cudaMemcpyDeviceToDevice, st));
                        if (d_off_rows_.p) cpy(d_off_rows_.p, (size_t)D_ * 4);
                    }
                }
                for (auto& pc : P.content) {
                    const uint64_t pos = pc.first, orig = pc.second;
                    if (pos >= P.count) {
                        if (pos < groups * 32) clear.push_back(id_at(false, r, pos));
                    } else if (orig != pos) {
                        msrc_p.push_back(pay_at(false, old, orig));
                        msrc_i.push_back(id_at(false, old, orig));
                        mdst_p.push_back(pay_at(false, r, pos));
                        mdst_i.push_back(id_at(false, r, pos));
                    }
                }
                ListPub& pb = pub_of(c);
                pb.start = groups ? r : 0;
                pb.count = P.count;
            }
        }
        copy_block_set(cp_src, cp_dst);
        apply_moves();
        write_rows(row_lists, rows1, sel1);
        std::vector<ListPub> pv;
        for (auto& kv : pubs) pv.push_back(kv.second);
        publish(pv);
        // host mirror follows the published state; retired offline regions wait for a grace
        for (auto& kv : pubs) {
            const uint32_t c = kv.first;
            const ListPub& pb = kv.second;
            if (new_region.count(c)) {
                auto it = off_region_.find(h_off_start_[c]);
                if (h_off_count_[c] > 0 && it != off_region_.end() && it->second.first == c) {
                    off_pending_.emplace_back(it->first, it->second.second);
                    off_region_.erase(it);
                }
                if (pb.count > 0) off_region_[pb.start] = {c, (pb.count + 31ull) / 32 * 32};
                h_off_start_[c] = pb.start;
                h_off_count_[c] = pb.count;
            }
            h_len_[c] = pb.len;
        }
        for (size_t i = 0; i < row_lists.size(); ++i) h_sel_[row_lists[i]] = sel1[i];
        grace();
        // online: the new versions back into the reference's block positions
        if (!cp_src.empty()) {
            copy_block_set(cp_dst, cp_src);
            std::vector<std::vector<int32_t>> rows2;
            std::vector<uint8_t> sel2;
            std::vector<ListPub> pv2;
            for (uint32_t c : row_lists) {
                rows2.push_back(h_blocks_[c]);
                sel2.push_back((uint8_t)(1 - h_sel_[c]));
            }
            write_rows(row_lists, rows2, sel2);
            for (size_t i = 0; i < row_lists.size(); ++i) {
                h_sel_[row_lists[i]] = sel2[i];
                pv2.push_back(current_pub(row_lists[i]));
            }
            publish(pv2);
            BIVF_CUDA(cudaStreamSynchronize(st));
        }
        grace_pending_ = true;
        refresh_size();
        return removed;
    }

    // ---- quiescent fallback: compaction in place, searches fenced
    ++quiescent_ops_;
    if (trace_threshold_us() > 0)
        trace("remove_quiescent", 0.0 + trace_threshold_us(), "no copy-on-write space: need_blocks=" + std::to_string(need_blocks));
    std::vector<uint32_t> len_idx, len_val, off_idx, off_val;
    for (auto& kv : parts) {
        const uint64_t key = kv.first;
        Part& P = kv.second;
        const uint32_t c = (uint32_t)(key / 2);
        const bool arena = key & 1;
        for (auto& pc : P.content) {
            const uint64_t pos = pc.first, orig = pc.second;
            auto loc_of = [&](uint64_t q, uint64_t& base, uint64_t& slot) {
                if (arena) {
                    base = (uint64_t)h_blocks_[c][q / T_];
                    slot = q % T_;
                } else {
                    base = h_off_start_[c];
                    slot = q;
                }
            };
            uint64_t b1, s1;
            loc_of(pos, b1, s1);
            if (pos >= P.count) {
                clear.push_back(id_at(arena, b1, s1));
            } else if (orig != pos) {
                uint64_t b0, s0;
                loc_of(orig, b0, s0);
                msrc_p.push_back(pay_at(arena, b0, s0));
                msrc_i.push_back(id_at(arena, b0, s0));
                mdst_p.push_back(pay_at(arena, b1, s1));
                mdst_i.push_back(id_at(arena, b1, s1));
            }
        }
        if (arena) {
            len_idx.push_back(c);
            len_val.push_back(P.count);
        } else {
            off_idx.push_back(c);
            off_val.push_back(P.count);
        }
    }
    DevBuf &dli = s_rm_[8], &dlv = s_rm_[9], &doi = s_rm_[10], &dov = s_rm_[11];
    dli.ensure(std::max<size_t>(len_idx.size(), 1) * 4);
    dlv.ensure(std::max<size_t>(len_idx.size(), 1) * 4);
    doi.ensure(std::max<size_t>(off_idx.size(), 1) * 4);
    dov.ensure(std::max<size_t>(off_idx.size(), 1) * 4);
    if (!len_idx.empty()) {
        BIVF_CUDA(cudaMemcpyAsync(dli.p, len_idx.data(), len_idx.size() * 4, cudaMemcpyHostToDevice, st));
        BIVF_CUDA(cudaMemcpyAsync(dlv.p, len_val.data(), len_val.size() * 4, cudaMemcpyHostToDevice, st));
    }
    if (!off_idx.empty()) {
        BIVF_CUDA(cudaMemcpyAsync(doi.p, off_idx.data(), off_idx.size() * 4, cudaMemcpyHostToDevice, st));
        BIVF_CUDA(cudaMemcpyAsync(dov.p, off_val.data(), off_val.size() * 4, cudaMemcpyHostToDevice, st));
    }
    {
        std::unique_lock<std::shared_mutex> g(gate_);
        begin_maintenance();
        apply_moves();
        BIVF_CUDA(launch_set_u32(d_len_.as<uint32_t>(), dli.as<uint32_t>(), dlv.as<uint32_t>(),
                                 (uint32_t)len_idx.size(), st));
        BIVF_CUDA(launch_set_u32(d_off_count_.as<uint32_t>(), doi.as<uint32_t>(),
                                 dov.as<uint32_t>(), (uint32_t)off_idx.size(), st));
        end_maintenance();
    }
    BIVF_CUDA(cudaStreamSynchronize(st));
    for (size_t i = 0; i < len_idx.size(); ++i) h_len_[len_idx[i]] = len_val[i];
    for (size_t i = 0; i < off_idx.size(); ++i) h_off_count_[off_idx[i]] = off_val[i];
    refresh_size();
    return removed;
}

// ========================================================================
// rearrangement (Alg. 3, ivf_index.cpp:356-511) — planned on the header
// mirror, applied on device as one block permutation
// ========================================================================

bool GpuIndex::exceed(uint32_t c) const {
    if (c >= C_) throw Error(BIVF_ERANGE, "exceed: bad cluster");
    std::lock_guard<std::mutex> lk(data_mu_);
    // Eq. 3: sum of committed slots over the online list (= its length), strict
    return (uint64_t)h_len_[c] > cfg_.rearrange_threshold;
}

namespace {
// Planner state shared by rearrange / sweep: the mirror plus the content
// permutation accumulated by the swaps (content_at[x] = original block whose
// data now sits at physical x).
struct Planner {
    std::vector<int32_t>& prev;
    std::vector<int32_t>& next;
    std::vector<int32_t>& owner;
    std::vector<int32_t>& mid;
    std::vector<uint8_t>& merged;
    std::vector<int32_t>& head;
    std::vector<int32_t>& tail;
    std::vector<std::vector<int32_t>>& blocks;
    std::vector<int32_t> content_at;
    uint32_t allocated;
    uint32_t C;
    std::deque<uint32_t> work;
    std::vector<char> queued;
    uint64_t merges = 0;
    std::vector<char> list_touched;

    static int32_t remap(int32_t x, int32_t a, int32_t b) { return x == a ? b : (x == b ? a : x); }

    void enqueue(int32_t blk) {
        const int32_t o = owner[blk];
        if (o < 0) return;
        if (!queued[o]) {
            queued[o] = 1;
            work.push_back((uint32_t)o);
        }
    }
    // ivf_index.cpp:414-434 (split_runs_around)
    void split_runs_around(int32_t x) {
        if (merged[x]) {
            merged[x] = 0;
            enqueue(x);
        }
        const int32_t nx = next[x];
        if (nx >= 0 && merged[nx]) {
            merged[nx] = 0;
            enqueue(x);
        }
    }
    // ivf_index.cpp:370-412 (swap_blocks) (headers), data via content_at
    void swap_blocks(int32_t a, int32_t b) {
        if (a == b) return;
        const int32_t pa = prev[a], na = next[a], pb = prev[b], nb = next[b];
        const int32_t oa = owner[a], ob = owner[b];
        const int32_t ma = mid[a], mb = mid[b];
        std::swap(content_at[a], content_at[b]);
        prev[a] = remap(pb, a, b);
        next[a] = remap(nb, a, b);
        owner[a] = ob;
        mid[a] = mb;
        prev[b] = remap(pa, a, b);
        next[b] = remap(na, a, b);
        owner[b] = oa;
        mid[b] = ma;
        merged[a] = 0;
        merged[b] = 0;
        if (pa >= 0 && pa != a && pa != b) next[pa] = b;
        if (na >= 0 && na != a && na != b) prev[na] = b;
        if (pb >= 0 && pb != a && pb != b) next[pb] = a;
        if (nb >= 0 && nb != a && nb != b) prev[nb] = a;
        auto fix_list = [&](int32_t c) {
            if (head[c] == a || head[c] == b) head[c] = remap(head[c], a, b);
            if (tail[c] == a || tail[c] == b) tail[c] = remap(tail[c], a, b);
            list_touched[c] = 1;
        };
        if (oa >= 0) fix_list(oa);
        if (ob >= 0 && ob != oa) fix_list(ob);
        // the per-list block tables follow the content
        if (ob >= 0) blocks[ob][mb] = a;
        if (oa >= 0) blocks[oa][ma] = b;
    }
    // ivf_index.cpp:436-474 (rearrange_locked)
    void rearrange_list(uint32_t c) {
        int32_t u = head[c];
        if (u < 0) return;
        const uint64_t cap = 4ull * allocated + 64;
        for (uint64_t guard = 0; guard < cap; ++guard) {
            const int32_t v = next[u];
            if (v < 0) break;
            if (merged[v]) {
                u = v;
                continue;
            }
            const int32_t p = u + 1;
            if ((uint32_t)p >= allocated) {
                u = v;
                continue;
            }
            if (p == v) {
                merged[v] = 1;
                ++merges;
                u = v;
                continue;
            }
            split_runs_around(p);
            split_runs_around(v);
            swap_blocks(p, v);
            merged[p] = 1;
            ++merges;
            u = p;
        }
    }
    // ivf_index.cpp:476-505 (work queue bounded by 2C+8 rounds)
    void rearrange(uint32_t k) {
        work.clear();
        std::fill(queued.begin(), queued.end(), 0);
        work.push_back(k);
        queued[k] = 1;
        uint64_t rounds = 0;
        while (!work.empty() && rounds++ < 2ull * C + 8) {
            const uint32_t c = work.front();
            work.pop_front();
            queued[c] = 0;
            rearrange_list(c);
        }
    }
};
}  // namespace

uint64_t GpuIndex::hop_count(uint32_t c) const {
    if (c >= C_) throw Error(BIVF_ERANGE, "hop_count: bad cluster");
    std::lock_guard<std::mutex> lk(data_mu_);
    uint64_t hops = 0, visited = 0;
    for (int32_t b = h_head_[c]; b >= 0; b = h_next_[b]) {
        if (++visited > NB_) throw Error(BIVF_ECORRUPT, "hop_count: cycle detected");
        const int32_t nx = h_next_[b];
        if (nx >= 0 && !h_merged_[nx]) ++hops;
    }
    return hops;
}

void GpuIndex::rearrange(uint32_t c) {
    if (c >= C_) throw Error(BIVF_ERANGE, "rearrange: bad cluster");
    std::lock_guard<std::mutex> lk(data_mu_);
    rearrange_lists({c});
}

void GpuIndex::rearrange_sweep() {
    // ivf_index.cpp:507-511: every list above T'_m, in cluster order; planned one
    // after the other on the header mirror, the data moves applied once
    std::lock_guard<std::mutex> lk(data_mu_);
    std::vector<uint32_t> ex;
    for (uint32_t c = 0; c < C_; ++c)
        if ((uint64_t)h_len_[c] > cfg_.rearrange_threshold) ex.push_back(c);
    if (!ex.empty()) rearrange_lists(ex);
}

void GpuIndex::rearrange_lists(const std::vector<uint32_t>& lists) {
    BIVF_CUDA(cudaSetDevice(device_));
    const auto t_in = TClock::now();
    uint64_t moved = 0;
    struct Tr {
        TClock::time_point t;
        const std::vector<uint32_t>& l;
        uint64_t& moved;
        ~Tr() {
            if (trace_threshold_us() > 0)
                trace("rearrange", us_since(t),
                      "lists=" + std::to_string(l.size()) + " moved_blocks=" + std::to_string(moved));
        }
    } tr{t_in, lists, moved};
    auto hops_of = [&](uint32_t k) {
        uint64_t hops = 0, visited = 0;
        for (int32_t b = h_head_[k]; b >= 0; b = h_next_[b]) {
            if (++visited > NB_) throw Error(BIVF_ECORRUPT, "hop_count: cycle detected");
            const int32_t nx = h_next_[b];
            if (nx >= 0 && !h_merged_[nx]) ++hops;
        }
        return hops;
    };
    Planner P{h_prev_, h_next_, h_owner_, h_mid_, h_merged_, h_head_, h_tail_, h_blocks_};
    P.allocated = h_cursor_;
    P.C = C_;
    P.queued.assign(C_, 0);
    P.list_touched.assign(C_, 0);
    P.content_at.resize(h_cursor_);
    for (uint32_t b = 0; b < h_cursor_; ++b) P.content_at[b] = (int32_t)b;
    std::vector<RearrangeEvent> evs;
    for (uint32_t c : lists) {
        const auto t0 = std::chrono::steady_clock::now();
        RearrangeEvent ev{c, hops_of(c), 0, 0, 0.0};
        const uint64_t m0 = P.merges;
        P.rearrange(c);
        ev.hops_after = hops_of(c);
        ev.merges = P.merges - m0;
        ev.duration_us =
            std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        evs.push_back(ev);
    }
    // the accumulated content permutation, applied on device
    const auto t1 = std::chrono::steady_clock::now();
    std::vector<int32_t> src, dst;
    for (uint32_t x = 0; x < h_cursor_; ++x)
        if (P.content_at[x] != (int32_t)x) {
            src.push_back(P.content_at[x]);
            dst.push_back((int32_t)x);
        }
    moved = src.size();
    if (!src.empty()) {
        std::vector<uint32_t> touched;
        for (uint32_t k = 0; k < C_; ++k)
            if (P.list_touched[k]) touched.push_back(k);
        apply_block_moves(src, dst, touched);
    }
    // the data moves are part of every rearrangement they serve
    const double apply_us =
        std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t1).count();
    std::lock_guard<std::mutex> lk2(events_mu_);
    for (auto& ev : evs) {
        ev.duration_us += apply_us;
        events_.push_back(ev);
    }
}

// Block contents move src[i] -> dst[i] (a permutation of pool blocks), the
// touched lists' rows become h_blocks_ (already updated by the planner).
void GpuIndex::apply_block_moves(const std::vector<int32_t>& src, const std::vector<int32_t>& dst,
                                 const std::vector<uint32_t>& lists) {
    const uint32_t nm = (uint32_t)src.size();
    cudaStream_t st = data_stream_;
    if (cow_on_ && nm <= NS_) {
        ++cow_ops_;
        reclaim();
        // phase 1: the moving contents into scratch blocks; rows in final logical
        // order, a moved content read from its scratch copy
        std::vector<int32_t> sc(nm);
        std::unordered_map<int32_t, int32_t> sc_of_dst;
        for (uint32_t i = 0; i < nm; ++i) {
            sc[i] = (int32_t)(NB_ + i);
            sc_of_dst[dst[i]] = sc[i];
        }
        copy_block_set(src, sc);
        std::vector<std::vector<int32_t>> rows;
        std::vector<uint8_t> sel;
        for (uint32_t k : lists) {
            std::vector<int32_t> r = h_blocks_[k];
            for (auto& x : r) {
                auto it = sc_of_dst.find(x);
                if (it != sc_of_dst.end()) x = it->second;
            }
            rows.push_back(std::move(r));
            sel.push_back((uint8_t)(1 - h_sel_[k]));
        }
        write_rows(lists, rows, sel);
        std::vector<ListPub> pubs;
        for (size_t i = 0; i < lists.size(); ++i) {
            h_sel_[lists[i]] = sel[i];
            pubs.push_back(current_pub(lists[i]));
        }
        publish(pubs);
        grace();
        // phase 2: contents to their final (reference) blocks, rows to them
        copy_block_set(sc, dst);
        rows.clear();
        for (size_t i = 0; i < lists.size(); ++i) {
            rows.push_back(h_blocks_[lists[i]]);
            sel[i] = (uint8_t)(1 - h_sel_[lists[i]]);
        }
        write_rows(lists, rows, sel);
        pubs.clear();
        for (size_t i = 0; i < lists.size(); ++i) {
            h_sel_[lists[i]] = sel[i];
            pubs.push_back(current_pub(lists[i]));
        }
        publish(pubs);
        BIVF_CUDA(cudaMemcpyAsync(d_owner_.p, h_owner_.data(), (size_t)h_cursor_ * 4,
                                  cudaMemcpyHostToDevice, st));
        BIVF_CUDA(cudaStreamSynchronize(st));
        grace_pending_ = true;
        return;
    }
    // quiescent fallback: searches fenced, blocks permuted in place
    ++quiescent_ops_;
    DevBuf &ds = s_rr_src_, &dd = s_rr_dst_, &sp = s_rr_pay_, &si = s_rr_ids_;
    ds.ensure(nm * 4);
    dd.ensure(nm * 4);
    sp.ensure((size_t)nm * std::max<uint64_t>(PS_, mir_on_ ? MPS_ : 0) * 4);
    si.ensure((size_t)nm * T_ * 8);
    BIVF_CUDA(cudaMemcpyAsync(ds.p, src.data(), nm * 4, cudaMemcpyHostToDevice, st));
    BIVF_CUDA(cudaMemcpyAsync(dd.p, dst.data(), nm * 4, cudaMemcpyHostToDevice, st));
    std::vector<std::vector<int32_t>> rows;
    std::vector<uint8_t> sel;
    for (uint32_t k : lists) {
        rows.push_back(h_blocks_[k]);
        sel.push_back(h_sel_[k]);
    }
    {
        std::unique_lock<std::shared_mutex> g(gate_);
        begin_maintenance();
        BIVF_CUDA(launch_block_moves(d_arena_.as<float>(), d_bids_.as<long long>(), PS_, T_,
                                     ds.as<int32_t>(), dd.as<int32_t>(), nm, sp.as<float>(),
                                     si.as<long long>(), st));
        if (mir_on_) {
            BIVF_CUDA(launch_block_moves(d_arena_mir_.as<float>(), nullptr, MPS_, T_,
                                         ds.as<int32_t>(), dd.as<int32_t>(), nm, sp.as<float>(),
                                         nullptr, st));
            BIVF_CUDA(launch_block_moves(d_arena_nrm_.as<float>(), nullptr,
                                         (uint64_t)gpb_ * kNormFloats, T_, ds.as<int32_t>(),
                                         dd.as<int32_t>(), nm, sp.as<float>(), nullptr, st));
            if (d_arena_rows_.p)
                BIVF_CUDA(launch_block_moves(d_arena_rows_.as<float>(), nullptr, PS_, T_,
                                             ds.as<int32_t>(), dd.as<int32_t>(), nm, sp.as<float>(),
                                             nullptr, st));
        }
        // rows rewritten in place: no search runs until the maintenance event
        write_rows(lists, rows, sel);
        BIVF_CUDA(cudaMemcpyAsync(d_owner_.p, h_owner_.data(), (size_t)h_cursor_ * 4,
                                  cudaMemcpyHostToDevice, st));
        end_maintenance();
    }
    BIVF_CUDA(cudaStreamSynchronize(st));
}

// oldest `cap` events; the rest stay queued for the next call
uint64_t GpuIndex::seed_samples(int64_t* out, uint64_t cap) const {
    std::lock_guard<std::mutex> lk(data_mu_);
    if (!samp_on_) return 0;
    const uint64_t n = (uint64_t)C_ * kSampS;
    if (out && cap) {
        BIVF_CUDA(cudaSetDevice(device_));
        BIVF_CUDA(cudaMemcpy(out, d_samp_ids_.p, std::min(cap, n) * 8, cudaMemcpyDeviceToHost));
    }
    return n;
}

std::vector<RearrangeEvent> GpuIndex::take_events(size_t cap) {
    std::lock_guard<std::mutex> lk(events_mu_);
    std::vector<RearrangeEvent> out;
    if (cap >= events_.size()) {
        out.swap(events_);
    } else {
        out.assign(events_.begin(), events_.begin() + (std::ptrdiff_t)cap);
        events_.erase(events_.begin(), events_.begin() + (std::ptrdiff_t)cap);
    }
    return out;
}

// ========================================================================
// introspection
// ========================================================================

// lock-free (VectorIndex::size, an atomic load in the reference): the
// executor's lanes read it per request and must not wait for the data lane
uint64_t GpuIndex::size() const { return size_total_.load(std::memory_order_acquire); }

void GpuIndex::refresh_size() {  // caller holds data_mu_
    uint64_t t = 0;
    for (uint32_t c = 0; c < C_; ++c) t += (uint64_t)h_off_count_[c] + h_len_[c];
    size_total_.store(t, std::memory_order_release);
}

uint64_t GpuIndex::list_length(uint32_t c) const {
    if (c >= C_) throw Error(BIVF_ERANGE, "list_length: bad cluster");
    std::lock_guard<std::mutex> lk(data_mu_);
    return h_len_[c];
}

uint64_t GpuIndex::offline_count(uint32_t c) const {
    if (c >= C_) throw Error(BIVF_ERANGE, "offline_count: bad cluster");
    std::lock_guard<std::mutex> lk(data_mu_);
    return h_off_count_[c];
}

int32_t GpuIndex::online_head(uint32_t c) const {
    if (c >= C_) throw Error(BIVF_ERANGE, "online_head: bad cluster");
    std::lock_guard<std::mutex> lk(data_mu_);
    return h_head_[c];
}

uint64_t GpuIndex::allocated_blocks() const {
    std::lock_guard<std::mutex> lk(data_mu_);
    return h_cursor_;
}

void GpuIndex::check_block(int32_t b) const {
    if (b < 0 || (uint32_t)b >= h_cursor_)
        throw Error(BIVF_ERANGE, "block index " + std::to_string(b) + " not allocated");
}

uint32_t GpuIndex::committed_of(int32_t b) const {
    const int32_t c = h_owner_[b];
    if (c < 0) return 0;
    const int64_t v = (int64_t)h_len_[c] - (int64_t)h_mid_[b] * T_;
    return (uint32_t)std::max<int64_t>(0, std::min<int64_t>(T_, v));
}

void GpuIndex::block_header(int32_t b, int32_t* out5) const {
    std::lock_guard<std::mutex> lk(data_mu_);
    check_block(b);
    out5[0] = h_prev_[b];
    out5[1] = h_next_[b];
    out5[2] = (int32_t)committed_of(b);
    out5[3] = h_owner_[b];
    out5[4] = h_merged_[b];
}

void GpuIndex::block_ids(int32_t b, int64_t* out) const {
    std::lock_guard<std::mutex> lk(data_mu_);
    check_block(b);
    BIVF_CUDA(cudaSetDevice(device_));
    BIVF_CUDA(d2h(out, d_bids_.as<long long>() + (size_t)b * T_, (size_t)T_ * 8));
}

void GpuIndex::block_payload(int32_t b, float* out) const {
    std::lock_guard<std::mutex> lk(data_mu_);
    check_block(b);
    BIVF_CUDA(cudaSetDevice(device_));
    BIVF_CUDA(d2h(out, d_arena_.as<float>() + (size_t)b * PS_, (size_t)PS_ * 4));
}

uint64_t GpuIndex::cluster_contents(uint32_t c, int64_t* ids, float* vecs) const {
    if (c >= C_) throw Error(BIVF_ERANGE, "cluster_contents: bad cluster");
    std::lock_guard<std::mutex> lk(data_mu_);
    const uint64_t noff = h_off_count_[c], non = h_len_[c];
    if (!ids) return noff + non;
    BIVF_CUDA(cudaSetDevice(device_));
    uint64_t n = 0;
    if (noff) {
        const uint64_t groups = (noff + 31) / 32;
        std::vector<float> pay(groups * 32 * D_);
        std::vector<long long> oid(noff);
        const uint64_t s0 = h_off_start_[c];
        BIVF_CUDA(d2h(pay.data(), d_off_pay_.as<float>() + s0 * D_, pay.size() * 4));
        BIVF_CUDA(d2h(oid.data(), d_off_ids_.as<long long>() + s0, noff * 8));
        for (uint64_t i = 0; i < noff; ++i, ++n) {
            ids[n] = oid[i];
            const float* base = pay.data() + (i / 32) * 32 * D_ + i % 32;
            for (uint32_t d = 0; d < D_; ++d) vecs[n * D_ + d] = base[(size_t)d * 32];
        }
    }
    std::vector<float> pay(PS_);
    std::vector<long long> bid(T_);
    uint64_t left = non;
    for (int32_t b : h_blocks_[c]) {
        if (!left) break;
        const uint32_t m = (uint32_t)std::min<uint64_t>(T_, left);
        BIVF_CUDA(d2h(pay.data(), d_arena_.as<float>() + (size_t)b * PS_, PS_ * 4));
        BIVF_CUDA(d2h(bid.data(), d_bids_.as<long long>() + (size_t)b * T_, (size_t)T_ * 8));
        for (uint32_t s = 0; s < m; ++s, ++n) {
            ids[n] = bid[s];
            const float* base = pay.data() + (s / 32) * 32 * D_ + s % 32;
            for (uint32_t d = 0; d < D_; ++d) vecs[n * D_ + d] = base[(size_t)d * 32];
        }
        left -= m;
    }
    return n;
}

std::string GpuIndex::dump_pool() const {
    // block_store.cpp:188-201 line format
    std::lock_guard<std::mutex> lk(data_mu_);
    std::ostringstream os;
    std::vector<long long> all((size_t)h_cursor_ * T_);
    if (h_cursor_) {
        BIVF_CUDA(cudaSetDevice(device_));
        BIVF_CUDA(d2h(all.data(), d_bids_.p, all.size() * 8));
    }
    for (uint32_t b = 0; b < h_cursor_; ++b) {
        const uint32_t sz = committed_of((int32_t)b);
        os << b << " prev=" << h_prev_[b] << " next=" << h_next_[b] << " size=" << sz << " ids=";
        for (uint32_t s = 0; s < sz; ++s) {
            if (s) os << ',';
            os << all[(size_t)b * T_ + s];
        }
        os << '\n';
    }
    return os.str();
}

// ========================================================================
// BIVFSNAP v1 (ivf_index.cpp:513-619)
// ========================================================================

namespace {
constexpr char kMagic[8] = {'B', 'I', 'V', 'F', 'S', 'N', 'A', 'P'};
template <class T>
void put(std::ostream& os, const T& v) {
    os.write(reinterpret_cast<const char*>(&v), sizeof(v));
}
template <class T>
T get(std::istream& is) {
    T v{};
    is.read(reinterpret_cast<char*>(&v), sizeof(v));
    if (!is) throw Error(BIVF_EIO, "snapshot: truncated file");
    return v;
}
}  // namespace

void GpuIndex::save(const std::string& path) const {
    std::ofstream os(path, std::ios::binary | std::ios::trunc);
    if (!os) throw Error(BIVF_EIO, "snapshot: cannot open " + path + " for writing");
    os.write(kMagic, 8);
    put<uint32_t>(os, 1);
    put<uint64_t>(os, C_);
    put<uint64_t>(os, D_);
    put<uint64_t>(os, cfg_.nprobe_default);
    put<uint64_t>(os, cfg_.rearrange_threshold);
    put<uint64_t>(os, cfg_.kmeans_iters);
    put<uint64_t>(os, cfg_.kmeans_seed);
    put<uint64_t>(os, NB_);
    put<uint64_t>(os, T_);
    put<uint64_t>(os, 32);
    put<double>(os, cfg_.alert_watermark);
    put<int64_t>(os, next_id_);
    std::vector<float> cent((size_t)C_ * D_);
    get_centroids(cent.data());
    os.write(reinterpret_cast<const char*>(cent.data()), cent.size() * 4);
    // online lists flattened into the offline segments (ivf_index.cpp:554-563)
    std::vector<int64_t> ids;
    std::vector<float> vecs;
    for (uint32_t c = 0; c < C_; ++c) {
        const uint64_t n = cluster_contents(c, nullptr, nullptr);
        ids.resize(n);
        vecs.resize(n * D_);
        cluster_contents(c, ids.data(), vecs.data());
        put<uint64_t>(os, n);
        for (uint64_t i = 0; i < n; ++i) {
            put<int64_t>(os, ids[i]);
            os.write(reinterpret_cast<const char*>(vecs.data() + i * D_), (std::streamsize)D_ * 4);
        }
    }
    if (!os) throw Error(BIVF_EIO, "snapshot: write failed for " + path);
}

std::unique_ptr<GpuIndex> GpuIndex::load(const std::string& path, const bivf_config* ov, uint32_t shard,
                                         uint32_t nshards) {
    if (nshards == 0 || shard >= nshards) throw Error(BIVF_EINVAL, "load: shard out of [0, nshards)");
    std::ifstream is(path, std::ios::binary);
    if (!is) throw Error(BIVF_EIO, "snapshot: cannot open " + path);
    char magic[8];
    is.read(magic, 8);
    if (!is || std::memcmp(magic, kMagic, 8) != 0) throw Error(BIVF_EIO, "snapshot: bad magic in " + path);
    if (get<uint32_t>(is) != 1) throw Error(BIVF_EIO, "snapshot: unsupported version in " + path);
    bivf_config cfg{};
    if (ov) cfg = *ov;
    cfg.num_clusters = get<uint64_t>(is);
    cfg.dim = get<uint64_t>(is);
    cfg.nprobe_default = get<uint64_t>(is);
    cfg.rearrange_threshold = get<uint64_t>(is);
    cfg.kmeans_iters = get<uint64_t>(is);
    cfg.kmeans_seed = get<uint64_t>(is);
    cfg.kmeans_seed_set = 1;
    cfg.num_blocks = get<uint64_t>(is);
    cfg.block_capacity = get<uint64_t>(is);
    if (get<uint64_t>(is) != 32) throw Error(BIVF_EIO, "snapshot: interleave_group must be 32");
    cfg.alert_watermark = get<double>(is);
    const int64_t next_id = get<int64_t>(is);
    if (!ov || ov->max_list_blocks == 0) cfg.max_list_blocks = 0;
    auto idx = std::make_unique<GpuIndex>(cfg);
    std::vector<float> cent(cfg.num_clusters * cfg.dim);
    is.read(reinterpret_cast<char*>(cent.data()), (std::streamsize)cent.size() * 4);
    if (!is) throw Error(BIVF_EIO, "snapshot: truncated centroids in " + path);
    idx->set_centroids(cent.data());
    std::vector<float> rows;
    std::vector<int64_t> ids;
    std::vector<uint32_t> asg;
    const uint32_t D = (uint32_t)cfg.dim;
    for (uint64_t c = 0; c < cfg.num_clusters; ++c) {
        const uint64_t n = get<uint64_t>(is);
        const size_t r0 = ids.size();
        ids.resize(r0 + n);
        asg.resize(r0 + n, (uint32_t)c);
        rows.resize((r0 + n) * D);
        size_t kept = r0;
        for (uint64_t i = 0; i < n; ++i) {
            ids[kept] = get<int64_t>(is);
            is.read(reinterpret_cast<char*>(rows.data() + kept * D), (std::streamsize)D * 4);
            if (!is) throw Error(BIVF_EIO, "snapshot: truncated vectors in " + path);
            if (nshards == 1 || (uint64_t)ids[kept] % nshards == shard) ++kept;
        }
        ids.resize(kept);
        asg.resize(kept);
        rows.resize(kept * D);
    }
    idx->bulk_load(rows.data(), ids.size(), asg.data(), ids.data());
    // flattened contents carry every id ever handed out (ivf_index.cpp:615-617)
    idx->supplied_.clear();
    idx->next_id_ = next_id;
    idx->offline_end_ = next_id;
    return idx;
}

}  // namespace bivf
