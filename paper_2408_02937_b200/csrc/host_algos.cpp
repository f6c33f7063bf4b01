// Host-side algorithms either side of the hot path:
//   synthetic_dataset  — restated from dataset.cpp:92-112 (same engine and
//                        libstdc++ distributions -> identical bits on this image)
//   kmeans_gpu         — kmeans.cpp:31-142 with every O(n*k*D) sweep on the GPU
//                        (k-means++ distance folds, Lloyd assignments via the
//                        exact quantizer kernel); the O(n*D) double-precision
//                        updates and the RNG-driven picks stay on the host in
//                        the reference's order, so centroids/assignments are
//                        bit-identical to the reference for the same seed.
// Compiled with -ffp-contract=off: host_l2 must round like distance.hpp.
#include <algorithm>
#include <cstring>
#include <limits>
#include <random>
#include <vector>

#include "index.h"
#include "insert.cuh"
#include "scan.cuh"

namespace bivf {

float host_l2(const float* a, const float* b, uint32_t dim) {
    float acc = 0.0f;
    for (uint32_t d = 0; d < dim; ++d) {
        const float t = a[d] - b[d];
        acc += t * t;
    }
    return acc;
}

void synthetic_dataset(uint64_t n, uint64_t dim, uint64_t comps, uint64_t seed, float* out) {
    if (dim == 0 || comps == 0) throw Error(BIVF_EINVAL, "synthetic_dataset: bad shape");
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<float> center_dist(0.0f, 100.0f);
    std::normal_distribution<float> noise_dist(0.0f, 3.0f);
    std::vector<float> centers(comps * dim);
    for (auto& v : centers) v = center_dist(rng);
    std::uniform_int_distribution<std::size_t> comp_dist(0, comps - 1);
    for (uint64_t i = 0; i < n; ++i) {
        const std::size_t c = comp_dist(rng);
        const float* ctr = centers.data() + c * dim;
        float* row = out + i * dim;
        for (uint64_t d = 0; d < dim; ++d) row[d] = ctr[d] + noise_dist(rng);
    }
}

namespace {

// kmeans.cpp:17-27: prefix walk over the weights with one uniform draw.
std::size_t weighted_pick(const std::vector<double>& w, double total, std::mt19937_64& rng) {
    std::uniform_real_distribution<double> u(0.0, total);
    const double r = u(rng);
    double acc = 0.0;
    for (std::size_t i = 0; i < w.size(); ++i) {
        acc += w[i];
        if (r <= acc) return i;
    }
    return w.size() - 1;
}

}  // namespace

uint64_t kmeans_gpu(const float* points, uint64_t n, uint64_t dim, uint64_t k, uint64_t iters,
                    uint64_t seed, int device, float* centroids, uint32_t* assignment) {
    if (k < 1) throw Error(BIVF_EINVAL, "kmeans: k must be >= 1");
    if (n < k) throw Error(BIVF_EINVAL, "kmeans: need at least k points");
    if (n > 0xffffffffull || k > 0xffffffffull) throw Error(BIVF_EINVAL, "kmeans: too large");
    BIVF_CUDA(cudaSetDevice(device));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const uint32_t N = (uint32_t)n, K = (uint32_t)k, D = (uint32_t)dim, Dp = pad4(D);
    cudaStream_t st;
    BIVF_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct SG {
        cudaStream_t s;
        ~SG() { cudaStreamDestroy(s); }
    } sg{st};

    DevBuf d_raw, d_pts_il, d_pts_q, d_cent, d_cent_il, d_min, d_cd, d_ci, d_od, d_oi, d_ctr;
    d_raw.alloc((size_t)n * D * 4);
    d_pts_il.alloc((size_t)((n + 31) / 32) * 32 * D * 4);
    d_pts_q.alloc((size_t)n * Dp * 4);
    d_cent.alloc((size_t)k * D * 4);
    d_cent_il.alloc((size_t)((k + 31) / 32) * 32 * D * 4);
    d_min.alloc((size_t)n * 8);
    d_ctr.alloc(16);
    BIVF_CUDA(cudaMemcpyAsync(d_raw.p, points, (size_t)n * D * 4, cudaMemcpyHostToDevice, st));
    BIVF_CUDA(launch_interleave(d_raw.as<float>(), N, D, d_pts_il.as<float>(), st));
    BIVF_CUDA(launch_pad_rows(d_raw.as<float>(), N, D, Dp, d_pts_q.as<float>(), st));

    std::mt19937_64 rng(seed);
    std::vector<float> cent((size_t)k * D, 0.0f);
    std::vector<uint32_t> asg(n, 0);
    PinBuf pin;
    pin.ensure((size_t)n * 8);
    double* hmin = pin.as<double>();
    std::vector<double> min_d2(n);

    // ---- k-means++ seeding (kmeans.cpp:42-70)
    {
        std::uniform_int_distribution<std::size_t> first(0, n - 1);
        const std::size_t c0 = first(rng);
        std::memcpy(cent.data(), points + c0 * D, D * 4);
        double total = 0.0;
        for (uint64_t c = 0; c < k; ++c) {
            if (c > 0) {
                std::size_t pick;
                if (total <= 0.0) {
                    std::uniform_int_distribution<std::size_t> any(0, n - 1);
                    pick = any(rng);
                } else {
                    pick = weighted_pick(min_d2, total, rng);
                }
                std::memcpy(cent.data() + c * D, points + pick * D, D * 4);
            }
            BIVF_CUDA(cudaMemcpyAsync(d_cent.as<float>() + c * D, cent.data() + c * D, D * 4,
                                      cudaMemcpyHostToDevice, st));
            BIVF_CUDA(launch_seed_update(d_pts_il.as<float>(), N, D, d_cent.as<float>() + c * D,
                                         d_min.as<double>(), c == 0 ? 1 : 0, st));
            BIVF_CUDA(cudaMemcpyAsync(hmin, d_min.p, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
            BIVF_CUDA(cudaStreamSynchronize(st));
            std::memcpy(min_d2.data(), hmin, (size_t)n * 8);
            total = 0.0;
            for (uint64_t i = 0; i < n; ++i) total += min_d2[i];
        }
    }

    // ---- Lloyd (kmeans.cpp:72-140)
    const uint32_t qt = qt_for(1, D);
    const uint64_t tiles = (n + qt - 1) / qt;
    const uint32_t ng = (K + 31) / 32;
    const uint32_t fnch = (uint32_t)std::min<uint64_t>(
        ng, std::max<uint64_t>(1, ((uint64_t)sms * 8 + tiles - 1) / tiles));
    d_cd.alloc((size_t)n * fnch * 4);
    d_ci.alloc((size_t)n * fnch * 8);
    d_od.alloc((size_t)n * 4);
    d_oi.alloc((size_t)n * 8);
    std::vector<long long> nearest(n);
    std::vector<double> sums((size_t)k * D);
    std::vector<std::size_t> counts(k);
    std::vector<uint32_t> prev(n, std::numeric_limits<uint32_t>::max());
    uint64_t iters_run = 0;
    for (uint64_t iter = 0; iter < iters; ++iter) {
        iters_run = iter + 1;
        BIVF_CUDA(cudaMemcpyAsync(d_cent.p, cent.data(), (size_t)k * D * 4, cudaMemcpyHostToDevice, st));
        BIVF_CUDA(launch_interleave(d_cent.as<float>(), K, D, d_cent_il.as<float>(), st));
        // nearest centroid, strict '<' = lowest index on ties (kmeans.cpp:79-90)
        BIVF_CUDA(launch_flat_topk(d_cent_il.as<float>(), K, D, d_pts_q.as<float>(), N, 1, BIVF_METRIC_L2, fnch,
                                   d_cd.as<float>(), d_ci.as<long long>(), d_od.as<float>(),
                                   d_oi.as<long long>(), nullptr, d_ctr.as<uint32_t>(), sms, st));
        BIVF_CUDA(cudaMemcpyAsync(nearest.data(), d_oi.p, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
        BIVF_CUDA(cudaStreamSynchronize(st));
        bool changed = false;
        for (uint64_t i = 0; i < n; ++i) {
            asg[i] = (uint32_t)nearest[i];
            if (asg[i] != prev[i]) changed = true;
        }
        if (!changed) break;
        prev = asg;
        std::fill(sums.begin(), sums.end(), 0.0);
        std::fill(counts.begin(), counts.end(), 0);
        for (uint64_t i = 0; i < n; ++i) {
            const uint32_t c = asg[i];
            const float* p = points + i * D;
            double* s = sums.data() + (size_t)c * D;
            for (uint32_t d = 0; d < D; ++d) s[d] += p[d];
            ++counts[c];
        }
        // empty-cluster repair (kmeans.cpp:106-131)
        for (uint64_t c = 0; c < k; ++c) {
            if (counts[c] != 0) continue;
            const std::size_t big = std::max_element(counts.begin(), counts.end()) - counts.begin();
            if (counts[big] <= 1) continue;
            float far_d = -1.0f;
            std::size_t far_i = 0;
            for (uint64_t i = 0; i < n; ++i) {
                if (asg[i] != big) continue;
                const float d2 = host_l2(points + i * D, cent.data() + big * D, D);
                if (d2 > far_d) {
                    far_d = d2;
                    far_i = i;
                }
            }
            const float* p = points + far_i * D;
            for (uint32_t d = 0; d < D; ++d) {
                sums[big * D + d] -= p[d];
                sums[c * D + d] += p[d];
            }
            --counts[big];
            ++counts[c];
            asg[far_i] = (uint32_t)c;
        }
        for (uint64_t c = 0; c < k; ++c) {
            if (counts[c] == 0) continue;
            float* ce = cent.data() + c * D;
            const double inv = 1.0 / static_cast<double>(counts[c]);
            for (uint32_t d = 0; d < D; ++d) ce[d] = static_cast<float>(sums[c * D + d] * inv);
        }
    }
    std::memcpy(centroids, cent.data(), (size_t)k * D * 4);
    std::memcpy(assignment, asg.data(), (size_t)n * 4);
    return iters_run;
}

// oracle.cpp:11-49 exact_knn on the GPU: the rows as ONE flat interleaved list
// scanned by the exact CUDA-core top-k kernel (sequential fp32 sums, (key, row)
// order), query batches of up to 64K.
void exact_knn_gpu(const float* base, uint64_t n, uint64_t dim, const float* q, uint64_t nq, uint64_t k,
                   int metric, int device, int64_t* ids, float* d, uint32_t* cnt) {
    if (dim == 0 || k == 0 || k > 256) throw Error(BIVF_EINVAL, "exact_knn: dim >= 1 and k in [1, 256]");
    if (metric != BIVF_METRIC_L2 && metric != BIVF_METRIC_IP) throw Error(BIVF_EINVAL, "exact_knn: bad metric");
    if (n > 0xffffffffull) throw Error(BIVF_EINVAL, "exact_knn: too many rows");
    if (nq == 0) return;
    const uint32_t D = (uint32_t)dim, Dp = pad4(D), N = (uint32_t)n, K = (uint32_t)k;
    if (N == 0) {
        for (uint64_t i = 0; i < nq * k; ++i) {
            ids[i] = -1;
            d[i] = 0.f;
        }
        if (cnt)
            for (uint64_t i = 0; i < nq; ++i) cnt[i] = 0;
        return;
    }
    BIVF_CUDA(cudaSetDevice(device));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaStream_t st;
    BIVF_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct SG {
        cudaStream_t s;
        ~SG() { cudaStreamDestroy(s); }
    } sg{st};
    DevBuf raw, il, dq, dqp, cd, ci, od, oi, oc, ctr;
    raw.alloc((size_t)N * D * 4);
    il.alloc((size_t)((N + 31) / 32) * 32 * D * 4);
    ctr.alloc(16);
    BIVF_CUDA(cudaMemcpyAsync(raw.p, base, (size_t)N * D * 4, cudaMemcpyHostToDevice, st));
    BIVF_CUDA(launch_interleave(raw.as<float>(), N, D, il.as<float>(), st));
    const uint64_t chunk = 65536;
    const uint32_t ng = (N + 31) / 32;
    for (uint64_t s = 0; s < nq; s += chunk) {
        const uint32_t m = (uint32_t)std::min<uint64_t>(chunk, nq - s);
        const uint32_t qt = qt_for(K, D);
        const uint64_t tiles = (m + qt - 1) / qt;
        const uint32_t nch = (uint32_t)std::min<uint64_t>(ng, std::max<uint64_t>(1, ((uint64_t)sms * 8 + tiles - 1) / tiles));
        dq.ensure((size_t)m * D * 4);
        dqp.ensure((size_t)m * Dp * 4);
        cd.ensure((size_t)m * nch * K * 4);
        ci.ensure((size_t)m * nch * K * 8);
        od.ensure((size_t)m * K * 4);
        oi.ensure((size_t)m * K * 8);
        oc.ensure((size_t)m * 4);
        BIVF_CUDA(cudaMemcpyAsync(dq.p, q + s * D, (size_t)m * D * 4, cudaMemcpyHostToDevice, st));
        BIVF_CUDA(launch_pad_rows(dq.as<float>(), m, D, Dp, dqp.as<float>(), st));
        BIVF_CUDA(launch_flat_topk(il.as<float>(), N, D, dqp.as<float>(), m, K, metric, nch, cd.as<float>(),
                                   ci.as<long long>(), od.as<float>(), oi.as<long long>(), oc.as<uint32_t>(),
                                   ctr.as<uint32_t>(), sms, st));
        BIVF_CUDA(cudaMemcpyAsync(d + s * k, od.p, (size_t)m * K * 4, cudaMemcpyDeviceToHost, st));
        BIVF_CUDA(cudaMemcpyAsync(ids + s * k, oi.p, (size_t)m * K * 8, cudaMemcpyDeviceToHost, st));
        if (cnt) BIVF_CUDA(cudaMemcpyAsync(cnt + s, oc.p, (size_t)m * 4, cudaMemcpyDeviceToHost, st));
        BIVF_CUDA(cudaStreamSynchronize(st));
    }
}

}  // namespace bivf
