// Probe for the vector-major ("swapped") list-scan filter (scan_tc.cu scan_vm):
// A = 128 stored vectors (M) = four 32-slot groups of the scan mirror's bf16
// hi plane, each staged by one TMA box {32, K} (SWIZZLE_64B) into consecutive
// K*64-byte slots; MN-major, LBO = K*64 (next 32 vectors), SBO = 512.
// B = the query tile's residuals (N columns) as two bf16 planes (hi, lo)
// written by threads into the same MN-major SW64 layout (64-byte rows of 32
// queries, 16-byte chunk index XOR (row >> 1) & 3), LBO = K*64 (next 32
// queries).  kind::f16, bf16 in, fp32 accumulate, D = A * (B_hi + B_lo).
//   mode 0: exact small-integer check of both layouts (B_lo = 0)
//   mode 2: A_hi * (B_hi + B_lo) against fp64 (error / sum|ab|)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_probe_swap tools/tc_probe_swap.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

constexpr int K = 128, M = 128, NMAX = 64;
constexpr int kSlot = K * 64;  // one group's hi plane

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t ph) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
            smem_u32(bar)),
        "r"(ph)
        : "memory");
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;
    d |= (uint64_t)layout << 61;
    return d;
}
// byte offset of element (row k, column n) in an MN-major SW64 plane of 32-wide column blocks
__device__ __forceinline__ uint32_t sw64_off(uint32_t k, uint32_t n) {
    const uint32_t blk = n >> 5, nn = n & 31u;
    const uint32_t chunk = (nn >> 3) ^ ((k >> 1) & 3u);
    return blk * (uint32_t)kSlot + k * 64u + chunk * 16u + (nn & 7u) * 2u;
}

// gA: [4 groups][2K rows][32] bf16 (rows [0,K) = hi plane); Bq: [N][K] fp32 queries
__global__ void probe(const __grid_constant__ CUtensorMap mapA, const float* Bq, int N, float* out, int mode) {
    extern __shared__ __align__(1024) unsigned char raw[];
    unsigned char* sm =
        reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    unsigned char* sA = sm;                      // 4 * kSlot
    unsigned char* sBh = sm + 4 * kSlot;         // 2 * kSlot (64 queries)
    unsigned char* sBl = sBh + 2 * kSlot;
    __shared__ uint64_t bar, mbar;
    __shared__ uint32_t tslot;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    if (t == 0) {
        mbar_init(&bar, 1);
        mbar_init(&mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tb = tslot;
    if (t == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(4 * kSlot)
                     : "memory");
        for (int g = 0; g < 4; ++g)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                "%3}], [%4];" ::"r"(smem_u32(sA + g * kSlot)),
                "l"(reinterpret_cast<uint64_t>(&mapA)), "r"(0), "r"(g * 2 * K), "r"(smem_u32(&bar))
                : "memory");
    }
    // B planes: thread t writes column n = t / 2 (two threads per column, half the rows each)
    for (int idx = t; idx < NMAX * K; idx += blockDim.x) {
        const int n = idx / K, k = idx % K;
        float x = n < N ? Bq[n * K + k] : 0.f;
        const __nv_bfloat16 h = __float2bfloat16_rn(x);
        const __nv_bfloat16 l = __float2bfloat16_rn(x - __bfloat162float(h));
        *reinterpret_cast<__nv_bfloat16*>(sBh + sw64_off(k, n)) = h;
        *reinterpret_cast<__nv_bfloat16*>(sBl + sw64_off(k, n)) = mode == 0 ? __float2bfloat16_rn(0.f) : l;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy writes -> MMA (async proxy)
    __syncthreads();
    mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t acc = tb;
    if (t == 0) {
        const uint32_t Nr = (uint32_t)((N + 15) / 16 * 16);
        // D f32, A bf16, B bf16, A MN-major, B MN-major, N, M
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((Nr >> 3) << 17) |
                               (((uint32_t)M >> 4) << 24);
        const uint32_t a0 = smem_u32(sA), bh0 = smem_u32(sBh), bl0 = smem_u32(sBl);
        for (int ks = 0; ks < K / 16; ++ks) {
            const uint64_t ad = desc(a0 + ks * 1024, kSlot, 512, 4);
            const uint64_t bh = desc(bh0 + ks * 1024, kSlot, 512, 4);
            const uint64_t bl = desc(bl0 + ks * 1024, kSlot, 512, 4);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(acc),
                "l"(ad), "l"(bh), "r"(idesc), "r"(ks)
                : "memory");
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(acc),
                "l"(ad), "l"(bl), "r"(idesc)
                : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&mbar))
                     : "memory");
    }
    __syncwarp();
    mbar_wait(&mbar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp < 4) {
        for (int c0 = 0; c0 < NMAX; c0 += 32) {
            uint32_t r[32];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
                "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                  "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                  "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                  "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                : "r"(acc + c0 + ((uint32_t)(32 * warp) << 16)));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            const int m = 32 * warp + lane;
            for (int n = 0; n < 32; ++n) out[m * NMAX + c0 + n] = __uint_as_float(r[n]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb) : "memory");
}

static uint16_t bf16_bits(float x) {
    __nv_bfloat16 b = __float2bfloat16_rn(x);
    uint16_t u;
    memcpy(&u, &b, 2);
    return u;
}
static float bf16_val(uint16_t u) {
    uint32_t w = (uint32_t)u << 16;
    float f;
    memcpy(&f, &w, 4);
    return f;
}

int main() {
    std::vector<float> X(M * K), Q(NMAX * K);  // X[m][k] vectors, Q[n][k] queries
    float *dQ, *dO;
    uint16_t* dA;
    cudaMalloc(&dQ, Q.size() * 4);
    cudaMalloc(&dA, (size_t)4 * 2 * K * 32 * 2);
    cudaMalloc(&dO, M * NMAX * 4);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
    CUtensorMap map;
    cuuint64_t dims[2] = {32, (cuuint64_t)4 * 2 * K};
    cuuint64_t strides[1] = {64};
    cuuint32_t box[2] = {32, (cuuint32_t)K};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dA, dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("tensor map encode: %d\n", (int)cr);
    const int smem = 4 * kSlot + 4 * kSlot + 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    srand(7);
    int fails = 0;
    for (int mode : {0, 2}) {
        for (int N : {16, 32, 48, 64}) {
            for (auto& x : X)
                x = mode == 0 ? (float)(rand() % 17 - 8) : (float)((rand() / (double)RAND_MAX) * 600.0 - 300.0);
            for (auto& x : Q)
                x = mode == 0 ? (float)(rand() % 17 - 8) : (float)((rand() / (double)RAND_MAX) * 600.0 - 300.0);
            std::vector<uint16_t> gA((size_t)4 * 2 * K * 32, 0);
            for (int m = 0; m < M; ++m)
                for (int k = 0; k < K; ++k) gA[((size_t)(m / 32) * 2 * K + k) * 32 + m % 32] = bf16_bits(X[m * K + k]);
            cudaMemcpy(dQ, Q.data(), Q.size() * 4, cudaMemcpyHostToDevice);
            cudaMemcpy(dA, gA.data(), gA.size() * 2, cudaMemcpyHostToDevice);
            cudaMemset(dO, 0, M * NMAX * 4);
            probe<<<1, 128, smem>>>(map, dQ, N, dO, mode);
            cudaError_t e = cudaDeviceSynchronize();
            std::vector<float> O(M * NMAX);
            cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
            double worst = 0;
            int bad = 0;
            for (int m = 0; m < M; ++m)
                for (int n = 0; n < N; ++n) {
                    double s = 0, a = 0;
                    for (int k = 0; k < K; ++k) {
                        const double xv = mode == 0 ? X[m * K + k] : bf16_val(bf16_bits(X[m * K + k]));
                        s += xv * Q[n * K + k];
                        a += fabs((double)X[m * K + k] * Q[n * K + k]);
                    }
                    const double err = fabs(O[m * NMAX + n] - s);
                    if (mode == 0 && err != 0) ++bad;
                    if (err / a > worst) worst = err / a;
                }
            printf("mode %d N %d: %s bad=%d max|err|/sum|ab| = %.3g (2^%.1f)  O[0]=%.8g O[%d]=%.8g\n", mode, N,
                   cudaGetErrorString(e), bad, worst, log2(worst + 1e-300), O[0], 33 * NMAX + N - 1,
                   O[33 * NMAX + N - 1]);
            fails += (e != cudaSuccess) || bad;
        }
    }
    printf(fails ? "PROBE FAILED\n" : "PROBE OK\n");
    return fails;
}
