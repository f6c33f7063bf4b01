// Probe for the bf16x3 scan filter: A (128 x K) bf16 pairs packed in TMEM
// (tcgen05.st, TS form), B = two 32-slot groups in two smem stages, each an
// MN-major bf16 plane pair (rows [0,K) hi, [K,2K) lo, 64-byte rows) staged by
// ONE TMA box {32, 2K} with SWIZZLE_64B, UMMA layout SW64, LBO = stage stride
// (N = 64 spans both stages), SBO = 512 B.  kind::f16 (bf16 in, fp32 accumulate).
//   mode 0: exact small-integer check of the layouts (A_hi*B_hi only)
//   mode 1: A_hi*B_hi;  mode 3: A_hi*B_hi + A_hi*B_lo + A_lo*B_hi (RN splits)
// Reports max |err| / sum|a b| against fp64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_probe_bf16 tools/tc_probe_bf16.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

constexpr int K = 128, M = 128, NG = 2, N = 32 * NG;
constexpr int kStage = 2 * K * 64;  // one group: 2K rows x 64 B

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

#define ST32(addr, v)                                                                                    \
    asm volatile(                                                                                        \
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),               \
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), \
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),     \
        "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),    \
        "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])                 \
        : "memory")

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
    return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(lo)) |
           ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(hi)) << 16);
}

// A: [M][K] fp32 row-major; gB: [NG groups][2K rows][32] bf16 (prepared on the host)
__global__ void probe(const __grid_constant__ CUtensorMap mapB, const float* A, float* out, int mode) {
    extern __shared__ __align__(1024) unsigned char raw[];
    unsigned char* sm =
        reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
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
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                     "r"(NG * kStage)
                     : "memory");
        for (int g = 0; g < NG; ++g)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                "%3}], [%4];" ::"r"(smem_u32(sm + g * kStage)),
                "l"(reinterpret_cast<uint64_t>(&mapB)), "r"(0), "r"(g * 2 * K), "r"(smem_u32(&bar))
                : "memory");
    }
    mbar_wait(&bar, 0);
    if (warp < 4) {  // A rows -> TMEM lanes; columns [0,K/2) hi pairs, [K/2,K) lo pairs
        const int m = 32 * warp + lane;
        for (int c0 = 0; c0 < K; c0 += 64) {
            uint32_t h[32], l[32];
            for (int i = 0; i < 32; ++i) {
                const float x0 = A[m * K + c0 + 2 * i], x1 = A[m * K + c0 + 2 * i + 1];
                const float h0 = __bfloat162float(__float2bfloat16_rn(x0));
                const float h1 = __bfloat162float(__float2bfloat16_rn(x1));
                h[i] = pack2(h0, h1);
                l[i] = pack2(x0 - h0, x1 - h1);
            }
            const uint32_t ta = tb + ((uint32_t)(32 * warp) << 16) + c0 / 2;
            ST32(ta, h);
            ST32(ta + K / 2, l);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t acc = tb + K;  // after A hi/lo (K/2 + K/2 columns)
    if (t == 0) {
        // D f32, A bf16, B bf16, A K-major, B MN-major, N, M
        const uint32_t idesc =
            (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | (((uint32_t)N >> 3) << 17) | (((uint32_t)M >> 4) << 24);
        int first = 1;
        const uint32_t s0 = smem_u32(sm);
        for (int ks = 0; ks < K / 16; ++ks) {
            const uint64_t bh = desc(s0 + ks * 1024, kStage, 512, 4);
            const uint64_t bl = desc(s0 + K * 64 + ks * 1024, kStage, 512, 4);
            const uint32_t ah = tb + ks * 8, al = tb + K / 2 + ks * 8;
            const int nterm = mode == 3 ? 3 : 1;
            for (int term = 0; term < nterm; ++term) {
                const uint32_t a = term == 2 ? al : ah;
                const uint64_t b = term == 1 ? bl : bh;
                const uint32_t en = first ? 0u : 1u;
                first = 0;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(acc),
                    "r"(a), "l"(b), "r"(idesc), "r"(en)
                    : "memory");
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&mbar))
                     : "memory");
    }
    __syncwarp();
    mbar_wait(&mbar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp < 4) {
        for (int c0 = 0; c0 < N; c0 += 32) {
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
            for (int n = 0; n < 32; ++n) out[m * N + c0 + n] = __uint_as_float(r[n]);
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
    std::vector<float> A(M * K), B(K * N);  // B[k][n], n = 32*g + slot
    float *dA, *dO;
    uint16_t* dB;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, (size_t)NG * 2 * K * 32 * 2);
    cudaMalloc(&dO, M * N * 4);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
    CUtensorMap map;
    cuuint64_t dims[2] = {32, (cuuint64_t)NG * 2 * K};
    cuuint64_t strides[1] = {64};
    cuuint32_t box[2] = {32, (cuuint32_t)(2 * K)};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dB, dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("tensor map encode: %d\n", (int)cr);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, NG * kStage + 1024);
    srand(7);
    for (int mode : {0, 1, 3}) {
        for (auto& x : A)
            x = mode == 0 ? (float)(rand() % 17 - 8) : (float)((rand() / (double)RAND_MAX) * 600.0 - 300.0);
        for (auto& x : B)
            x = mode == 0 ? (float)(rand() % 17 - 8) : (float)((rand() / (double)RAND_MAX) * 600.0 - 300.0);
        // host split of B into the mirror layout: group g rows [0,K) hi, [K,2K) lo
        std::vector<uint16_t> gB((size_t)NG * 2 * K * 32);
        std::vector<float> Bh(K * N), Bl(K * N);
        for (int k = 0; k < K; ++k)
            for (int n = 0; n < N; ++n) {
                const float x = B[k * N + n];
                const uint16_t h = bf16_bits(x);
                const float hv = bf16_val(h);
                const uint16_t l = bf16_bits(x - hv);
                Bh[k * N + n] = hv;
                Bl[k * N + n] = bf16_val(l);
                const int g = n / 32, s = n % 32;
                gB[((size_t)g * 2 * K + k) * 32 + s] = h;
                gB[((size_t)g * 2 * K + K + k) * 32 + s] = l;
            }
        cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, gB.data(), gB.size() * 2, cudaMemcpyHostToDevice);
        probe<<<1, 128, NG * kStage + 1024>>>(map, dA, dO, mode);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> O(M * N);
        cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
        double worst = 0, worst_abs = 0;
        int bad = 0;
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                double s = 0, a = 0;
                for (int k = 0; k < K; ++k) {
                    const double av = A[m * K + k], bv = B[k * N + n];
                    if (mode == 1) {
                        const double ah = bf16_val(bf16_bits(A[m * K + k]));
                        s += ah * Bh[k * N + n];
                    } else {
                        s += av * bv;
                    }
                    a += fabs(av * bv);
                }
                const double err = fabs(O[m * N + n] - s);
                if (mode == 0 && err != 0) ++bad;
                if (err / a > worst) worst = err / a;
                if (err > worst_abs) worst_abs = err;
            }
        printf("mode %d: %s  bad=%d  max|err|/sum|ab| = %.3g (2^%.1f)  max abs %.3g  O[0]=%.8g O[33]=%.8g\n", mode,
               cudaGetErrorString(e), bad, worst, log2(worst + 1e-300), worst_abs, O[0], O[33]);
    }
    return 0;
}
