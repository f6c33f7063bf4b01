// Probe: A (128 x K fp32) in TMEM (tcgen05.st), B in smem (MN-major, TMA
// SWIZZLE_128B_ATOM_32B, layout BASE32B), 3xTF32 split (A_hi*B_hi + A_hi*B_lo +
// A_lo*B_hi, explicit truncation), kind::tf32 TS form.  Reports the max error
// relative to sum|a||b| for 1x and 3x.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_probe_ts tools/tc_probe_ts.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

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
__device__ __forceinline__ float trunc_tf32(float x) {
    return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
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

__global__ void probe(const __grid_constant__ CUtensorMap mapB, const float* A, float* out, int K, int mode) {
    extern __shared__ __align__(1024) unsigned char raw[];
    unsigned char* sm =
        reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    unsigned char* sB = sm;           // 16 KB (B, then B_hi in place)
    unsigned char* sBl = sm + 16384;  // 16 KB B_lo
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
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(K * 128)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
            "[%4];" ::"r"(smem_u32(sB)),
            "l"(reinterpret_cast<uint64_t>(&mapB)), "r"(0), "r"(0), "r"(smem_u32(&bar))
            : "memory");
    }
    mbar_wait(&bar, 0);
    for (int i = t; i < K * 32 && mode != 0; i += blockDim.x) {  // split B in place (offsets unchanged)
        float* p = reinterpret_cast<float*>(sB) + i;
        const float x = *p, h = trunc_tf32(x);
        *p = h;
        reinterpret_cast<float*>(sBl)[i] = x - h;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp < 4) {  // A rows -> TMEM lanes; columns [0,K) hi, [K,2K) lo
        const int m = 32 * warp + lane;
        for (int c0 = 0; c0 < K; c0 += 32) {
            uint32_t h[32], l[32];
            for (int i = 0; i < 32; ++i) {
                const float x = A[m * K + c0 + i], hh = mode == 0 ? x : trunc_tf32(x);
                h[i] = __float_as_uint(hh);
                l[i] = __float_as_uint(x - hh);
            }
            const uint32_t ta = tb + ((uint32_t)(32 * warp) << 16) + c0;
            ST32(ta, h);
            ST32(ta + K, l);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t acc = tb + 2 * K;
    if (t == 0) {
        const uint32_t idesc =
            (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
        int first = 1;
        for (int ks = 0; ks < K / 8; ++ks) {
            const uint64_t bh = desc(smem_u32(sB) + ks * 1024, 16384, 512, 1);
            const uint64_t bl = desc(smem_u32(sBl) + ks * 1024, 16384, 512, 1);
            const uint32_t ah = tb + ks * 8, al = tb + K + ks * 8;
            const int nterm = mode == 3 ? 3 : 1;
            for (int term = 0; term < nterm; ++term) {
                const uint32_t a = term == 2 ? al : ah;
                const uint64_t b = term == 1 ? bl : bh;
                const uint32_t en = first ? 0u : 1u;
                first = 0;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(acc),
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
        uint32_t r[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
            "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
              "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
              "=r"(r[30]), "=r"(r[31])
            : "r"(acc + ((uint32_t)(32 * warp) << 16)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int m = 32 * warp + lane;
        for (int n = 0; n < 32; ++n) out[m * 32 + n] = __uint_as_float(r[n]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb) : "memory");
}

int main() {
    const int K = 128;
    std::vector<float> A(128 * K), B(K * 32);
    srand(7);
    for (auto& x : A) x = (float)((rand() / (double)RAND_MAX) * 600.0 - 300.0);
    for (auto& x : B) x = (float)((rand() / (double)RAND_MAX) * 600.0 - 300.0);
    std::vector<double> ref(128 * 32), mag(128 * 32);
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 32; ++n) {
            double s = 0, a = 0;
            for (int k = 0; k < K; ++k) {
                s += (double)A[m * K + k] * B[k * 32 + n];
                a += fabs((double)A[m * K + k] * B[k * 32 + n]);
            }
            ref[m * 32 + n] = s;
            mag[m * 32 + n] = a;
        }
    float *dA, *dB, *dO;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dO, 128 * 32 * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
    CUtensorMap map;
    cuuint64_t dims[2] = {32, (cuuint64_t)K};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {32, (cuuint32_t)K};
    cuuint32_t es[2] = {1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dB, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
    {   // conversion rule: raw fp32 operands (no explicit truncation), A = 1, B = 1 + 2^-11 + 2^-20
        std::vector<float> A1(128 * K, 1.0f), B1(K * 32, 1.0f + ldexpf(1.f, -11) + ldexpf(1.f, -20));
        cudaMemcpy(dA, A1.data(), A1.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B1.data(), B1.size() * 4, cudaMemcpyHostToDevice);
        probe<<<1, 128, 40 * 1024>>>(map, dA, dO, K, 0);
        cudaDeviceSynchronize();
        float o = 0;
        cudaMemcpy(&o, dO, 4, cudaMemcpyDeviceToHost);
        printf("raw-fp32 conversion: K*B = %.9g  (truncate -> %.9g, round-nearest -> %.9g)\n", o, (double)K,
               K * (1.0 + ldexp(1.0, -10)));
        cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    }
    for (int mode : {1, 3}) {
        cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
        probe<<<1, 128, 40 * 1024>>>(map, dA, dO, K, mode);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> O(128 * 32);
        cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
        double worst = 0, worst_abs = 0;
        for (int i = 0; i < 128 * 32; ++i) {
            const double r = fabs(O[i] - ref[i]) / mag[i];
            if (r > worst) worst = r;
            if (fabs(O[i] - ref[i]) > worst_abs) worst_abs = fabs(O[i] - ref[i]);
        }
        printf("mode %dxTF32 (A in TMEM): err=%s  max |err|/sum|ab| = %.3g (= 2^%.1f)  max abs %.3g  O[0]=%.6g ref=%.6g\n",
               mode, cudaGetErrorString(e), worst, log2(worst + 1e-300), worst_abs, O[0], ref[0]);
    }
    return 0;
}
