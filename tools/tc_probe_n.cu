// Probe: tcgen05.mma kind::tf32, A (128 x K) in TMEM, B MN-major in smem made
// of G 32-column tiles (TMA SWIZZLE_128B_ATOM_32B, one per 32-vector group)
// placed `stride` bytes apart; N = 32*G with LBO = stride.  Checks the result
// exactly (small-integer operands) and times back-to-back MMA issue for each N.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_probe_n tools/tc_probe_n.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
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

__global__ void probe(const __grid_constant__ CUtensorMap mapB, const float* A, float* out, int K, int G,
                      int stride, int reps, long long* cycles) {
    extern __shared__ __align__(1024) unsigned char raw[];
    unsigned char* sm =
        reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar, mbar;
    __shared__ uint32_t tslot;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)) : "memory");
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
                     "r"(G * K * 128)
                     : "memory");
        for (int g = 0; g < G; ++g)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                "%3}], [%4];" ::"r"(smem_u32(sm + g * stride)),
                "l"(reinterpret_cast<uint64_t>(&mapB)), "r"(0), "r"(g * K), "r"(smem_u32(&bar))
                : "memory");
    }
    mbar_wait(&bar, 0);
    if (warp < 4) {  // A rows -> TMEM lanes, columns [0,K)
        const int m = 32 * warp + lane;
        for (int c0 = 0; c0 < K; c0 += 32) {
            uint32_t v[32];
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(A[m * K + c0 + i]);
            const uint32_t ta = tb + ((uint32_t)(32 * warp) << 16) + c0;
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
                "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
                "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
                "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
                "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
                : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t acc = tb + 256;
    if (warp == 0) {
        const uint32_t N = 32 * G;
        const uint32_t idesc =
            (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | ((N >> 3) << 17) | ((128u >> 4) << 24);
        const uint64_t b0 = desc(smem_u32(sm), stride, 512, 1);
        long long c0 = clock64();
        for (int r = 0; r < reps; ++r)
            for (int ks = 0; ks < K / 8; ++ks) {
                const uint32_t en = (r == 0 && ks == 0) ? 0u : (r == 0 ? 1u : 1u);
                const uint32_t e2 = (ks == 0) ? 0u : 1u;  // each rep recomputes D
                (void)en;
                asm volatile(
                    "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(acc),
                    "r"(tb + ks * 8), "l"(b0 + ks * 64ull), "r"(idesc), "r"(e2)
                    : "memory");
            }
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
                smem_u32(&mbar))
            : "memory");
        mbar_wait(&mbar, 0);
        long long c1 = clock64();
        if (lane == 0) *cycles = c1 - c0;
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp < 4) {
        for (int n0 = 0; n0 < 32 * G; n0 += 32) {
            uint32_t r[32];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                  "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                  "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                  "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                : "r"(acc + ((uint32_t)(32 * warp) << 16) + n0));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            const int m = 32 * warp + lane;
            for (int n = 0; n < 32; ++n) out[m * 256 + n0 + n] = __uint_as_float(r[n]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb) : "memory");
}

int main() {
    const int K = 128, GMAX = 8;
    std::vector<float> A(128 * K), B(GMAX * K * 32);  // B: tile g = rows [g*K, (g+1)*K) of 32 floats
    srand(7);
    for (auto& x : A) x = (float)(rand() % 17 - 8);
    for (auto& x : B) x = (float)(rand() % 17 - 8);
    float *dA, *dB, *dO;
    long long* dc;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dO, 128 * 256 * 4);
    cudaMalloc(&dc, 8);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
    CUtensorMap map;
    cuuint64_t dims[2] = {32, (cuuint64_t)(GMAX * K)};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {32, (cuuint32_t)K};
    cuuint32_t es[2] = {1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dB, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int G : {1, 2, 4, 8}) {
        for (int stride : {16384, 20480}) {
            if (G * stride > 190 * 1024) continue;
            const int reps = 100;
            probe<<<1, 128, 200 * 1024>>>(map, dA, dO, K, G, stride, reps, dc);
            cudaError_t e = cudaDeviceSynchronize();
            std::vector<float> O(128 * 256);
            long long cyc = 0;
            cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
            cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
            int bad = 0;
            for (int m = 0; m < 128; ++m)
                for (int n = 0; n < 32 * G; ++n) {
                    const int g = n / 32, c = n % 32;
                    double s = 0;
                    for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * B[(g * K + k) * 32 + c];
                    if (O[m * 256 + n] != (float)s) ++bad;
                }
            const double nmma = (double)reps * (K / 8);
            printf("G=%d N=%d stride=%d: %s, mismatches %d / %d, %.1f cycles per MMA (%.2f per 32 columns)\n", G,
                   32 * G, stride, cudaGetErrorString(e), bad, 128 * 32 * G, cyc / nmma, cyc / nmma / G);
        }
    }
    return 0;
}
