// Layout probe for the tensor-core scan: one CTA stages a 32-vector group with
// TMA (SWIZZLE_128B) as the MN-major B operand, builds A (128 x K, K-major
// SW128) exactly like scan_tc.cu, runs tcgen05.mma.kind::tf32 into TMEM and
// checks the 128x32 dot products against the host (integer-valued inputs, so
// TF32 is exact).  Several descriptor variants are tried in one run.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_probe tools/tc_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
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

struct Variant {
    uint32_t a_lbo, a_sbo, b_lbo, b_sbo, b_major, b_step, b_layout, map;
};

__global__ void probe(const __grid_constant__ CUtensorMap mapB0, const __grid_constant__ CUtensorMap mapB1, const float* A, float* out, Variant v, int K) {
    const CUtensorMap* pm = v.map ? &mapB1 : &mapB0;
    extern __shared__ __align__(1024) unsigned char raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    unsigned char* sA = sm;               // 64 KB
    unsigned char* sB = sm + 65536;       // 16 KB
    __shared__ uint64_t bar, mbar;
    __shared__ uint32_t tslot;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    if (t == 0) {
        mbar_init(&bar, 1);
        mbar_init(&mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tslot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    // A: row m, K-block kb at kb*16KB + m*128, chunk (k%32)/4 ^ (m%8)
    for (int m = t; m < 128; m += blockDim.x)
        for (int k0 = 0; k0 < K; k0 += 4) {
            float4 r = make_float4(A[m * K + k0], A[m * K + k0 + 1], A[m * K + k0 + 2], A[m * K + k0 + 3]);
            const int kb = k0 >> 5, ch = (k0 & 31) >> 2;
            *reinterpret_cast<float4*>(sA + kb * 16384 + m * 128 + ((ch ^ (m & 7)) << 4)) = r;
        }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = tslot;
    if (t == 0) {
        mbar_arrive_expect_tx(&bar, K * 128);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                smem_u32(sB)),
            "l"(reinterpret_cast<uint64_t>(pm)), "r"(0), "r"(0), "r"(smem_u32(&bar)) : "memory");
        mbar_wait(&bar, 0);
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (v.b_major << 16) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
        for (int ks = 0; ks < K / 8; ++ks) {
            const uint32_t kb = ks >> 2, kin = ks & 3;
            const uint64_t ad = desc(smem_u32(sA) + kb * 16384 + kin * 32, v.a_lbo, v.a_sbo, 2);
            const uint64_t bd = desc(smem_u32(sB) + ks * v.b_step, v.b_lbo, v.b_sbo, v.b_layout);
            const uint32_t acc = ks > 0;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase),
                "l"(ad), "l"(bd), "r"(idesc), "r"(acc) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)) : "memory");
    }
    __syncwarp();
    mbar_wait(&mbar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp < 4) {
        uint32_t r[32];
        const uint32_t ta = tbase + ((uint32_t)(32 * warp) << 16);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
              "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
              "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
              "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int m = 32 * warp + lane;
        for (int n = 0; n < 32; ++n) out[m * 32 + n] = __uint_as_float(r[n]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tbase) : "memory");
}

int main() {
    const int K = 128;
    std::vector<float> A(128 * K), B(K * 32);  // B stored [k][n] (group layout rows)
    srand(1);
    for (auto& x : A) x = (float)(rand() % 7 - 3);
    for (auto& x : B) x = (float)(rand() % 7 - 3);
    std::vector<double> ref(128 * 32, 0);
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 32; ++n) {
            double s = 0;
            for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * B[k * 32 + n];
            ref[m * 32 + n] = s;
        }
    float *dA, *dB, *dO;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dO, 128 * 32 * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
    CUtensorMap map, map32;
    cuuint64_t dims[2] = {32, (cuuint64_t)K};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {32, (cuuint32_t)K};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dB, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult cr2 = enc(&map32, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dB, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d %d\n", (int)cr, (int)cr2);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    Variant vs[] = {
        {16, 1024, 4096, 1024, 1, 1024, 2, 0},   // SW128 (zeros last run)
        {16, 1024, 4096, 512, 1, 1024, 1, 1},    // 128B_BASE32B, TMA ATOM_32B, SBO 512
        {16, 1024, 512, 4096, 1, 1024, 1, 1},    // swapped
        {16, 1024, 16384, 512, 1, 1024, 1, 1},
        {16, 1024, 128, 512, 1, 1024, 1, 1},
        {16, 1024, 4096, 1024, 1, 1024, 1, 1},
        {16, 1024, 4096, 512, 1, 1024, 1, 0},    // BASE32B desc on plain SW128 data
    };
    for (int i = 0; i < (int)(sizeof(vs) / sizeof(vs[0])); ++i) {
        cudaMemset(dO, 0, 128 * 32 * 4);
        probe<<<1, 192, 100 * 1024>>>(map, map32, dA, dO, vs[i], K);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> O(128 * 32);
        cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        double maxe = 0;
        for (int j = 0; j < 128 * 32; ++j) {
            double d = fabs(O[j] - ref[j]);
            if (d > 1e-3) ++bad;
            if (d > maxe) maxe = d;
        }
        printf("variant %d (layout %u map %u aLBO %u aSBO %u bLBO %u bSBO %u bmaj %u): err=%s bad=%d maxerr=%g  O[0..3]=%g %g %g %g ref=%g %g %g %g\n",
               i, vs[i].b_layout, vs[i].map, vs[i].a_lbo, vs[i].a_sbo, vs[i].b_lbo, vs[i].b_sbo, vs[i].b_major, cudaGetErrorString(e), bad, maxe,
               O[0], O[1], O[2], O[3], ref[0], ref[1], ref[2], ref[3]);
        if (e != cudaSuccess) break;
    }
    return 0;
}
