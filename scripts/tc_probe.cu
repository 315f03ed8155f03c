// Standalone probe of the tcgen05 kind::tf32 mechanics used by k_dstream_tc:
//  - TMA 2-D loads with SWIZZLE_128B for a K-major A tile (128 x 32 fp32) and B tile (N x 32)
//  - SS MMA (A, B from shared memory descriptors), K advance inside the 128B swizzle atom
//  - TS MMA (A from TMEM, written by tcgen05.st from registers)
//  - tcgen05.ld epilogue
//  - whether kind::tf32 truncates or rounds the low 13 mantissa bits of fp32 operands
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 scripts/tc_probe.cu -o /tmp/tc_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra WAIT_%=;\n\t}"
                 ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                 ::"r"(smem_u32(dst)), "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1) : "memory");
}

__device__ __forceinline__ uint64_t sdesc_k_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);          // start address
    d |= (uint64_t)1 << 16;                           // LBO (ignored for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;                 // SBO: 8 rows x 128 B
    d |= (uint64_t)1 << 46;                           // version = 1 (sm100)
    d |= (uint64_t)2 << 61;                           // SWIZZLE_128B
    return d;
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_ss(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                 ::"r"(tmem_d), "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// K = 32 (one SW128 atom width), M = 128, N = NB (B rows). out1 = A * B^T (SS), out2 = lo(A) * B^T (TS)
template <int NB>
__global__ void probe(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                      float* out1, float* out2, float* outlo) {
    __shared__ __align__(1024) uint8_t sA[128 * 128];
    __shared__ __align__(1024) uint8_t sB[NB * 128];
    __shared__ uint64_t bar_tma, bar_mma, bar_lo;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(&bar_tma, 1);
        mbar_init(&bar_mma, 1);
        mbar_init(&bar_lo, 128);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = tmem_base;
    // columns: acc1 [0, NB), acc2 [64, 64+NB), A_lo [128, 160)
    if (threadIdx.x == 0) {
        mbar_expect(&bar_tma, 128 * 128 + NB * 128);
        tma2d(sA, &mapA, &bar_tma, 0, 0);
        tma2d(sB, &mapB, &bar_tma, 0, 0);
    }
    mbar_wait(&bar_tma, 0);
    // converters: all 4 warps, thread = row
    {
        const int r = threadIdx.x;
        float v[32];
        for (int c = 0; c < 8; ++c) {
            const float4 q = *reinterpret_cast<const float4*>(sA + r * 128 + ((c ^ (r & 7)) * 16));
            v[4 * c] = q.x; v[4 * c + 1] = q.y; v[4 * c + 2] = q.z; v[4 * c + 3] = q.w;
        }
        uint32_t lo[32];
        for (int j = 0; j < 32; ++j) {
            const float hi = __uint_as_float(__float_as_uint(v[j]) & 0xFFFFE000u);
            lo[j] = __float_as_uint(v[j] - hi);
            outlo[r * 32 + j] = v[j] - hi;
        }
        const uint32_t ta = tb + ((uint32_t)(32 * warp) << 16) + 128;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                     "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                     ::"r"(ta), "r"(lo[0]), "r"(lo[1]), "r"(lo[2]), "r"(lo[3]), "r"(lo[4]), "r"(lo[5]), "r"(lo[6]), "r"(lo[7]),
                     "r"(lo[8]), "r"(lo[9]), "r"(lo[10]), "r"(lo[11]), "r"(lo[12]), "r"(lo[13]), "r"(lo[14]), "r"(lo[15]),
                     "r"(lo[16]), "r"(lo[17]), "r"(lo[18]), "r"(lo[19]), "r"(lo[20]), "r"(lo[21]), "r"(lo[22]), "r"(lo[23]),
                     "r"(lo[24]), "r"(lo[25]), "r"(lo[26]), "r"(lo[27]), "r"(lo[28]), "r"(lo[29]), "r"(lo[30]), "r"(lo[31]));
        asm volatile("tcgen05.wait::st.sync.aligned;");
        asm volatile("tcgen05.fence::before_thread_sync;");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar_lo)) : "memory");
    }
    if (threadIdx.x == 0) {
        mbar_wait(&bar_lo, 0);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t id = idesc_tf32(128, NB);
        for (int k = 0; k < 4; ++k) {
            const uint64_t da = sdesc_k_sw128(smem_u32(sA) + 32 * k);
            const uint64_t db = sdesc_k_sw128(smem_u32(sB) + 32 * k);
            mma_ss(tb + 0, da, db, id, k > 0);
            mma_ts(tb + 64, tb + 128 + 8 * k, db, id, k > 0);
        }
        mma_commit(&bar_mma);
    }
    mbar_wait(&bar_mma, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    {
        const int r = threadIdx.x;
        for (int half = 0; half < 2; ++half) {
            uint32_t v[NB];
            const uint32_t ta = tb + ((uint32_t)(32 * warp) << 16) + (half ? 64 : 0);
            for (int c0 = 0; c0 < NB; c0 += 8) {
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=r"(v[c0]), "=r"(v[c0 + 1]), "=r"(v[c0 + 2]), "=r"(v[c0 + 3]), "=r"(v[c0 + 4]),
                               "=r"(v[c0 + 5]), "=r"(v[c0 + 6]), "=r"(v[c0 + 7])
                             : "r"(ta + c0));
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            float* o = half ? out2 : out1;
            for (int c = 0; c < NB; ++c) o[r * NB + c] = __uint_as_float(v[c]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(256));
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    constexpr int NB = 32;
    EncodeFn enc;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    std::vector<float> A(128 * 32), B(NB * 32);
    srand(1);
    for (int i = 0; i < 128 * 32; ++i) A[i] = (float)((rand() % 20001) - 10000) / 137.0f + 1e-3f * (rand() % 7);
    for (int i = 0; i < NB * 32; ++i) B[i] = (float)((rand() % 2001) - 1000) / 1000.0f;
    // rounding probe in row 0: A[0][0] = 1 + 0.75*2^-10 (nearest tf32 = 1 + 2^-10, truncation = 1)
    for (int j = 0; j < 32; ++j) A[j] = 0.f;
    A[0] = 1.0f + 0.75f * ldexpf(1.0f, -10);
    for (int c = 0; c < NB; ++c) B[c * 32 + 0] = (c == 0) ? 1.0f : 0.0f;
    float *dA, *dB, *o1, *o2, *olo;
    CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4));
    CK(cudaMalloc(&o1, 128 * NB * 4)); CK(cudaMalloc(&o2, 128 * NB * 4)); CK(cudaMalloc(&olo, 128 * 32 * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    CUtensorMap mA, mB;
    cuuint64_t dimsA[2] = {32, 128}, strA[1] = {32 * 4};
    cuuint32_t boxA[2] = {32, 128}, es[2] = {1, 1};
    if (enc(&mA, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dA, dimsA, strA, boxA, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("encA fail\n"); return 1; }
    cuuint64_t dimsB[2] = {32, NB}, strB[1] = {32 * 4};
    cuuint32_t boxB[2] = {32, NB};
    if (enc(&mB, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dB, dimsB, strB, boxB, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("encB fail\n"); return 1; }
    probe<NB><<<1, 128>>>(mA, mB, o1, o2, olo);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> r1(128 * NB), r2(128 * NB);
    CK(cudaMemcpy(r1.data(), o1, r1.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(r2.data(), o2, r2.size() * 4, cudaMemcpyDeviceToHost));
    printf("rounding probe: acc[0][0] = %.10f (trunc -> 1.0, nearest -> %.10f)\n", r1[0], 1.0 + ldexp(1.0, -10));
    // reference with truncated tf32 A_hi and B_hi, fp64
    auto tr = [](float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; float y; memcpy(&y, &u, 4); return y; };
    double e1 = 0, n1 = 0, e2 = 0, n2 = 0, efull = 0;
    for (int r = 1; r < 128; ++r)
        for (int c = 0; c < NB; ++c) {
            double s1 = 0, s2 = 0, sf = 0;
            for (int k = 0; k < 32; ++k) {
                const float a = A[r * 32 + k], b = B[c * 32 + k];
                s1 += (double)tr(a) * tr(b);
                s2 += (double)(a - tr(a)) * tr(b);
                sf += (double)a * b;
            }
            e1 = fmax(e1, fabs(r1[r * NB + c] - s1)); n1 = fmax(n1, fabs(s1));
            e2 = fmax(e2, fabs(r2[r * NB + c] - s2)); n2 = fmax(n2, fabs(s2));
            efull = fmax(efull, fabs(r1[r * NB + c] + r2[r * NB + c] - sf));
        }
    printf("SS max err vs trunc-tf32 ref: %.3e (scale %.3e)\n", e1, n1);
    printf("TS max err vs lo*trunc(B) ref: %.3e (scale %.3e)\n", e2, n2);
    printf("hi+lo vs exact (B trunc only): %.3e\n", efull);
    printf("sample r=5: gpu %f ref %f\n", r1[5 * NB + 3], 0.0);
    return 0;
}
