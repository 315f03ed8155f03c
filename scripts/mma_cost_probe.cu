// Cost model of tcgen05.mma kind::tf32 for the D-stream shapes: one thread issues NMMA
// back-to-back MMAs (same smem operands, accumulate), commit, wait; cycles per MMA.
// Shapes: SS / TS, M = 64 / 128, N = 16 .. 256, A K-major SW128 or MN-major SW128_32B.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 scripts/mma_cost_probe.cu -o scripts/mma_cost_probe
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, int a_mn, int b_mn, int bf16 = 0) {
    return (1u << 4) | ((bf16 ? 1u : 2u) << 7) | ((bf16 ? 1u : 2u) << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

constexpr int NMMA = 2048;

// mode: 0 SS A K-major, 1 SS A MN-major (BASE32B), 2 TS (A from TMEM), 3 SS B MN-major (BASE32B)
__global__ void probe(int M, int N, int mode, int nacc, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];   // 64 KB A region + 64 KB B region (zeros)
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 128 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = tslot;
    if (warp == 0 && (nacc < 0)) {
        // warp-converged issue: all 32 lanes run the loop, one elected lane issues (elect.sync)
        const int na = -nacc;
        const uint32_t sa = smem_u32(sm), sb = sa + 64 * 1024;
        const uint32_t id = idesc(M, N, mode == 1, mode == 3);
        const uint64_t da = mode == 1 ? desc(sa, 4096, 512, 1) : desc(sa, 16, 1024, 2);
        const uint64_t db = mode == 3 ? desc(sb, 4096, 512, 1) : desc(sb, 16, 1024, 2);
        const uint32_t at = tb + 256;
        const long long c0 = clock64();
        for (int i = 0; i < NMMA; ++i) {
            const uint32_t dt = tb + (uint32_t)((i & (na - 1)) * (256 / na));
            if (mode == 2)
                asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                             ::"r"(dt), "r"(at), "l"(db), "r"(id), "r"(1));
            else
                asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                             ::"r"(dt), "l"(da), "l"(db), "r"(id), "r"(1));
        }
        const long long c1 = clock64();
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("{\n\t.reg .pred P1;\n\tW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W2;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
        const long long c2 = clock64();
        if (threadIdx.x == 0) {
            out[0] = (unsigned long long)(c1 - c0);
            out[1] = (unsigned long long)(c2 - c0);
        }
    }
    if (threadIdx.x == 0 && nacc > 0 && mode >= 20) {
        // kind::i8 (signed 8-bit A and B, s32 accumulate): a/b_format = 1 (signed), c_format = 2 (S32)
        const uint32_t sa = smem_u32(sm), sb = sa + 64 * 1024;
        const uint32_t id = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        const uint64_t da = desc(sa, 16, 1024, 2), db = desc(sb, 16, 1024, 2);
        const long long c0 = clock64();
        for (int i = 0; i < NMMA; ++i)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                         ::"r"(tb), "l"(da), "l"(db), "r"(id), "r"(1));
        const long long c1 = clock64();
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("{\n\t.reg .pred P1;\n\tW4:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W4;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
        const long long c2 = clock64();
        out[0] = (unsigned long long)(c1 - c0);
        out[1] = (unsigned long long)(c2 - c0);
    }
    if (threadIdx.x == 0 && nacc > 0 && mode >= 10 && mode < 20) {
        const uint32_t sa = smem_u32(sm), sb = sa + 64 * 1024;
        const uint32_t id = idesc(M, N, 0, 0, 1);
        const uint64_t da = desc(sa, 16, 1024, 2), db = desc(sb, 16, 1024, 2);
        const uint32_t at = tb + 256;
        const long long c0 = clock64();
        for (int i = 0; i < NMMA; ++i) {
            if (mode == 12)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                             ::"r"(tb), "r"(at), "l"(db), "r"(id), "r"(1));
            else
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                             ::"r"(tb), "l"(da), "l"(db), "r"(id), "r"(1));
        }
        const long long c1 = clock64();
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("{\n\t.reg .pred P1;\n\tW3:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W3;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
        const long long c2 = clock64();
        out[0] = (unsigned long long)(c1 - c0);
        out[1] = (unsigned long long)(c2 - c0);
    }
    if (threadIdx.x == 0 && nacc > 0 && mode < 10) {
        const uint32_t sa = smem_u32(sm), sb = sa + 64 * 1024;
        const uint32_t id = idesc(M, N, mode == 1, mode == 3);
        const uint64_t da = mode == 1 ? desc(sa, 4096, 512, 1) : desc(sa, 16, 1024, 2);
        const uint64_t db = mode == 3 ? desc(sb, 4096, 512, 1) : desc(sb, 16, 1024, 2);
        const uint32_t at = tb + 256;      // A in TMEM for TS
        const long long c0 = clock64();
        for (int i = 0; i < NMMA; ++i) {
            const uint32_t dt = tb;
            if (mode == 2)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                             ::"r"(dt), "r"(at), "l"(db), "r"(id), "r"(1));
            else
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                             ::"r"(dt), "l"(da), "l"(db), "r"(id), "r"(1));
        }
        const long long c1 = clock64();
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
        const long long c2 = clock64();
        out[0] = (unsigned long long)(c1 - c0);
        out[1] = (unsigned long long)(c2 - c0);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
    const char* nmv[21] = {"tf32 SS", "tf32 SS-MN", "tf32 TS", "tf32 SS-BMN", "", "", "", "", "", "", "bf16 SS", "", "bf16 TS",
                           "", "", "", "", "", "", "", "i8 SS"};
    const char** nm = nmv;
    for (int nacc : {1})
    for (int mode : {0, 10, 20})
        for (int M : {128})
            for (int N : {16, 32, 48, 64, 128, 256}) {
                if (N * (nacc < 0 ? -nacc : nacc) > 256) continue;
                probe<<<1, 128, 128 * 1024>>>(M, N, mode, nacc, d);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("%s M=%d N=%d: %s\n", nm[mode], M, N, cudaGetErrorString(e)); return 1; }
                unsigned long long h[2];
                cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
                const double cyc = (double)h[1] / NMMA;
                const double abytes = M * 32, bbytes = N * 32;
                printf("nacc=%d ", nacc);
                printf("%s M=%3d N=%3d: %6.1f cyc/MMA (issue %6.1f)  A %4.0f B/cyc  B %4.0f B/cyc  %6.0f flop/cyc\n", nm[mode], M,
                       N, cyc, (double)h[0] / NMMA, abytes / cyc, bbytes / cyc, 2.0 * M * N * 8 / cyc);
            }
    return 0;
}
