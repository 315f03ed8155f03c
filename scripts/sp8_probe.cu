// Probe: tcgen05.mma kind::i8 on NO-SWIZZLE (interleaved core-matrix) shared-memory images,
// the layout of the row-blocked S images (k_sp8.cuh). One image of 128 rows x KD int8
// (core matrix = 8 rows x 16 contiguous bytes, core (rg, kc) at ((kc * 16 + rg) * 128)) is used
//   N: as a K-major A (M = row r, K = column k) against B_N (K-major, 48 x KD),
//   T: as an MN-major A (M = column k, K = row r) against B_T (K-major, 48 x 128).
// For each product, all four (LBO, SBO) assignments are tried and compared with the host.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 scripts/sp8_probe.cu -o scripts/sp8_probe
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int KD = 128, NB = 48;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, int a_mn) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}
__host__ __device__ inline int off_img(int r, int k) { return ((k / 16) * 16 + r / 8) * 128 + (r % 8) * 16 + k % 16; }
__host__ __device__ inline int off_b(int n, int k) { return ((k / 16) * (NB / 8) + n / 8) * 128 + (n % 8) * 16 + k % 16; }
// MN-major B: core = 8 K-rows x 16 contiguous N bytes, core (k group, n group) at (kg * NB/16 + ng) * 128
__host__ __device__ inline int off_bmn(int n, int k) { return ((k / 8) * (NB / 16) + n / 16) * 128 + (k % 8) * 16 + n % 16; }
__host__ __device__ constexpr uint32_t idesc_i8b(int M, int N, int a_mn, int b_mn) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}

__global__ void probe(const int8_t* S, const int8_t* Yd, const int8_t* Z, int mode, int variant, int* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    int8_t* img = reinterpret_cast<int8_t*>(sm);              // 128 x KD
    int8_t* bn = img + 128 * KD;                              // 48 x KD
    int8_t* bt = bn + NB * KD;                                // 48 x 128
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int e = threadIdx.x; e < 128 * KD; e += blockDim.x) img[off_img(e / KD, e % KD)] = S[e];
    for (int e = threadIdx.x; e < KD * NB; e += blockDim.x)
        bn[mode == 2 ? off_bmn(e % NB, e / NB) : off_b(e % NB, e / NB)] = Yd[e];   // Yd[k][n]
    for (int e = threadIdx.x; e < 128 * NB; e += blockDim.x) bt[off_b(e % NB, e / NB)] = Z[e];    // Z[r][n]
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
    if (threadIdx.x == 0) {
        const uint32_t si = smem_u32(img), sn = smem_u32(bn), st = smem_u32(bt);
        const uint32_t bl = (variant & 2) ? 128 : 768, bs = (variant & 2) ? 768 : 128;   // B: LBO / SBO
        if (mode == 2) {   // N product with an MN-major B (SBO along N = 128, LBO along K = 384)
            const uint32_t bl2 = (variant & 2) ? 128 : 384, bs2 = (variant & 2) ? 384 : 128;
            for (int j = 0; j < KD / 32; ++j) {
                const uint64_t a = desc_none(si + 4096 * j, 2048, 128), b = desc_none(sn + 1536 * j, bl2, bs2);
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tb),
                             "l"(a), "l"(b), "r"(idesc_i8b(128, NB, 0, 1)), "r"(j > 0 ? 1u : 0u));
            }
        } else if (mode == 0) {
            const uint32_t al = (variant & 1) ? 128 : 2048, as = (variant & 1) ? 2048 : 128;
            for (int j = 0; j < KD / 32; ++j) {
                const uint64_t a = desc_none(si + 4096 * j, al, as), b = desc_none(sn + 1536 * j, bl, bs);
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tb),
                             "l"(a), "l"(b), "r"(idesc_i8(128, NB, 0)), "r"(j > 0 ? 1u : 0u));
            }
        } else {
            const uint32_t al = (variant & 1) ? 2048 : 128, as = (variant & 1) ? 128 : 2048;
            for (int j = 0; j < 4; ++j) {
                const uint64_t a = desc_none(si + 4 * 128 * j, al, as), b = desc_none(st + 1536 * j, bl, bs);
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tb),
                             "l"(a), "l"(b), "r"(idesc_i8(128, NB, 1)), "r"(j > 0 ? 1u : 0u));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                     : "memory");
    }
    __syncwarp();
    {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\tselp.u32 %0,1,0,P1;\n\t}"
                         : "=r"(ok)
                         : "r"(smem_u32(&bar)));
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp < 4) {
        for (int c = 0; c < NB; c += 8) {
            uint32_t v[8];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                         : "r"(tb + ((uint32_t)(32 * warp) << 16) + c));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            for (int u = 0; u < 8; ++u) out[(32 * warp + lane) * NB + c + u] = (int)v[u];
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

// timing: one thread issues nm MMAs (mode 0: N product, A K-major; 1: T product, A MN-major;
// 2: N product with MN-major B), commit, wait; cycles per MMA
__global__ void timing(int mode, int nm, int N, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 7);
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
    if (threadIdx.x == 0) {
        const uint32_t sa = smem_u32(sm), sb = sa + 48 * 1024;
        uint64_t a, b;
        uint32_t id;
        if (mode == 0) { a = desc_none(sa, 2048, 128); b = desc_none(sb, 384, 128); id = idesc_i8b(128, N, 0, 1); }
        else if (mode == 1) { a = desc_none(sa, 128, 2048); b = desc_none(sb, 384, 128); id = idesc_i8b(128, N, 1, 1); }
        else { a = desc_none(sa, 2048, 128); b = desc_none(sb, 768, 128); id = idesc_i8b(128, N, 0, 0); }
        const long long c0 = clock64();
        for (int i = 0; i < nm; ++i)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tb + 64 * (i & 3)),
                         "l"(a), "l"(b), "r"(id), "r"(1u));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\tselp.u32 %0,1,0,P1;\n\t}"
                         : "=r"(ok) : "r"(smem_u32(&bar)));
        out[0] = (unsigned long long)(clock64() - c0);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

int main(int argc, char** argv) {
    if (argc > 1 && argv[1][0] == 't') {
        unsigned long long* d;
        cudaMalloc(&d, 8);
        cudaFuncSetAttribute(timing, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        for (int mode = 0; mode < 3; ++mode)
            for (int N : {16, 32, 48, 64}) {
                unsigned long long c = 0;
                timing<<<1, 128, 64 * 1024>>>(mode, 2048, N, d);
                cudaDeviceSynchronize();
                cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
                printf("mode %d (%s) N=%d: %.1f cycles per MMA\n", mode,
                       mode == 0 ? "N: A K-major, B MN-major" : (mode == 1 ? "T: A MN-major, B MN-major" : "N: A K-major, B K-major"),
                       N, (double)c / 2048);
            }
        return 0;
    }
    const int only_mode = argc > 1 ? atoi(argv[1]) : -1, only_var = argc > 2 ? atoi(argv[2]) : -1;
    std::vector<int8_t> S(128 * KD), Yd(KD * NB), Z(128 * NB);
    srand(1);
    for (auto& v : S) v = (int8_t)(rand() % 256 - 128);
    for (auto& v : Yd) v = (int8_t)(rand() % 256 - 128);
    for (auto& v : Z) v = (int8_t)(rand() % 256 - 128);
    int8_t *dS, *dY, *dZ;
    int* dO;
    cudaMalloc(&dS, S.size());
    cudaMalloc(&dY, Yd.size());
    cudaMalloc(&dZ, Z.size());
    cudaMalloc(&dO, 128 * NB * 4);
    cudaMemcpy(dS, S.data(), S.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dY, Yd.data(), Yd.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dZ, Z.data(), Z.size(), cudaMemcpyHostToDevice);
    const int smem = 128 * KD + NB * KD + NB * 128 + 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int mode = 0; mode < 3; ++mode) {
        for (int variant = 0; variant < 4; ++variant) {
            if ((only_mode >= 0 && mode != only_mode) || (only_var >= 0 && variant != only_var)) continue;
            cudaMemset(dO, 0, 128 * NB * 4);
            probe<<<1, 128, smem>>>(dS, dY, dZ, mode, variant, dO);
            cudaError_t e = cudaDeviceSynchronize();
            std::vector<int> O(128 * NB);
            cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
            long bad = 0;
            for (int m = 0; m < 128; ++m)
                for (int n = 0; n < NB; ++n) {
                    long ref = 0;
                    if (mode != 1)
                        for (int k = 0; k < KD; ++k) ref += (long)S[m * KD + k] * Yd[k * NB + n];
                    else
                        for (int r = 0; r < 128; ++r) ref += (long)S[r * KD + m] * Z[r * NB + n];
                    bad += (ref != O[m * NB + n]);
                }
            printf("mode %s variant %d (A %s, B %s): %s, mismatches %ld / %d\n", mode == 1 ? "T (A MN-major)" : (mode == 2 ? "N, B MN-major" : "N (A K-major)"),
                   variant, (variant & 1) ? "swapped" : "assumed", (variant & 2) ? "swapped" : "assumed",
                   cudaGetErrorString(e), bad, 128 * NB);
            if (e != cudaSuccess) return 1;
        }
    }
    return 0;
}
