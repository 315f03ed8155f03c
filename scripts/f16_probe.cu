// Probe of the 2xFP16 split on tcgen05 kind::f16 (f32 accumulate), A from TMEM (TS):
//   A (128 x 64 fp32, scaled) -> h1 = f16(a), h2 = f16(a - h1) packed in TMEM (two f16 per column)
//   B (N x 64 fp32, scaled)   -> [y1; y2] f16, K-major SWIZZLE_128B in smem (64 f16 = 128 B per row)
//   acc = h1 * [y1 | y2] + h2 * [y1 | y2] (N = 2 * NB)
// Checks the TMEM packing order (low half = even k) and the accuracy against fp64.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 scripts/f16_probe.cu -o scripts/f16_probe
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <random>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_k_sw128(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
           ((uint64_t)2 << 61);
}
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {   // A, B f16 (format 0), f32 accumulate
    return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

constexpr int NB = 16;   // y columns; B rows = 2 * NB

__global__ void probe(const float* A, const float* Bm, float* out) {
    __shared__ __align__(1024) __half sB[2 * NB * 64];   // 2NB rows x 64 k, SW128
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, r = threadIdx.x;
    // B: row n (< NB: y1 of column n, else y2 of column n - NB), k = 0..63; SW128: 16-byte granule g at g ^ (row & 7)
    for (int e = threadIdx.x; e < 2 * NB * 64; e += 128) {
        const int n = e / 64, k = e % 64, c = n % NB;
        const float y = Bm[c * 64 + k];
        const __half y1 = __float2half_rn(y);
        const __half y2 = __float2half_rn(y - __half2float(y1));
        const int g = k / 8, w = k % 8;
        sB[n * 64 + ((g ^ (n & 7)) * 8) + w] = n < NB ? y1 : y2;
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = tslot;
    // A pieces into TMEM: lane r, h1 at columns [64, 96), h2 at [96, 128); column j holds k = 2j (low), 2j+1 (high)
    {
        uint32_t p1[32], p2[32];
        for (int j = 0; j < 32; ++j) {
            const float a0 = A[r * 64 + 2 * j], a1 = A[r * 64 + 2 * j + 1];
            const __half2 h = __floats2half2_rn(a0, a1);                 // .x = a0 (low 16 bits)
            const float2 hf = __half22float2(h);
            const __half2 l = __floats2half2_rn(a0 - hf.x, a1 - hf.y);
            p1[j] = *reinterpret_cast<const uint32_t*>(&h);
            p2[j] = *reinterpret_cast<const uint32_t*>(&l);
        }
        const uint32_t ta = tb + ((uint32_t)(32 * warp) << 16);
#define ST32(addr, v)                                                                                                  \
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16," \
                 "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),                        \
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),      \
                 "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),          \
                 "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),         \
                 "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]))
        ST32(ta + 64, p1);
        ST32(ta + 96, p2);
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x == 0) {
        const uint32_t id = idesc_f16(128, 2 * NB);
        for (int ks = 0; ks < 4; ++ks) {   // K = 16 per MMA: 8 TMEM columns, 32 bytes of a B row
            const uint64_t db = desc_k_sw128(smem_u32(sB) + 32 * ks);
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                         ::"r"(tb), "r"(tb + 64 + 8 * ks), "l"(db), "r"(id), "r"(ks));
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                         ::"r"(tb), "r"(tb + 96 + 8 * ks), "l"(db), "r"(id), "r"(1));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    }
    __syncwarp();
    asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t v[2 * NB];
    const uint32_t ta = tb + ((uint32_t)(32 * warp) << 16);
    for (int c0 = 0; c0 < 2 * NB; c0 += 8)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[c0]), "=r"(v[c0 + 1]), "=r"(v[c0 + 2]), "=r"(v[c0 + 3]), "=r"(v[c0 + 4]),
                       "=r"(v[c0 + 5]), "=r"(v[c0 + 6]), "=r"(v[c0 + 7])
                     : "r"(ta + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int c = 0; c < NB; ++c) out[r * NB + c] = __uint_as_float(v[c]) + __uint_as_float(v[NB + c]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tb));
}

int main() {
    std::mt19937 g(3);
    std::uniform_real_distribution<float> ua(0.f, 16384.f), ub(-32768.f, 32768.f);
    std::vector<float> A(128 * 64), B(NB * 64), O(128 * NB);
    for (auto& x : A) x = ua(g);
    for (auto& x : B) x = ub(g) * (g() % 4 == 0 ? 1e-3f : 1.f);
    float *dA, *dB, *dO;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dO, O.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    probe<<<1, 128>>>(dA, dB, dO);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    double emax = 0, nrm = 0, eabs = 0;
    for (int r = 0; r < 128; ++r)
        for (int c = 0; c < NB; ++c) {
            double s = 0, sa = 0;
            for (int k = 0; k < 64; ++k) { s += (double)A[r * 64 + k] * B[c * 64 + k]; sa += fabs((double)A[r * 64 + k] * B[c * 64 + k]); }
            emax = fmax(emax, fabs(O[r * NB + c] - s) / sa);
            eabs = fmax(eabs, fabs(O[r * NB + c] - s));
            nrm = fmax(nrm, fabs(s));
        }
    printf("2xF16 TS: max |err| / sum|a b| = %.3e (fp32 eps 6e-8), max abs err %.3e, scale %.3e\n", emax, eabs, nrm);
    return 0;
}
