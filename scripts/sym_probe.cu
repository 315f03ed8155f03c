// Probes for a paired (normal + transposed) symmetric-half D stream:
//  1. the smem layout TMA produces with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B (fp32, 128 B rows)
//  2. tcgen05 kind::tf32 SS MMA with an MN-major A operand in that layout (SWIZZLE_128B_BASE32B
//     descriptor): out[j][c] = sum_i D[i][j] * Y[i][c], against an fp64 reference
//  3. bulk-copy streaming: every CTA streams unique bytes vs CTA pairs streaming the same bytes
//     (plain grid and 2-CTA clusters) -> does L2 merge the pair's requests, and how fast is L2->SM
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 scripts/sym_probe.cu -o /tmp/sym_probe -lcuda
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
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"((uint64_t)src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// ---- 1. layout dump: box {32 cols, 8 rows}, value = row*32+col
__global__ void dump(const __grid_constant__ CUtensorMap map, float* out) {
    __shared__ __align__(1024) float s[8 * 32];
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_expect(&bar, sizeof(s));
        tma2d(s, &map, &bar, 0, 0);
    }
    __syncthreads();
    mbar_wait(&bar, 0);
    for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = s[i];
}

// ---- 2. MN-major A: D tile KR rows (i) x 128 cols (j) in 4 boxes {32, KR}; B = Y^T (NB x KR) K-major SW128
template <int KR, int NB>
__global__ void mnmajor(const __grid_constant__ CUtensorMap mapD, const __grid_constant__ CUtensorMap mapY,
                        float* out, uint32_t lbo, uint32_t sbo, uint32_t kstep) {
    __shared__ __align__(1024) uint8_t sD[4 * KR * 128];
    __shared__ __align__(1024) uint8_t sY[(KR / 32) * NB * 128];
    __shared__ uint64_t bar_tma, bar_mma;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        mbar_init(&bar_tma, 1);
        mbar_init(&bar_mma, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = tmem_base;
    if (threadIdx.x == 0) {
        mbar_expect(&bar_tma, sizeof(sD) + sizeof(sY));
        for (int a = 0; a < 4; ++a) tma2d(sD + a * KR * 128, &mapD, &bar_tma, 32 * a, 0);
        for (int q = 0; q < KR / 32; ++q) tma2d(sY + q * NB * 128, &mapY, &bar_tma, 32 * q, 0);
        mbar_wait(&bar_tma, 0);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t id = idesc_tf32(128, NB, 1, 0);
        for (int k = 0; k < KR / 8; ++k) {
            const uint64_t da = sdesc(smem_u32(sD) + k * kstep, lbo, sbo, 1);
            const int q = k / 4, kk = k % 4;
            const uint64_t db = sdesc(smem_u32(sY) + q * NB * 128 + 32 * kk, 16, 1024, 2);
            mma_ss(tb, da, db, id, k > 0);
        }
        mma_commit(&bar_mma);
    }
    __syncwarp();
    mbar_wait(&bar_mma, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int r = threadIdx.x;
    uint32_t v[NB];
    const uint32_t ta = tb + ((uint32_t)(32 * warp) << 16);
    for (int c0 = 0; c0 < NB; c0 += 8)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[c0]), "=r"(v[c0 + 1]), "=r"(v[c0 + 2]), "=r"(v[c0 + 3]), "=r"(v[c0 + 4]),
                       "=r"(v[c0 + 5]), "=r"(v[c0 + 6]), "=r"(v[c0 + 7])
                     : "r"(ta + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int c = 0; c < NB; ++c) out[r * NB + c] = __uint_as_float(v[c]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(64));
}

// ---- 3. streaming: unit u of U streams chunks u, u+U, ... (CHUNK bytes each) through an NS-stage ring
constexpr int CHUNK = 48 * 1024, NS = 4;
__global__ void stream(const uint8_t* buf, int64_t nchunks, int pair, float* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[NS];
    const int U = pair ? gridDim.x / 2 : gridDim.x;
    const int u = pair ? blockIdx.x / 2 : blockIdx.x;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    float acc = 0.f;
    int64_t issued = 0, done = 0;
    const int64_t mine = nchunks > u ? (nchunks - 1 - u) / U + 1 : 0;
    for (; issued < mine && issued < NS; ++issued) {
        const int s = issued % NS;
        mbar_expect(&full[s], CHUNK);
        bulk(sm + s * CHUNK, buf + (u + issued * U) * (int64_t)CHUNK, CHUNK, &full[s]);
    }
    for (; done < mine; ++done) {
        const int s = done % NS;
        mbar_wait(&full[s], (done / NS) & 1);
        acc += reinterpret_cast<const float*>(sm + s * CHUNK)[done & 255];
        if (issued < mine) {
            const int s2 = issued % NS;
            mbar_expect(&full[s2], CHUNK);
            bulk(sm + s2 * CHUNK, buf + (u + issued * U) * (int64_t)CHUNK, CHUNK, &full[s2]);
            ++issued;
        }
    }
    if (acc == 12345.f) sink[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn enc;
static void encode(CUtensorMap* m, float* p, uint64_t cols, uint64_t rows, uint32_t bc, uint32_t br, CUtensorMapSwizzle sw) {
    cuuint64_t dims[2] = {cols, rows}, str[1] = {cols * 4};
    cuuint32_t box[2] = {bc, br}, es[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, p, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); exit(1); }
}

template <int KR, int NB>
static void run_mn(uint32_t lbo, uint32_t sbo, uint32_t kstep) {
    std::vector<float> D(KR * 128), Y(NB * KR);
    srand(7);
    for (auto& x : D) x = (float)((rand() % 20001) - 10000) / 137.0f;
    for (auto& x : Y) x = (float)((rand() % 2001) - 1000) / 1000.0f;
    float *dD, *dY, *dO;
    CK(cudaMalloc(&dD, D.size() * 4)); CK(cudaMalloc(&dY, Y.size() * 4)); CK(cudaMalloc(&dO, 128 * NB * 4));
    CK(cudaMemcpy(dD, D.data(), D.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dY, Y.data(), Y.size() * 4, cudaMemcpyHostToDevice));
    CUtensorMap mD, mY;
    encode(&mD, dD, 128, KR, 32, KR, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    encode(&mY, dY, KR, NB, 32, NB, CU_TENSOR_MAP_SWIZZLE_128B);   // Y^T stored NB rows x KR
    mnmajor<KR, NB><<<1, 128>>>(mD, mY, dO, lbo, sbo, kstep);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> O(128 * NB);
    CK(cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost));
    auto tr = [](float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; float y; memcpy(&y, &u, 4); return y; };
    double e = 0, sc = 0;
    for (int j = 0; j < 128; ++j)
        for (int c = 0; c < NB; ++c) {
            double s = 0;
            for (int i = 0; i < KR; ++i) s += (double)tr(D[i * 128 + j]) * tr(Y[c * KR + i]);
            e = fmax(e, fabs(O[j * NB + c] - s)); sc = fmax(sc, fabs(s));
        }
    printf("MN-major KR=%d NB=%d lbo=%u sbo=%u kstep=%u: max err %.3e (scale %.3e) %s\n", KR, NB, lbo, sbo, kstep, e, sc,
           e < 1e-4 * sc ? "OK" : "BAD");
    cudaFree(dD); cudaFree(dY); cudaFree(dO);
}

int main() {
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    // 1. layout
    {
        std::vector<float> h(8 * 32);
        for (int i = 0; i < 256; ++i) h[i] = (float)i;
        float *d, *o;
        CK(cudaMalloc(&d, 1024)); CK(cudaMalloc(&o, 1024));
        CK(cudaMemcpy(d, h.data(), 1024, cudaMemcpyHostToDevice));
        for (int mode = 0; mode < 2; ++mode) {
            CUtensorMap m;
            encode(&m, d, 32, 8, 32, 8, mode ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B);
            dump<<<1, 32>>>(m, o);
            CK(cudaDeviceSynchronize());
            std::vector<float> r(256);
            CK(cudaMemcpy(r.data(), o, 1024, cudaMemcpyDeviceToHost));
            printf("%s: smem row -> element col at each 16B slot (first elem of slot)\n", mode ? "128B_ATOM_32B" : "128B");
            for (int row = 0; row < 8; ++row) {
                printf("  row %d:", row);
                for (int sl = 0; sl < 8; ++sl) {
                    const int v = (int)r[row * 32 + sl * 4];
                    printf(" %d:%d", v / 32, v % 32);
                }
                printf("\n");
            }
        }
    }
    // 2. MN-major MMA
    run_mn<32, 16>(32 * 128, 512, 1024);
    run_mn<32, 16>(512, 32 * 128, 1024);
    run_mn<64, 16>(64 * 128, 512, 1024);
    run_mn<64, 32>(64 * 128, 512, 1024);
    // 3. streaming
    {
        const int64_t bytes = 6LL << 30;
        const int64_t nchunks = bytes / CHUNK;
        uint8_t* buf;
        float* sink;
        CK(cudaMalloc(&buf, nchunks * (int64_t)CHUNK));
        CK(cudaMalloc(&sink, 4));
        CK(cudaMemset(buf, 1, nchunks * (int64_t)CHUNK));
        CK(cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, NS * CHUNK));
        int sms;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
        for (int mode = 0; mode < 4; ++mode) {
            // mode 0: unique, full buffer; 1: unique, half buffer; 2: pairs over half buffer; 3: pairs in clusters of 2
            const int64_t nc = mode == 0 ? nchunks : nchunks / 2;
            float best = 1e30f;
            for (int rep = 0; rep < 4; ++rep) {
                CK(cudaEventRecord(e0));
                if (mode == 3) {
                    cudaLaunchConfig_t cfg = {};
                    cfg.gridDim = dim3(sms); cfg.blockDim = dim3(32); cfg.dynamicSmemBytes = NS * CHUNK;
                    cudaLaunchAttribute at[1];
                    at[0].id = cudaLaunchAttributeClusterDimension;
                    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
                    cfg.attrs = at; cfg.numAttrs = 1;
                    CK(cudaLaunchKernelEx(&cfg, stream, (const uint8_t*)buf, nc, 1, sink));
                } else {
                    stream<<<sms, 32, NS * CHUNK>>>(buf, nc, mode >= 2, sink);
                }
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
                CK(cudaGetLastError());
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                if (rep) best = fminf(best, ms);
            }
            const double uniq = (double)nc * CHUNK, sm_bytes = (mode >= 2 ? 2.0 : 1.0) * uniq;
            printf("stream mode %d: %.3f ms  unique %.2f GB -> %.0f GB/s HBM-side, %.0f GB/s L2->SM\n", mode, best,
                   uniq / 1e9, uniq / best / 1e6, sm_bytes / best / 1e6);
        }
    }
    return 0;
}
