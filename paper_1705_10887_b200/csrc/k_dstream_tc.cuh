// A3 on the 5th-gen tensor cores: Y2 = D_ll Y1 with tcgen05.mma kind::tf32 and a 3xTF32
// split, so the contraction keeps fp32 accuracy (1xTF32 gives ~1e-3, 3xTF32
// ~3e-6 against the 1e-5 bar) while D streams from HBM once ("W is small").
//
//   Y2 = D_hi [Y_hi | Y_lo] + D_lo Y_hi     (fp32 accumulate in TMEM, drained to fp64)
//
// kind::tf32 reads an fp32 word and ignores its low 13 mantissa bits (truncation; measured
// by scripts/tc_probe.cu on B200), so D_hi is the raw TMA tile and D_lo = D - (D & ~0x1FFF)
// is exact in fp32. Y1 is split once per apply into Y1T = [Y_hi; Y_lo] (2*bp x l_pad,
// K-major) by k_split_y1.
//
// CTA (one per SM, stream-K over (128-row tile, 32-k tile) iterations, like k_dstream_ffma):
//   warp 0  lane 0   TMA producer: D tile 128 x 32 fp32 (16 KB, SWIZZLE_128B) + B tile
//                    2bp x 32 (SWIZZLE_128B), complete_tx on full[s]
//   warp 1           TMEM allocator; lane 0 issues the MMAs (SS: A = D_hi from smem; TS:
//                    A = D_lo from TMEM) and tcgen05.commit -> empty[s] / acc_full[buf]
//   warps 4-7        converters: thread = tile row = TMEM lane; read the row's fp32 values
//                    from the swizzled tile, D_lo -> tcgen05.st into TMEM slot s, arrive
//                    lo_ready[s] (every stage)
//   warps 8-11       epilogue: every KC k-tiles wait acc_full, drain the accumulators
//                    (tcgen05.ld) into fp64 registers, arrive acc_empty; at a row-tile
//                    boundary write the fp64 partial for k_dreduce (deterministic, same
//                    layout as the FFMA path)
// Each mbarrier has one producer role and one consumer role (canonical warp specialisation);
// an earlier variant in which two converter groups also drained with a lag could deadlock.
#pragma once
#include "common.cuh"
#include "k_dstream.cuh"

namespace sbmds {

template <int BP>
struct TcCfg {
    static constexpr int TM = 128;                       // tile rows (MMA M)
    static constexpr int NA = BP >= 32 ? 2 : 3;          // 128B swizzle atoms (32 fp32 of k) per stage
    static constexpr int TK = 32 * NA;                   // k per stage: 256 contiguous bytes per D row
    static constexpr int NB = 2 * BP;                    // B rows: [Y_hi; Y_lo]
    static constexpr int N1 = NB;                        // D_hi * [Y_hi | Y_lo]
    static constexpr int N2 = BP < 16 ? 16 : BP;         // D_lo * Y_hi (b=8: also Y_lo rows)
    static constexpr int N1C = (N1 + 31) / 32 * 32;         // 32-column aligned TMEM regions
    static constexpr int N2C = (N2 + 31) / 32 * 32;
    static constexpr int ACC_COLS = N1C + N2C;
    static constexpr int A_ATOM = TM * 128;              // 16 KB: 128 rows x 32 fp32, SWIZZLE_128B
    static constexpr int B_ATOM = NB * 128;
    static constexpr int A_BYTES = NA * A_ATOM;
    static constexpr int B_BYTES = NA * B_ATOM;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int NS_SMEM = (200 * 1024) / STAGE_BYTES;
    static constexpr int NS_TMEM = (512 - 2 * ACC_COLS) / (32 * NA);
    static constexpr int NS = NS_SMEM < NS_TMEM ? (NS_SMEM < 8 ? NS_SMEM : 8) : (NS_TMEM < 8 ? NS_TMEM : 8);
    static constexpr int TMEM_COLS = 512;
    static constexpr int ACC0 = 0;                       // acc buffer b at column b*ACC_COLS
    static constexpr int LO0 = 2 * ACC_COLS;             // A_lo slots
    static constexpr int KC = NA == 3 ? 5 : 16 / NA;     // k-tiles per accumulator drain (~512 k)
    static constexpr int THREADS = 12 * 32;               // producer, MMA, 2 idle, converters, epilogue
    static constexpr int SMEM = NS * STAGE_BYTES + 1024 + 256;
    static_assert(NS >= 2, "stages");
    static_assert(LO0 + NS * 32 * NA <= TMEM_COLS, "tmem");
};

__device__ __forceinline__ uint64_t umma_desc_k_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);   // start address >> 4
    d |= (uint64_t)1 << 16;                    // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;          // SBO: 8 rows x 128 B atoms
    d |= (uint64_t)1 << 46;                    // descriptor version (sm100)
    d |= (uint64_t)2 << 61;                    // SWIZZLE_128B
    return d;
}

__host__ __device__ constexpr uint32_t idesc_tf32_f32acc(int M, int N) {
    // c_format F32 (bit 4), a/b_format TF32 (2 at bits 7, 10), K-major A and B,
    // n_dim = N >> 3 (bits 17..22), m_dim = M >> 4 (bits 24..28)
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void tc_mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tc_mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                 "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Y1 (l_pad x bp, row-major) -> Y1T (2bp x l_pad): rows [0, bp) = tf32 hi, rows [bp, 2bp) = lo.
// With Rinv (eigs, b x b upper triangular) the block is first right-multiplied by R^-1 in
// fp64 (the R^-1 fold). A block stages 256/bp rows of Y1 in shared memory.
__global__ void __launch_bounds__(256) k_split_y1(int64_t lpad, int b, int bp, const double* __restrict__ Rinv,
                                                  const float* __restrict__ Y1, float* __restrict__ Y1T) {
    __shared__ double Ms[64 * 64];
    __shared__ float ys[256];
    if (Rinv)
        for (int e = threadIdx.x; e < b * b; e += blockDim.x) Ms[e] = Rinv[e];
    const int rb = 256 / bp;
    const int r = threadIdx.x % rb, c = threadIdx.x / rb;   // consecutive threads: consecutive k
    for (int64_t k0 = (int64_t)blockIdx.x * rb; k0 < lpad; k0 += (int64_t)gridDim.x * rb) {
        __syncthreads();
        const int64_t k = k0 + r;
        ys[r * bp + c] = (k < lpad) ? Y1[k * bp + c] : 0.f;
        __syncthreads();
        if (k < lpad) {
            float v = ys[r * bp + c];
            if (Rinv && c < b) {
                double acc = 0.0;
                for (int p = 0; p <= c; ++p) acc = fma((double)ys[r * bp + p], Ms[p * b + c], acc);
                v = (float)acc;
            }
            const float hi = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
            Y1T[(int64_t)c * lpad + k] = hi;
            Y1T[(int64_t)(bp + c) * lpad + k] = v - hi;
        }
    }
}

template <int BP>
__global__ void __launch_bounds__(TcCfg<BP>::THREADS, 1)
    k_dstream_tc(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap, StreamK sk,
                 int maxseg, double* __restrict__ P) {
    using C = TcCfg<BP>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(base + C::NS * C::STAGE_BYTES);
    uint64_t* empty = full + C::NS;
    uint64_t* lo_ready = empty + C::NS;
    uint64_t* acc_full = lo_ready + C::NS;   // [2]
    uint64_t* acc_empty = acc_full + 2;      // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x;
    const int64_t it0 = sk.beg(c), it1 = sk.beg(c + 1);

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
            mbar_init(&lo_ready[s], 128);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 128);
        }
        fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(C::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;

    const int32_t KT = (int32_t)sk.KT;
    // k-tile kt (of the current row tile) ends an accumulator chunk?
    auto chunk_end = [&](int64_t it, int32_t kt) {
        return it + 1 == it1 || kt + 1 == KT || ((kt + 1) % C::KC) == 0;
    };

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            prefetch_tensormap(&amap);
            prefetch_tensormap(&bmap);
            const uint64_t pol = policy_evict_first();
            const uint64_t polb = policy_evict_last();
            int s = 0;
            uint32_t ph = 0;
            int32_t rt = (int32_t)(it0 / sk.KT), kt = (int32_t)(it0 % sk.KT);
            const int32_t KT = (int32_t)sk.KT;
            for (int64_t it = it0; it < it1; ++it) {
                mbar_wait(&empty[s], ph ^ 1u, 101 * 65536 + (int)((it - it0) & 0xFFFF));
                uint8_t* st = base + s * C::STAGE_BYTES;
                mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
#pragma unroll
                for (int a = 0; a < C::NA; ++a) {
                    tma_load_2d(st + a * C::A_ATOM, &amap, &full[s], kt * C::TK + 32 * a, rt * C::TM, pol);
                    tma_load_2d(st + C::A_BYTES + a * C::B_ATOM, &bmap, &full[s], kt * C::TK + 32 * a, 0, polb);
                }
                if (++s == C::NS) { s = 0; ph ^= 1u; }
                if (++kt == KT) { kt = 0; ++rt; }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            constexpr uint32_t id1 = idesc_tf32_f32acc(C::TM, C::N1);
            constexpr uint32_t id2 = idesc_tf32_f32acc(C::TM, C::N2);
            int buf = 0, nchunk = 0;
            bool first = true;
            int s = 0;
            uint32_t ph = 0;
            int32_t kt = (int32_t)(it0 % sk.KT);
            for (int64_t it = it0; it < it1; ++it) {
                if (first) {
                    // wait until the epilogue has drained this accumulator buffer (2 chunks ago)
                    mbar_wait(&acc_empty[buf], (uint32_t)(((nchunk >> 1) & 1) ^ 1), 102 * 65536 + (int)((it - it0) & 0xFFFF));
                    tc_fence_after();
                }
                mbar_wait(&full[s], ph, 103 * 65536 + (int)((it - it0) & 0xFFFF));
                mbar_wait(&lo_ready[s], ph, 104 * 65536 + (int)((it - it0) & 0xFFFF));
                tc_fence_after();
                const uint32_t sa = smem_u32(base + s * C::STAGE_BYTES);
                const uint32_t sb = sa + C::A_BYTES;
                const uint32_t d1 = tbase + C::ACC0 + buf * C::ACC_COLS;
                const uint32_t d2 = d1 + C::N1C;
                const uint32_t alo = tbase + C::LO0 + s * 32 * C::NA;
#pragma unroll
                for (int a = 0; a < C::NA; ++a) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t acc = (first && a == 0 && j == 0) ? 0u : 1u;
                        const uint64_t db = umma_desc_k_sw128(sb + a * C::B_ATOM + 32 * j);
                        tc_mma_ss(d1, umma_desc_k_sw128(sa + a * C::A_ATOM + 32 * j), db, id1, acc);
                        tc_mma_ts(d2, alo + 32 * a + 8 * j, db, id2, acc);
                    }
                }
                tc_commit(&empty[s]);
                first = false;
                if (chunk_end(it, kt)) {
                    tc_commit(&acc_full[buf]);
                    buf ^= 1;
                    ++nchunk;
                    first = true;
                }
                if (++s == C::NS) { s = 0; ph ^= 1u; }
                if (++kt == KT) kt = 0;
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ------------------------------------------------ converters (row = TMEM lane)
        const int q = warp - 4;
        const int row = 32 * q + lane;
        const uint32_t lane_off = (uint32_t)(32 * q) << 16;
        int s = 0;
        uint32_t ph = 0;
        for (int64_t it = it0; it < it1; ++it) {
            mbar_wait(&full[s], ph, 106 * 65536 + (int)((it - it0) & 0xFFFF));
#pragma unroll
            for (int a = 0; a < C::NA; ++a) {
                const uint8_t* ta = base + s * C::STAGE_BYTES + a * C::A_ATOM + row * 128;
                uint32_t lo[32];
#pragma unroll
                for (int cc = 0; cc < 8; ++cc) {
                    const float4 v = *reinterpret_cast<const float4*>(ta + ((cc ^ (row & 7)) << 4));
                    const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const float hi = __uint_as_float(__float_as_uint(x[u]) & 0xFFFFE000u);
                        lo[4 * cc + u] = __float_as_uint(x[u] - hi);
                    }
                }
                tmem_st32(tbase + lane_off + C::LO0 + (s * C::NA + a) * 32, lo);
            }
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&lo_ready[s]);
            if (++s == C::NS) { s = 0; ph ^= 1u; }
        }
    } else if (warp >= 8) {
        // ------------------------------------------------ epilogue (row = TMEM lane)
        const int q = warp - 8;
        const int row = 32 * q + lane;
        const uint32_t lane_off = (uint32_t)(32 * q) << 16;
        double acc64[BP];
#pragma unroll
        for (int j = 0; j < BP; ++j) acc64[j] = 0.0;
        int buf = 0, nchunk = 0;
        int32_t rt = (int32_t)(it0 / sk.KT), kt = (int32_t)(it0 % sk.KT);
        int seg = c - sk.cta_of((int64_t)rt * sk.KT);
        for (int64_t it = it0; it < it1; ++it) {
            if (chunk_end(it, kt)) {
                mbar_wait(&acc_full[buf], (uint32_t)((nchunk >> 1) & 1), 105 * 65536 + nchunk);
                tc_fence_after();
                const uint32_t t1 = tbase + lane_off + C::ACC0 + buf * C::ACC_COLS;
                const uint32_t t2 = t1 + C::N1C;
#pragma unroll
                for (int c0 = 0; c0 < BP; c0 += 8) {
                    float h0[8], h1[8], l0[8];
                    tmem_ld8(t1 + c0, h0);
                    tmem_ld8(t1 + BP + c0, h1);
                    tmem_ld8(t2 + c0, l0);
                    tmem_wait_ld();
#pragma unroll
                    for (int u = 0; u < 8; ++u) acc64[c0 + u] += ((double)h0[u] + (double)h1[u]) + (double)l0[u];
                    if constexpr (C::N2 > BP) {  // b = 8: the D_lo * Y_lo rows of the second product
                        float l1[8];
                        tmem_ld8(t2 + BP + c0, l1);
                        tmem_wait_ld();
#pragma unroll
                        for (int u = 0; u < 8; ++u) acc64[c0 + u] += (double)l1[u];
                    }
                }
                tc_fence_before();
                mbar_arrive(&acc_empty[buf]);
                buf ^= 1;
                ++nchunk;
                if (it + 1 == it1 || kt + 1 == KT) {   // row-tile boundary: write the partial
                    double* out = P + (((int64_t)rt * maxseg + seg) * (int64_t)C::TM + row) * BP;
#pragma unroll
                    for (int j = 0; j < BP; ++j) {
                        out[j] = acc64[j];
                        acc64[j] = 0.0;
                    }
                }
            }
            if (++kt == KT) { kt = 0; ++rt; seg = 0; }   // a later row tile starts with this CTA
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(C::TMEM_COLS));
    }
}

}  // namespace sbmds
