// NEXT-1: stream only the upper triangle of the symmetric D_ll.
//
// D = D^T ("d_M is symmetric"; W_ij = d(b_i, b_j)), so every
// 128 x 128 tile D_IJ with I < J serves two products:
//     Y2_I += D_IJ   Y1_J     (the row strip I, accumulated in TMEM along the strip)
//     Y2_J += D_IJ^T Y1_I     (one 128 x bp fp32 partial per tile, summed in fixed order later)
// and a diagonal tile D_II only the first. D is read once per pair: 2 l^2 bytes instead of
// 4 l^2, plus 2 * 4 * 128 * bp bytes of partial traffic per off-diagonal tile.
//
// Both products use the 3xTF32 split of k_dstream_tc.cuh. The normal product reads D_hi from
// the K-major SWIZZLE_128B tile (SS) and D_lo from TMEM (TS). The transposed product needs the
// tile MN-major, which for 32-bit operands wants a different (32 B atom) swizzle than the
// K-major tile, so its D_hi^T and D_lo^T (lane = j) are both written to TMEM by a second
// converter group that reads the tile column-wise (conflict-free: a warp reads one 128 B row
// of one atom) and both transposed MMAs are TS.
//
// CTA: one per SM, stream-K over the RT(RT+1)/2 upper tiles, strip-major.
//   warp 0      TMA: D tile (4 atoms, 64 KB) + B_J = [Y_hi; Y_lo]_J per tile; B_I per strip
//   warp 1      TMEM alloc; lane 0 issues 32 + 32 MMAs per tile and the commits
//   warps 4-7   normal D_lo (row-wise) + lagged drain of the strip accumulator (fp64)
//   warps 8-11  transposed D_lo (column-wise) + drain of the per-tile transposed partial
// TMEM (512 columns): accN (64) + accT (64) + D_lo (128) + D_hi^T (128) + D_lo^T (128).
#pragma once
#include "common.cuh"
#include "k_dstream.cuh"
#include "k_dstream_tc.cuh"

namespace sbmds {

template <int BP>
struct SymCfg {
    static constexpr int T = 128;                       // tile edge (rows i, cols j)
    static constexpr int NA = 4;                        // 32-k chunks (swizzle atoms) per tile
    static constexpr int NB = 2 * BP;                   // [Y_hi; Y_lo] rows
    static constexpr int N1 = NB;
    static constexpr int N2 = BP < 16 ? 16 : BP;
    static constexpr int N1C = (N1 + 31) / 32 * 32;
    static constexpr int N2C = (N2 + 31) / 32 * 32;
    static constexpr int ACC = N1C + N2C;               // one accumulator (hi and lo products)
    static constexpr int A_ATOM = T * 128;              // 16 KB
    static constexpr int A_BYTES = NA * A_ATOM;         // 64 KB
    static constexpr int B_ATOM = NB * 128;
    static constexpr int B_BYTES = NA * B_ATOM;         // B_J or B_I (K = 128)
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int NS = 2;                        // smem stages (tiles)
    static constexpr int TMEM_COLS = 512;
    static constexpr int ACCN0 = 0;                     // strip accumulator
    static constexpr int ACCT0 = ACC;                   // transposed accumulators [2]
    static constexpr int RING0 = 3 * ACC;               // chunk slots: [D_lo | D_hi^T | D_lo^T] x 32 cols
    static constexpr int SLOT = 96;
    static constexpr int NSLOT = (TMEM_COLS - RING0) / SLOT;
    static constexpr int KC = 4;                        // tiles per strip-accumulator drain (512 k)
    static constexpr int THREADS = 12 * 32;
    static constexpr int SMEM = NS * STAGE_BYTES + 2 * B_BYTES + 1024 + 512;
    static_assert(NSLOT >= 2, "tmem ring");
    static_assert(SMEM <= 227 * 1024, "smem budget");
};

struct SymSched {
    int64_t NT;       // tiles in the upper triangle
    int RT;           // row/col tiles
    int grid;
    __host__ __device__ int64_t beg(int c) const { return (int64_t)c * NT / grid; }
    // first linear index of strip I: I*RT - I(I-1)/2
    __host__ __device__ int64_t strip0(int I) const { return (int64_t)I * RT - (int64_t)I * (I - 1) / 2; }
    __host__ __device__ void decode(int64_t x, int& I, int& J) const {
        int lo = 0, hi = RT - 1;
        while (lo < hi) {   // largest I with strip0(I) <= x
            const int mid = (lo + hi + 1) >> 1;
            if (strip0(mid) <= x) lo = mid; else hi = mid - 1;
        }
        I = lo;
        J = I + (int)(x - strip0(I));
    }
    __host__ __device__ int cta_of(int64_t x) const {
        int c = (int)((x * grid) / NT);
        while (c + 1 < grid && beg(c + 1) <= x) ++c;
        while (c > 0 && beg(c) > x) --c;
        return c;
    }
};

// Transposed partial index: output tile J, source strip I < J.
__host__ __device__ inline int64_t pt_index(int J, int I) { return (int64_t)J * (J - 1) / 2 + I; }

template <int BP>
__global__ void __launch_bounds__(SymCfg<BP>::THREADS, 1)
    k_dstream_sym(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap, SymSched sk,
                  int maxseg, double* __restrict__ P, float* __restrict__ PT) {
    using C = SymCfg<BP>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* bI = base + C::NS * C::STAGE_BYTES;                        // [2] B_I buffers
    uint64_t* bars = reinterpret_cast<uint64_t*>(bI + 2 * C::B_BYTES);
    uint64_t* full = bars;                          // [NS] tile landed
    uint64_t* empty = full + C::NS;                 // [NS] tile consumed
    uint64_t* bi_full = empty + C::NS;              // [2]
    uint64_t* bi_empty = bi_full + 2;               // [2]
    uint64_t* slot_ready = bi_empty + 2;            // [NSLOT] chunk operands in TMEM (256 arrivals)
    uint64_t* slot_free = slot_ready + C::NSLOT;    // [NSLOT] chunk MMAs done
    uint64_t* accN_full = slot_free + C::NSLOT;     // 1
    uint64_t* accN_empty = accN_full + 1;           // 1
    uint64_t* accT_full = accN_empty + 1;           // [2]
    uint64_t* accT_empty = accT_full + 2;           // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accT_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x;
    const int64_t it0 = sk.beg(c), it1 = sk.beg(c + 1);
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&bi_full[b], 1);
            mbar_init(&bi_empty[b], 1);
            mbar_init(&accT_full[b], 1);
            mbar_init(&accT_empty[b], 128);
        }
        for (int k = 0; k < C::NSLOT; ++k) { mbar_init(&slot_ready[k], 256); mbar_init(&slot_free[k], 1); }
        mbar_init(accN_full, 1);
        mbar_init(accN_empty, 128);
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
    int I0 = 0, J0 = 0;
    if (it0 < it1) sk.decode(it0, I0, J0);
    const int RT = sk.RT;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            prefetch_tensormap(&amap);
            prefetch_tensormap(&bmap);
            const uint64_t pol = policy_evict_first();
            const uint64_t polb = policy_evict_last();
            int s = 0, I = I0, J = J0, nstrip = 0;
            uint32_t ph = 0;
            for (int64_t it = it0; it < it1; ++it) {
                if (it == it0 || J == I) {   // new strip: its B_I (K = rows of strip I)
                    const int bb = nstrip & 1;
                    mbar_wait(&bi_empty[bb], (uint32_t)(((nstrip >> 1) & 1) ^ 1));
                    mbar_arrive_expect_tx(&bi_full[bb], C::B_BYTES);
#pragma unroll
                    for (int a = 0; a < C::NA; ++a)
                        tma_load_2d(bI + bb * C::B_BYTES + a * C::B_ATOM, &bmap, &bi_full[bb], I * C::T + 32 * a, 0, polb);
                    ++nstrip;
                }
                mbar_wait(&empty[s], ph ^ 1u);
                uint8_t* st = base + s * C::STAGE_BYTES;
                mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
#pragma unroll
                for (int a = 0; a < C::NA; ++a) {
                    tma_load_2d(st + a * C::A_ATOM, &amap, &full[s], J * C::T + 32 * a, I * C::T, pol);
                    tma_load_2d(st + C::A_BYTES + a * C::B_ATOM, &bmap, &full[s], J * C::T + 32 * a, 0, polb);
                }
                if (++s == C::NS) { s = 0; ph ^= 1u; }
                if (++J == RT) { ++I; J = I; }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            constexpr uint32_t id1 = idesc_tf32_f32acc(C::T, C::N1);
            constexpr uint32_t id2 = idesc_tf32_f32acc(C::T, C::N2);
            int s = 0, I = I0, J = J0, nstrip = 0, nchunkN = 0, ntrans = 0, kcount = 0;
            uint32_t ph = 0;
            int64_t g = 0;   // global chunk counter (TMEM ring)
            bool firstN = true;
            for (int64_t it = it0; it < it1; ++it) {
                const bool new_strip = (it == it0 || J == I);
                if (new_strip) ++nstrip;
                const int bb = (nstrip - 1) & 1;
                const bool trans = J > I;
                const int bt = ntrans & 1;
                if (firstN) {
                    mbar_wait(accN_empty, (uint32_t)((nchunkN & 1) ^ 1));
                    tc_fence_after();
                }
                if (trans) {
                    mbar_wait(&accT_empty[bt], (uint32_t)(((ntrans >> 1) & 1) ^ 1));
                    tc_fence_after();
                }
                mbar_wait(&full[s], ph);
                mbar_wait(&bi_full[bb], (uint32_t)(((nstrip - 1) >> 1) & 1));
                const uint32_t sa = smem_u32(base + s * C::STAGE_BYTES);
                const uint32_t sbJ = sa + C::A_BYTES;
                const uint32_t sbI = smem_u32(bI + bb * C::B_BYTES);
                const uint32_t dN1 = tbase + C::ACCN0, dN2 = dN1 + C::N1C;
                const uint32_t dT1 = tbase + C::ACCT0 + bt * C::ACC, dT2 = dT1 + C::N1C;
#pragma unroll 1
                for (int a = 0; a < C::NA; ++a, ++g) {
                    const int slot = (int)(g % C::NSLOT);
                    mbar_wait(&slot_ready[slot], (uint32_t)((g / C::NSLOT) & 1));
                    tc_fence_after();
                    const uint32_t ring = tbase + C::RING0 + slot * C::SLOT;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t acc = (firstN && a == 0 && j == 0) ? 0u : 1u;
                        const uint64_t dbJ = umma_desc_k_sw128(sbJ + a * C::B_ATOM + 32 * j);
                        tc_mma_ss(dN1, umma_desc_k_sw128(sa + a * C::A_ATOM + 32 * j), dbJ, id1, acc);
                        tc_mma_ts(dN2, ring + 8 * j, dbJ, id2, acc);
                    }
                    if (trans) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) {   // K = i in [32a, 32a + 32), 8 rows per MMA
                            const uint32_t acc = (a == 0 && j == 0) ? 0u : 1u;
                            const uint64_t dbI = umma_desc_k_sw128(sbI + a * C::B_ATOM + 32 * j);
                            tc_mma_ts(dT1, ring + 32 + 8 * j, dbI, id1, acc);
                            tc_mma_ts(dT2, ring + 64 + 8 * j, dbI, id2, acc);
                        }
                    }
                    tc_commit(&slot_free[slot]);
                }
                tc_commit(&empty[s]);
                if (trans) {
                    tc_commit(&accT_full[bt]);
                    ++ntrans;
                }
                firstN = false;
                ++kcount;
                const bool strip_end = (it + 1 == it1) || (J + 1 == RT);
                if (strip_end || kcount == C::KC) {
                    tc_commit(accN_full);
                    ++nchunkN;
                    firstN = true;
                    kcount = 0;
                }
                if (strip_end) tc_commit(&bi_empty[bb]);
                if (++s == C::NS) { s = 0; ph ^= 1u; }
                if (++J == RT) { ++I; J = I; }
            }
        }
    } else if (warp >= 4) {
        const int grp = (warp - 4) / 4;          // 0: normal D_lo (rows), 1: transposed D_hi^T, D_lo^T (columns)
        const int q = (warp - 4) % 4;            // TMEM lane quarter
        const int row = 32 * q + lane;           // tile row (grp 0) or tile column (grp 1)
        const uint32_t lane_off = (uint32_t)(32 * q) << 16;
        double accN[BP];
#pragma unroll
        for (int j = 0; j < BP; ++j) accN[j] = 0.0;
        int s = 0, I = I0, J = J0, nchunkN = 0, ntrans = 0, kcount = 0;
        uint32_t ph = 0;
        int64_t g = 0;
        int seg = c - sk.cta_of(sk.strip0(I0));
        bool pend = false;   // grp 1: a finished transposed tile waiting to be drained
        int pend_n = 0, pendI = 0, pendJ = 0;
        auto drain_trans = [&]() {
            const int pb = pend_n & 1;
            mbar_wait(&accT_full[pb], (uint32_t)((pend_n >> 1) & 1));
            tc_fence_after();
            const uint32_t t1 = tbase + lane_off + C::ACCT0 + pb * C::ACC, t2 = t1 + C::N1C;
            float* out = PT + (pt_index(pendJ, pendI) * C::T + row) * BP;
#pragma unroll
            for (int c0 = 0; c0 < BP; c0 += 8) {
                float h0[8], h1[8], l0[8], o[8];
                tmem_ld8(t1 + c0, h0);
                tmem_ld8(t1 + BP + c0, h1);
                tmem_ld8(t2 + c0, l0);
                tmem_wait_ld();
#pragma unroll
                for (int u = 0; u < 8; ++u) o[u] = (h0[u] + h1[u]) + l0[u];
                if constexpr (C::N2 > BP) {
                    float l1[8];
                    tmem_ld8(t2 + BP + c0, l1);
                    tmem_wait_ld();
#pragma unroll
                    for (int u = 0; u < 8; ++u) o[u] += l1[u];
                }
#pragma unroll
                for (int u = 0; u < 8; u += 4)
                    *reinterpret_cast<float4*>(out + c0 + u) = make_float4(o[u], o[u + 1], o[u + 2], o[u + 3]);
            }
            tc_fence_before();
            mbar_arrive(&accT_empty[pb]);
            pend = false;
        };
        for (int64_t it = it0; it < it1; ++it) {
            const bool trans = J > I;
            mbar_wait(&full[s], ph);
            const uint8_t* st = base + s * C::STAGE_BYTES;
#pragma unroll 1
            for (int a = 0; a < C::NA; ++a, ++g) {
                const int slot = (int)(g % C::NSLOT);
                mbar_wait(&slot_free[slot], (uint32_t)(((g / C::NSLOT) & 1) ^ 1));
                const uint32_t ring = tbase + lane_off + C::RING0 + slot * C::SLOT;
                if (grp == 0) {
                    const uint8_t* ta = st + a * C::A_ATOM + row * 128;
                    uint32_t lo[32];
#pragma unroll
                    for (int cc = 0; cc < 8; ++cc) {
                        const float4 v = *reinterpret_cast<const float4*>(ta + ((cc ^ (row & 7)) << 4));
                        const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            lo[4 * cc + u] = __float_as_uint(x[u] - __uint_as_float(__float_as_uint(x[u]) & 0xFFFFE000u));
                    }
                    tmem_st32(ring, lo);
                    tmem_wait_st();
                } else if (trans) {
                    // column j = row (TMEM lane) of atom q: element (i, j) sits in row i, chunk
                    // ((j % 32) / 4) ^ (i % 8), word j % 4 of atom q; this chunk holds i in [32a, 32a+32)
                    const uint8_t* ta = st + q * C::A_ATOM + ((lane & 3) << 2);
                    const int ch = lane >> 2;
                    uint32_t hi[32], lo[32];
#pragma unroll
                    for (int u = 0; u < 32; ++u) {
                        const int i = 32 * a + u;
                        const float x = *reinterpret_cast<const float*>(ta + i * 128 + ((ch ^ (i & 7)) << 4));
                        hi[u] = __float_as_uint(x);   // the MMA reads its tf32 part
                        lo[u] = __float_as_uint(x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u));
                    }
                    tmem_st32(ring + 32, hi);
                    tmem_st32(ring + 64, lo);
                    tmem_wait_st();
                }
                tc_fence_before();
                mbar_arrive(&slot_ready[slot]);
            }
            if (grp == 0) {
                ++kcount;
                const bool strip_end = (it + 1 == it1) || (J + 1 == RT);
                if (strip_end || kcount == C::KC) {
                    // drain the strip accumulator now (the MMA waits for it before the next chunk)
                    mbar_wait(accN_full, (uint32_t)(nchunkN & 1));
                    tc_fence_after();
                    const uint32_t t1 = tbase + lane_off + C::ACCN0, t2 = t1 + C::N1C;
#pragma unroll
                    for (int c0 = 0; c0 < BP; c0 += 8) {
                        float h0[8], h1[8], l0[8];
                        tmem_ld8(t1 + c0, h0);
                        tmem_ld8(t1 + BP + c0, h1);
                        tmem_ld8(t2 + c0, l0);
                        tmem_wait_ld();
#pragma unroll
                        for (int u = 0; u < 8; ++u) accN[c0 + u] += ((double)h0[u] + (double)h1[u]) + (double)l0[u];
                        if constexpr (C::N2 > BP) {
                            float l1[8];
                            tmem_ld8(t2 + BP + c0, l1);
                            tmem_wait_ld();
#pragma unroll
                            for (int u = 0; u < 8; ++u) accN[c0 + u] += (double)l1[u];
                        }
                    }
                    tc_fence_before();
                    mbar_arrive(accN_empty);
                    ++nchunkN;
                    kcount = 0;
                    if (strip_end) {
                        double* out = P + (((int64_t)I * maxseg + seg) * (int64_t)C::T + row) * BP;
#pragma unroll
                        for (int j = 0; j < BP; ++j) { out[j] = accN[j]; accN[j] = 0.0; }
                    }
                }
            } else {
                if (pend) drain_trans();   // the previous transposed tile (its MMAs precede this tile's)
                if (trans) {
                    pend = true;
                    pend_n = ntrans;
                    pendI = I;
                    pendJ = J;
                    ++ntrans;
                }
            }
            if (++s == C::NS) { s = 0; ph ^= 1u; }
            if (++J == RT) { ++I; J = I; seg = 0; }
        }
        if (grp == 1 && pend) drain_trans();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(C::TMEM_COLS));
    }
}

// Y2 rows of tile J = (strip partials of J in CTA order) + (transposed partials from strips
// I < J in ascending I), then t = w^T Y2 (fp64, block partials + last block).
__global__ void __launch_bounds__(256) k_dreduce_sym(int64_t l, int bp, int b, SymSched sk, int maxseg,
                                                     const double* __restrict__ P, const float* __restrict__ PT,
                                                     const double* __restrict__ w, float* __restrict__ Y2,
                                                     double* __restrict__ tpart, double* __restrict__ t,
                                                     unsigned int* __restrict__ counter) {
    __shared__ double red[256];
    const int rows_per_blk = 256 / bp;
    const int tid = threadIdx.x;
    const int cidx = tid % bp, rloc = tid / bp;
    double acc_t = 0.0;
    for (int64_t r0 = (int64_t)blockIdx.x * rows_per_blk; r0 < l; r0 += (int64_t)gridDim.x * rows_per_blk) {
        const int64_t r = r0 + rloc;
        if (rloc < rows_per_blk && r < l) {
            const int J = (int)(r / 128);
            const int rr = (int)(r - (int64_t)J * 128);
            const int c0 = sk.cta_of(sk.strip0(J));
            const int c1 = sk.cta_of(sk.strip0(J) + (sk.RT - J) - 1);
            double v = 0.0;
            for (int seg = 0; seg <= c1 - c0; ++seg)
                v += P[(((int64_t)J * maxseg + seg) * 128 + rr) * bp + cidx];
            const float* pt = PT + (pt_index(J, 0) * 128 + rr) * bp + cidx;
            int I = 0;
            for (; I + 16 <= J; I += 16) {   // 16 loads in flight, added in ascending I
                float x[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) x[u] = __ldg(pt + (int64_t)(I + u) * 128 * bp);
#pragma unroll
                for (int u = 0; u < 16; ++u) v += (double)x[u];
            }
            for (; I < J; ++I) v += (double)pt[(int64_t)I * 128 * bp];
            Y2[r * bp + cidx] = (float)v;
            if (cidx < b) acc_t += w[r] * v;
        }
    }
    red[tid] = (rloc < rows_per_blk) ? acc_t : 0.0;
    __syncthreads();
    if (tid < bp) {
        double v = 0.0;
        for (int q = 0; q < rows_per_blk; ++q) v += red[q * bp + tid];
        tpart[blockIdx.x * kMaxB + tid] = v;
    }
    if (last_block_done(counter)) {
        if (tid < bp) t[tid] = ordered_sum(tpart + tid, gridDim.x, kMaxB);
        if (tid == 0) *counter = 0;
    }
}

}  // namespace sbmds
