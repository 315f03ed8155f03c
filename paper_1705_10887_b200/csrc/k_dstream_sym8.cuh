// A3 on the symmetric half of D with 24-bit fixed point on the int8 tensor cores
// (DESIGN.md §4). The default D stream for b in 5..32.
//
// Y2 = D Y1 reading only the 128 x 128 tiles D_IJ with I <= J, each applied as D_IJ Y1_J (to
// rows I, "N") and, for I < J, as D_IJ^T Y1_I (to rows J, "T"); D is symmetric (P:111 E,
// P:215 W = D_ll).
//
// Arithmetic. D is scaled by an exact power of two 2^sD so that |v| = |rint(D 2^sD)| <=
// 8,355,711 (just under 2^23) and stored as three balanced signed 8-bit digits,
// v = d0 2^16 + d1 2^8 + d2, d_i in [-128, 127] (k_pack_sym8, once per handle); each column c
// of the (R^-1-folded) Y1 likewise as y = y0 2^16 + y1 2^8 + y2 with scale 2^e_c (k_y8_split,
// per apply). tcgen05.mma kind::i8 multiplies digits exactly and accumulates in int32 exactly
// (|d y| <= 2^14 and a CTA's accumulator sums at most a few thousand products), keeping
// d0 [y0|y1|y2] + d1 [y0|y1] + d2 y0 in three column groups c0, c1, c2 of the accumulator; the
// product D Y1 = 2^(32-sD-e_c) (c0 + c1 2^-8 + c2 2^-16) up to the dropped d1 y2, d2 y1, d2 y2
// terms and the rounding of D and y to 24 bits: <= ~2^-23 of max|D| max|y_c| per product.
// Why int8: a kind::i8 M = 128 MMA covers K = 32 in ~44 cycles where kind::f16 covers K = 16
// in ~94 (scripts/mma_cost_probe.cu), and the three digits are 3 bytes per element of D
// instead of 4 -- the stream is HBM-bound again (the 2xFP16 kernel k_dstream_pair was
// bound by MMA instructions).
//
// One CTA does both products of a tile: for 8-bit types one SWIZZLE_128B image (row i = 128
// consecutive j in 128 bytes, 16-byte granule g at g ^ (i & 7)) is both a K-major A (N: M = i,
// K = j) and an MN-major A (T: M = j, K = i). A packed tile is three such 16 KB planes (d0,
// d1, d2); a stage is one tile (one 48 KB bulk copy) plus the 128-k slices of [y0; y1; y2] for
// J (N) and I (T) (2-D TMA, SWIZZLE_128B).
//
// Walk and accumulation: blocks of S x S tiles (block rows bi, block columns bj >= bi,
// row-major inside a block; tiles with J < I or beyond l absent); each CTA owns a contiguous,
// balanced range. Inside a block the N accumulators are the S tile rows, the T accumulators
// the S tile columns (TMEM, int32, exact); when the walk leaves a block every touched
// accumulator becomes one fp32 partial (c0 + c1/256 + c2/65536, formed in fp64) in a slot
// numbered by the host schedule; row accumulators persist across up to GN blocks of a block
// row (halving the partials), and the slots are laid out row tile by row tile, so
// k_dreduce_pair reads each row tile's partials contiguously, in slot order, in fp64 and
// undoes the scales (deterministic).
//
// Roles (192 threads): warp 0 producer, warp 1 TMEM alloc + MMA issue (converged warp, one
// elected lane issues), warps 2-5 epilogue. Each mbarrier has one producer role and one
// consumer role.
#pragma once
#include "common.cuh"
#include "k_dstream_pair.cuh"

namespace sbmds {

template <int BP>
struct Sym8Cfg {
    static constexpr int TT = 128;
    static constexpr int NB = 3 * BP;                      // B rows [y0; y1; y2]
    static constexpr int N3 = BP < 16 ? 16 : BP;           // N of the d2 product (>= 16 for M = 128)
    static constexpr int ACCW = BP < 16 ? 32 : 3 * BP;     // TMEM columns per accumulator: c0 | c1 | c2
    // Blocks of SR x SC tiles: SR row ("N") accumulators and SC column ("T") accumulators in the 512
    // TMEM columns. A T accumulator becomes a partial at every block change (1 / SR partials per
    // tile), an N accumulator after GN blocks of its block row, so the blocks are as tall as TMEM
    // allows and one tile wide: 9 x 1 at b = 16 writes 0.115 partials per tile where 5 x 5 wrote 0.204
    // (132 -> 74 MB per launch at config 4).
    static constexpr int NACC = 512 / ACCW > 17 ? 17 : 512 / ACCW;
    static constexpr int SC = 1;
    static constexpr int SR = NACC - SC;
    static constexpr int T0 = SR * ACCW;                    // first column of the T accumulators
    // a row accumulator spans at most GN blocks (GN * SC <= 256 tiles = 32,768 k): the int32 sums
    // of up to 3 digit products (|.| <= 16,129) stay below 2^31
    static constexpr int GN = 256 / SC;
    static constexpr int PLANE = TT * 128;                  // 16 KB: 128 rows x 128 int8
    static constexpr int A_BYTES = 3 * PLANE;               // 48 KB packed tile
    static constexpr int BOX_B = NB * 128;                  // 128 k of [y0; y1; y2]
    static constexpr int STAGE = A_BYTES + 2 * BOX_B;       // tile + Y_J slice + Y_I slice
    static constexpr int NS = (216 * 1024) / STAGE > 6 ? 6 : (216 * 1024) / STAGE;
    static constexpr int THREADS = 6 * 32;
    static constexpr int SMEM = NS * STAGE + 1024 + 1024;
    static_assert(STAGE % 1024 == 0 && BOX_B % 1024 == 0, "stage alignment");
    static_assert(SR >= 1 && SR <= 16 && (SR + SC) * ACCW <= 512, "tmem");
};

struct Sym8Event {
    uint32_t maskN, maskT, slotN, slotT, last, pad0, pad1, pad2;
};

__host__ __device__ constexpr uint32_t idesc_i8_s32acc(int M, int N, int a_mn) {
    // c_format S32 (2 at bit 4), a/b_format signed 8-bit (1 at bits 7, 10), A K- or MN-major
    // (bit 15), B K-major, n_dim = N >> 3, m_dim = M >> 4
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void tc_mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void tmem_ld8_u(uint32_t taddr, int (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}

// largest e with mx 2^e <= 2^22 (<= 8,355,711 with margin); 0 for mx = 0 or non-finite
__host__ __device__ __forceinline__ int i8_scale_exp(float mx) {
    if (!(mx > 0.f) || !(mx < 3.0e38f)) return 0;
    int e;
    frexpf(mx, &e);   // mx = f 2^e, f in [0.5, 1)
    return 22 - e;    // mx 2^(22-e) in [2^21, 2^22)
}

// balanced base-256 digits of an integer |v| <= 8,355,711: v = d0 2^16 + d1 2^8 + d2
__device__ __forceinline__ void digits3(int v, int& d0, int& d1, int& d2) {
    d2 = ((v + 128) & 255) - 128;
    const int v1 = (v - d2) >> 8;
    d1 = ((v1 + 128) & 255) - 128;
    d0 = (v1 - d1) >> 8;
}

template <int BP>
__global__ void __launch_bounds__(Sym8Cfg<BP>::THREADS, 1)
    k_dstream_sym8(const int8_t* __restrict__ Dt, const __grid_constant__ CUtensorMap bmap,
                   const uint32_t* __restrict__ tiles, const int64_t* __restrict__ cbeg,
                   const int* __restrict__ sbase, const int* __restrict__ smap, int NT, float* __restrict__ P,
                   int dbg_mode) {
    using C = Sym8Cfg<BP>;
    constexpr int SR = C::SR, SC = C::SC;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(base + C::NS * C::STAGE);
    uint64_t* empty = full + C::NS;
    uint64_t* ev_full = empty + C::NS;        // [2] accumulators final + event written
    uint64_t* ev_empty = ev_full + 2;         // [2] event consumed
    uint64_t* emptyN = ev_empty + 2;          // [SR] N accumulator drained
    uint64_t* emptyT = emptyN + SR;           // [SC] T accumulator drained
    Sym8Event* evq = reinterpret_cast<Sym8Event*>(emptyT + SC + ((SR + SC) & 1));   // [2] (16-byte aligned)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(evq + 2);

    pdl_trigger();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t0 = cbeg[blockIdx.x], t1 = cbeg[blockIdx.x + 1];

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&ev_full[s], 2);   // tcgen05.commit + the MMA warp's event arrive
            mbar_init(&ev_empty[s], 128);
        }
        for (int a = 0; a < SR; ++a) mbar_init(&emptyN[a], 128);
        for (int a = 0; a < SC; ++a) mbar_init(&emptyT[a], 128);
        fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;
    pdl_wait();   // Y8T (k_y8_split) and the partial slots are written by earlier kernels

    auto tile_of = [&](int64_t t, int& I, int& J) {
        const uint32_t v = __ldg(tiles + t);
        I = (int)(v >> 16);
        J = (int)(v & 0xFFFFu);
    };

    if (warp == 0) {
        // ------------------------------------------------ producer: tile (bulk) + Y slices (TMA)
        if (lane == 0) {
            prefetch_tensormap(&bmap);
            const uint64_t polb = policy_evict_last();
            int s = 0;
            uint32_t ph = 0;
            for (int64_t t = t0; t < t1; ++t) {
                int I, J;
                tile_of(t, I, J);
                mbar_wait(&empty[s], ph ^ 1u, 121 * 65536 + (int)((t - t0) & 0xFFFF));
                uint8_t* st = base + s * C::STAGE;
                mbar_arrive_expect_tx(&full[s], C::STAGE);
                bulk_load(st, Dt + upper_tile_index(I, J, NT) * C::A_BYTES, C::A_BYTES, &full[s]);
                tma_load_2d(st + C::A_BYTES, &bmap, &full[s], J * C::TT, 0, polb);             // Y_J (N)
                tma_load_2d(st + C::A_BYTES + C::BOX_B, &bmap, &full[s], I * C::TT, 0, polb);  // Y_I (T)
                if (++s == C::NS) { s = 0; ph ^= 1u; }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (whole warp, one elected lane issues)
        constexpr uint32_t id1n = idesc_i8_s32acc(C::TT, C::NB, 0), id1t = idesc_i8_s32acc(C::TT, C::NB, 1);
        constexpr uint32_t id2n = idesc_i8_s32acc(C::TT, 2 * BP, 0), id2t = idesc_i8_s32acc(C::TT, 2 * BP, 1);
        constexpr uint32_t id3n = idesc_i8_s32acc(C::TT, C::N3, 0), id3t = idesc_i8_s32acc(C::TT, C::N3, 1);
        int s = 0;
        uint32_t ph = 0, ev = 0;
        uint32_t maskN = 0, maskT = 0, usedN = 0, usedT = 0, parN = 0, parT = 0;
        uint32_t slotN = (uint32_t)sbase[2 * blockIdx.x], slotT = (uint32_t)sbase[2 * blockIdx.x + 1];
        for (int64_t t = t0; t < t1; ++t) {
            int I, J;
            tile_of(t, I, J);
            const int bi = I / SR, bj = J / SC;
            // segment ends: T (column accumulators) at every block change, N (row accumulators)
            // when the block row or the group of GN block columns changes
            bool end_seg = (t + 1 == t1), end_n = end_seg;
            if (!end_seg) {
                int I2, J2;
                tile_of(t + 1, I2, J2);
                end_seg = (I2 / SR != bi) || (J2 / SC != bj);
                end_n = (I2 / SR != bi) || ((J2 / SC) / C::GN != bj / C::GN);
            }
            const bool diag = (I == J);
            const int aN = I - bi * SR, aT = J - bj * SC;
            const uint32_t bN = 1u << aN, bT = 1u << aT;
            const bool firstN = !(maskN & bN), firstT = !diag && !(maskT & bT);
            // an accumulator's first tile in a segment waits until its previous segment's drain
            if (firstN) {
                if (usedN & bN) {
                    mbar_wait(&emptyN[aN], (parN >> aN) & 1u, 122 * 65536 + aN);
                    parN ^= bN;
                }
                usedN |= bN;
                maskN |= bN;
            }
            if (firstT) {
                if (usedT & bT) {
                    mbar_wait(&emptyT[aT], (parT >> aT) & 1u, 123 * 65536 + aT);
                    parT ^= bT;
                }
                usedT |= bT;
                maskT |= bT;
            }
            mbar_wait(&full[s], ph, 124 * 65536 + (int)((t - t0) & 0xFFFF));
            tc_fence_after();
            const uint32_t sa = smem_u32(base + s * C::STAGE);
            const uint32_t sbN = sa + C::A_BYTES, sbT = sbN + C::BOX_B;
            const uint32_t dN = tbase + (uint32_t)(aN * C::ACCW), dT = tbase + (uint32_t)(C::T0 + aT * C::ACCW);
            if (elect_one()) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {   // K = 32 per MMA
                    if (dbg_mode & 1) break;     // diagnostics: stream only
                    // N: A = plane p, K-major (k = column j: 32 bytes per step inside the 128-byte rows)
                    const uint64_t bj0 = umma_desc_sw128(sbN + 32 * j, 16, 1024);
                    tc_mma_i8(dN, umma_desc_sw128(sa + 32 * j, 16, 1024), bj0, id1n, (firstN && j == 0) ? 0u : 1u);
                    tc_mma_i8(dN + BP, umma_desc_sw128(sa + C::PLANE + 32 * j, 16, 1024), bj0, id2n, 1u);
                    tc_mma_i8(dN + 2 * BP, umma_desc_sw128(sa + 2 * C::PLANE + 32 * j, 16, 1024), bj0, id3n, 1u);
                    if (!diag) {
                        // T: the same planes, MN-major (k = row i: 32 rows = 4 KB per step)
                        const uint64_t bi0 = umma_desc_sw128(sbT + 32 * j, 16, 1024);
                        tc_mma_i8(dT, umma_desc_sw128(sa + 4096 * j, 16384, 1024), bi0, id1t,
                                  (firstT && j == 0) ? 0u : 1u);
                        tc_mma_i8(dT + BP, umma_desc_sw128(sa + C::PLANE + 4096 * j, 16384, 1024), bi0, id2t, 1u);
                        tc_mma_i8(dT + 2 * BP, umma_desc_sw128(sa + 2 * C::PLANE + 4096 * j, 16384, 1024), bi0, id3t, 1u);
                    }
                }
                tc_commit(&empty[s]);
            }
            __syncwarp();
            if (++s == C::NS) { s = 0; ph ^= 1u; }
            if (end_seg) {
                const int eb = ev & 1;
                mbar_wait(&ev_empty[eb], ((ev >> 1) & 1u) ^ 1u, 125 * 65536 + (int)(ev & 0xFFFF));
                const uint32_t mN = end_n ? maskN : 0u;
                if (elect_one()) {
                    evq[eb] = Sym8Event{mN, maskT, slotN, slotT, (t + 1 == t1) ? 1u : 0u, 0u, 0u, 0u};
                    tc_commit(&ev_full[eb]);
                    mbar_arrive(&ev_full[eb]);
                }
                __syncwarp();
                slotN += (uint32_t)__popc(mN);
                slotT += (uint32_t)__popc(maskT);
                if (end_n) maskN = 0;
                maskT = 0;
                ++ev;
            }
        }
    } else {
        // ------------------------------------------------ epilogue warps 2-5 (TMEM lane = output row)
        const int qd = warp & 3;
        const int ln = 32 * qd + lane;
        const uint32_t lane_off = (uint32_t)(32 * qd) << 16;
        auto drain = [&](uint32_t col, uint32_t slot, uint64_t* emp) {
            float out[BP];
#pragma unroll
            for (int c0 = 0; c0 < BP; c0 += 8) {
                int g0[8], g1[8], g2[8];
                tmem_ld8_u(tbase + lane_off + col + c0, g0);
                tmem_ld8_u(tbase + lane_off + col + BP + c0, g1);
                tmem_ld8_u(tbase + lane_off + col + 2 * BP + c0, g2);
                tmem_wait_ld();
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    out[c0 + u] = (float)((double)g0[u] + (double)g1[u] * (1.0 / 256.0) + (double)g2[u] * (1.0 / 65536.0));
            }
            tc_fence_before();
            mbar_arrive(emp);
            float4* dst = reinterpret_cast<float4*>(P + ((int64_t)__ldg(smap + slot) * C::TT + ln) * BP);
#pragma unroll
            for (int c0 = 0; c0 < BP; c0 += 4) dst[c0 / 4] = make_float4(out[c0], out[c0 + 1], out[c0 + 2], out[c0 + 3]);
        };
        for (uint32_t ev = 0; t0 < t1; ++ev) {
            const int eb = ev & 1;
            mbar_wait(&ev_full[eb], (ev >> 1) & 1u, 126 * 65536 + (int)(ev & 0xFFFF));
            tc_fence_after();
            const Sym8Event e = evq[eb];
            uint32_t slot = e.slotN;
            for (uint32_t bits = e.maskN; bits; bits &= bits - 1) {
                const int a = __ffs(bits) - 1;
                drain((uint32_t)(a * C::ACCW), slot++, &emptyN[a]);
            }
            slot = e.slotT;
            for (uint32_t bits = e.maskT; bits; bits &= bits - 1) {
                const int a = __ffs(bits) - 1;
                drain((uint32_t)(C::T0 + a * C::ACCW), slot++, &emptyT[a]);
            }
            mbar_arrive(&ev_empty[eb]);
            if (e.last) break;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
    }
}

// Pack the upper tiles of row-major D (block upper triangle present), scaled by 2^sD with
// sD = i8_scale_exp(max |D|), as three digit planes of 128 x 128 int8 in the swizzled image
// above, 48 KB per tile at upper_tile_index(I, J); zero outside l. Block 0 also records the
// exponent k_dreduce_pair undoes (sD - 32, see below).
__global__ void __launch_bounds__(256) k_pack_sym8(const float* __restrict__ D, int64_t ldD, int64_t l,
                                                   const uint32_t* __restrict__ tiles, int64_t NT, int64_t ntiles,
                                                   const unsigned int* __restrict__ dmax, int* __restrict__ dexp,
                                                   int8_t* __restrict__ Dt) {
    const int sD = i8_scale_exp(__uint_as_float(*dmax));
    // the partials carry c0 + c1/256 + c2/65536 = D Y1 2^(sD + e_c) / 2^32 (the leading digits
    // d0, y0 have place value 2^16 each): k_dreduce_pair multiplies by 2^-(dexp + e_c)
    if (blockIdx.x == 0 && threadIdx.x == 0) *dexp = sD - 32;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint32_t v = tiles[t];
        const int I = (int)(v >> 16), J = (int)(v & 0xFFFFu);
        const int64_t r0 = (int64_t)I * 128, c0 = (int64_t)J * 128;
        int8_t* out = Dt + upper_tile_index(I, J, (int)NT) * (3 * 16384);
        for (int e = threadIdx.x; e < 128 * 8; e += 256) {
            const int r = e >> 3, c16 = (e & 7) * 16;   // 16 consecutive columns (one granule) of row r
            const int64_t gr = r0 + r;
            __align__(16) int8_t p0[16], p1[16], p2[16];
            // 16-byte loads (ldD % 4 == 0, the granule starts at a multiple of 16 columns; columns
            // in [l, ldD) are padding and read as 0 below, the rows past l are not read)
            float xv[16];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int64_t gc = c0 + c16 + 4 * q;
                float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
                if (gr < l && gc < l) f = __ldcs(reinterpret_cast<const float4*>(D + gr * ldD + gc));
                xv[4 * q] = f.x;
                xv[4 * q + 1] = f.y;
                xv[4 * q + 2] = f.z;
                xv[4 * q + 3] = f.w;
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int64_t gc = c0 + c16 + u;
                const float x = gc < l ? ldexpf(xv[u], sD) : 0.f;
                int d0, d1, d2;
                digits3(__float2int_rn(x), d0, d1, d2);
                p0[u] = (int8_t)d0;
                p1[u] = (int8_t)d1;
                p2[u] = (int8_t)d2;
            }
            const int off = r * 128 + (((c16 >> 4) ^ (r & 7)) << 4);
            *reinterpret_cast<uint4*>(out + off) = *reinterpret_cast<const uint4*>(p0);
            *reinterpret_cast<uint4*>(out + 16384 + off) = *reinterpret_cast<const uint4*>(p1);
            *reinterpret_cast<uint4*>(out + 32768 + off) = *reinterpret_cast<const uint4*>(p2);
        }
    }
}

// Per-column max |y| and sum of y^2 of Y1 (l x bp, columns < b): the standalone apply's check
// that the per-column fixed point of the int8 stream keeps the bulk of each column (sbmds.cu
// apply_device; DESIGN.md §4 precision contract). out: [0, 64) max bits, then 64 doubles.
__global__ void __launch_bounds__(256) k_ycheck(int64_t l, int b, int bp, const float* __restrict__ Y1,
                                                unsigned int* __restrict__ out) {
    __shared__ float smx[256];
    __shared__ double sss[256];
    const int rb = 256 / bp;
    const int r = threadIdx.x / bp, c = threadIdx.x % bp;
    float m = 0.f;
    double ss = 0.0;
    if (r < rb && c < b)
        for (int64_t k = (int64_t)blockIdx.x * rb + r; k < l; k += (int64_t)gridDim.x * rb) {
            const float v = Y1[k * bp + c];
            m = fmaxf(m, fabsf(v));
            ss += (double)v * v;
        }
    smx[threadIdx.x] = m;
    sss[threadIdx.x] = ss;
    __syncthreads();
    if (r == 0 && c < b) {
        for (int q = 1; q < rb; ++q) {
            m = fmaxf(m, smx[q * bp + c]);
            ss += sss[q * bp + c];
        }
        atomicMax(out + c, __float_as_uint(m));
        atomicAdd(reinterpret_cast<double*>(out + 64) + c, ss);
    }
}

// folded Y1 (Y1f, l_pad x bp) -> Y8T (3bp x l_pad int8): rows [y0; y1; y2], the balanced digits
// of rint(y 2^e_c), e_c = i8_scale_exp(max |column c|)
__global__ void __launch_bounds__(256) k_y8_split(int64_t lpad, int bp, const float* __restrict__ Y1f,
                                                  const unsigned int* __restrict__ cmax, int8_t* __restrict__ Y8T,
                                                  int* __restrict__ yexp) {
    pdl_trigger();
    pdl_wait();
    const int rb = 256 / bp;
    const int r = threadIdx.x % rb, c = threadIdx.x / rb;   // consecutive threads: consecutive k
    const int e = i8_scale_exp(__uint_as_float(cmax[c]));
    if (blockIdx.x == 0 && r == 0) yexp[c] = e;
    for (int64_t k = (int64_t)blockIdx.x * rb + r; k < lpad; k += (int64_t)gridDim.x * rb) {
        int d0, d1, d2;
        digits3(__float2int_rn(ldexpf(Y1f[k * bp + c], e)), d0, d1, d2);
        Y8T[(int64_t)c * lpad + k] = (int8_t)d0;
        Y8T[(int64_t)(bp + c) * lpad + k] = (int8_t)d1;
        Y8T[(int64_t)(2 * bp + c) * lpad + k] = (int8_t)d2;
    }
}

}  // namespace sbmds
