// The sparse products on the int8 tensor cores ("tensor-core sparse step"): inside
// sbmds_eigs A5 of this apply, the Gram step and A2 of the next apply in one kernel per block of
// S; in the standalone sbmds_apply A2 and A5 as two passes of the same kernel.
//
// Inside sbmds_eigs the block Y = B~X formed by A5 (Y = -1/2 (S Y2 - 1 t^T)
// "left-multiplying by P", PAPER.md:113 the -1/2) is consumed by the Gram step and by the next
// apply's A2 (S^T Y, "right-multiplying by P^T"), both linear in Y's rows. S is
// local: a block of <= 128 consecutive vertices (row range brow0[B] ..
// brow0[B + 1]; 128 rows unless the build split it) touches d_B <= 128 landmarks (config 4: 115
// on average), so the block's slice S_B (128 x d_B) is stored as a DENSE image and both
// products become tensor-core GEMMs with no gathers at all:
//   N:  Y_B   = S_B   Y2[dict_B]    (M = 128 rows,  K = d_pad, N = 3 b)   A K-major
//   T:  P1_B  = S_B^T Y_B           (M = 128 dict,  K = 128 rows, N = 3 b) A MN-major
// One shared-memory image serves both: with the no-swizzle core-matrix layout (core = 8 rows x
// 16 contiguous bytes; core (row group rg, column chunk kc) at (kc * 16 + rg) * 128 bytes) an
// 8-bit image is a K-major A for N (LBO = 2048 along K, SBO = 128 along M) and an MN-major A
// for T (LBO = 128 along K, SBO = 2048 along M) -- scripts/sp8_probe.cu checks both.
//
// Arithmetic (as k_dstream_sym8.cuh): S_B is scaled by 2^eS_B (per block) and stored as three
// balanced signed digits per entry (3 planes, k_sp8_build, once per handle); the B operands are
// digitised on the fly: Y2 with one scale 2^ey_c per column (from its column maxima), Y_B with
// one scale per column for the whole launch (from an a-priori bound on |Y|, so the epilogue
// warps exchange nothing). kind::i8 products and int32 sums are exact; the accumulator's four
// column groups give c0 + c1/256 + (c2 + c3/256)/65536, undone in fp32 (error <= ~2^-23 of the
// scaled maxima per product, the same bound as the D stream).
//
// Roles (persistent CTAs of 17 warps, contiguous block ranges):
//   warp 0       producer: the block's image (one bulk copy, 384 d_pad bytes) into a 3-stage ring,
//                the B operand of N (16-byte rows of Y2's digit planes, cp.async) and the block's
//                row-sum deviations; TONLY: the block's rows of X instead
//   warp 1       issues the N products (and owns the TMEM allocation); warp 16 the T products
//                (and, GRAM8, the Gram MMAs Yd^T [Yd | 1] into one accumulator per CTA)
//   warps 2-9    epilogue A: N accumulator -> Y rows (HBM), Y_B digits -> B operand of T
//                (+ fp32 rows for the FP64 Gram warps in the variants that use them)
//   warps 10-13  group B: T accumulator -> P1 partials; at the end (GRAM8) the Gram accumulator
//   warps 14-15  group C: G = Y^T Y, 1^T Y and (Rayleigh-Ritz steps) H' = Y_prev^T Y on the FP64
//                tensor cores; idle in the GRAM8 / TONLY variants
// Every sum has a fixed order (or is an exact integer sum): Y, P1 and the Grams are bitwise
// reproducible.
#pragma once
#include "common.cuh"
#include "k_dstream_sym8.cuh"
#include "k_small.cuh"
#include "k_dstream_pair.cuh"
#include <cooperative_groups.h>

namespace sbmds {

constexpr int kSp8RB = 128;   // rows per block (the MMA M of N)
constexpr int kSp8DK = 128;   // largest padded dictionary (the MMA M of T)

__device__ __forceinline__ uint64_t umma_desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

// byte offset of (row r, column k) in a core-matrix image with `rgroups` 8-row groups per
// 16-column chunk: ((k / 16) * rgroups + r / 8) * 128 + (r % 8) * 16 + k % 16
__host__ __device__ __forceinline__ int sp8_off(int r, int k, int rgroups) {
    return (((k >> 4) * rgroups + (r >> 3)) << 7) + ((r & 7) << 4) + (k & 15);
}

__host__ __device__ __forceinline__ int sp8_dpad(int d) { return d <= 32 ? 32 : (d + 31) / 32 * 32; }

// B operands are MN-major core-matrix images: core = 8 K-rows x 16 contiguous N bytes, core
// (K group kg, N group ng) at (kg * NB/16 + ng) * 128 (LBO = K stride, SBO = 128 along N;
// scripts/sp8_probe.cu mode 2). A thread owning K-row k writes digit plane p's 16 columns as
// one 16-byte store at sp8_boff(k, p).
template <int NB>
__device__ __forceinline__ int sp8_boff(int k, int p) {
    return (((k >> 3) * (NB / 16) + p) << 7) + ((k & 7) << 4);
}

__host__ __device__ constexpr uint32_t idesc_i8_bmn(int M, int N, int a_mn) {
    return idesc_i8_s32acc(M, N, a_mn) | (1u << 16);   // B MN-major
}

// 2^e as two normal floats whose product is 2^e (|e| <= 252): x 2^e = (x f.x) f.y, exact
// while the result is normal, no branches
__device__ __forceinline__ float2 pow2f2(int e) {
    const int e1 = e >> 1, e2 = e - e1;
    return make_float2(__int_as_float((127 + e1) << 23), __int_as_float((127 + e2) << 23));
}

// exact int -> float for |g| <= 2^22 without a conversion instruction (1.5 2^23 magic)
__device__ __forceinline__ float i22_to_f(int g) { return __int_as_float(0x4B400000 + g) - 12582912.0f; }

// 2^e as a float, e clamped to the normal range (a column whose maximum is below 2^-105 keeps
// fewer digits; nothing overflows)
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + max(-126, min(127, e))) << 23); }

// byte k of a, b, c, d as one little-endian word
template <int K>
__device__ __forceinline__ uint32_t pack4_byte(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    constexpr uint32_t sel = (uint32_t)K | ((4u + K) << 4);
    return __byte_perm(__byte_perm(a, b, sel), __byte_perm(c, d, sel), 0x5410);
}

// Balanced base-256 digits of x = rint(v_c 2^e_c) (|x| <= 2^22 by the choice of e_c), for 16
// columns, as the three 16-byte plane rows of one K-row: x = d0 2^16 + d1 2^8 + d2 (as digits3).
// fmaf(v, 2^e, 1.5 2^23) rounds v 2^e to the nearest integer (ties to even, as __float2int_rn)
// and leaves it in the low mantissa bits: with bits = that float's bits, d2 is byte 0 of bits,
// d1 = byte 1 of x + 128 = byte 1 of bits + 128, d0 = byte 2 of x + 32896 (signed bytes).
__device__ __forceinline__ void digit_rows16(const float (&v)[16], const float (&sc)[16], uint4& r0, uint4& r1,
                                             uint4& r2) {
    uint32_t b2[16], b1[16], b0[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
        const uint32_t bits = __float_as_uint(fmaf(v[c], sc[c], 12582912.0f));
        b2[c] = bits;
        b1[c] = bits + 128u;
        b0[c] = bits + (32896u - 0x4B400000u);
    }
    r0 = make_uint4(pack4_byte<2>(b0[0], b0[1], b0[2], b0[3]), pack4_byte<2>(b0[4], b0[5], b0[6], b0[7]),
                    pack4_byte<2>(b0[8], b0[9], b0[10], b0[11]), pack4_byte<2>(b0[12], b0[13], b0[14], b0[15]));
    r1 = make_uint4(pack4_byte<1>(b1[0], b1[1], b1[2], b1[3]), pack4_byte<1>(b1[4], b1[5], b1[6], b1[7]),
                    pack4_byte<1>(b1[8], b1[9], b1[10], b1[11]), pack4_byte<1>(b1[12], b1[13], b1[14], b1[15]));
    r2 = make_uint4(pack4_byte<0>(b2[0], b2[1], b2[2], b2[3]), pack4_byte<0>(b2[4], b2[5], b2[6], b2[7]),
                    pack4_byte<0>(b2[8], b2[9], b2[10], b2[11]), pack4_byte<0>(b2[12], b2[13], b2[14], b2[15]));
}

// as digit_rows16 for 8 columns (three 8-byte plane half-rows)
__device__ __forceinline__ void digit_rows8(const float (&v)[8], const float (&sc)[8], uint2& r0, uint2& r1, uint2& r2) {
    uint32_t b2[8], b1[8], b0[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const uint32_t bits = __float_as_uint(fmaf(v[c], sc[c], 12582912.0f));
        b2[c] = bits;
        b1[c] = bits + 128u;
        b0[c] = bits + (32896u - 0x4B400000u);
    }
    r0 = make_uint2(pack4_byte<2>(b0[0], b0[1], b0[2], b0[3]), pack4_byte<2>(b0[4], b0[5], b0[6], b0[7]));
    r1 = make_uint2(pack4_byte<1>(b1[0], b1[1], b1[2], b1[3]), pack4_byte<1>(b1[4], b1[5], b1[6], b1[7]));
    r2 = make_uint2(pack4_byte<0>(b2[0], b2[1], b2[2], b2[3]), pack4_byte<0>(b2[4], b2[5], b2[6], b2[7]));
}

// (c0 + c1/256 + c2/65536) 2^16 of the three accumulator groups, times 2^e = f.x f.y (fp32,
// like an fp32 accumulation). |c0| <= K 2^14 <= 2^21 and |c1| <= 2^22 (K <= 128) convert exactly
// by the magic add; c2 (up to 3 2^21) takes the one conversion instruction.
__device__ __forceinline__ float acc3f(int g0, int g1, int g2, float2 f) {
    return fmaf(i22_to_f(g0), 65536.0f, fmaf(i22_to_f(g1), 256.0f, __int2float_rn(g2))) * f.x * f.y;
}

// with the fourth group c3 = d1 y2 + d2 y1 (weight 2^-8; |c3| <= 2 K 2^14 <= 2^22): the only
// dropped term is d2 y2, <= 2^-30 of the product of the two scaled maxima
__device__ __forceinline__ float acc4f(int g0, int g1, int g2, int g3, float2 f) {
    return fmaf(i22_to_f(g0), 65536.0f, fmaf(i22_to_f(g1), 256.0f, fmaf(i22_to_f(g3), 0.00390625f, __int2float_rn(g2)))) *
           f.x * f.y;
}

// zero 16 TMEM columns of this warp's 32 lanes (group c3 of an accumulator: the first MMA of
// a chain initialises only groups 0-2, so c3 must start at zero)
__device__ __forceinline__ void tmem_zero16(uint32_t taddr) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
                 "r"(0u));
}
__device__ __forceinline__ void tmem_zero8(uint32_t taddr) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(0u));
}
__device__ __forceinline__ void tmem_wait_st_() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void named_bar(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// ------------------------------------------------------------------ create: images
// One CTA (128 threads) per 128-row block: eS_B from the block's largest |S_ij|, then each
// thread writes the three digits of its row's entries into the zero-filled image (planes of
// 128 x d_pad bytes at img + off[B]). Repeated (row, column) entries are summed first (as the
// CSR SpMM does), in entry order, before digitising.
__device__ __forceinline__ bool sp8_first_of_col(const uint16_t* __restrict__ lcol, int32_t beg, int32_t e) {
    const uint16_t c = lcol[e];
    for (int32_t e2 = beg; e2 < e; ++e2)
        if (lcol[e2] == c) return false;
    return true;
}
__device__ __forceinline__ float sp8_col_sum(const uint16_t* __restrict__ lcol, const float* __restrict__ val,
                                             int32_t e, int32_t end) {
    const uint16_t c = lcol[e];
    float v = 0.f;
    for (int32_t e2 = e; e2 < end; ++e2)
        if (lcol[e2] == c) v += val[e2];
    return v;
}

// One warp per row (rows w, w + 4, ... of the block): lane i holds entry beg + i; entries with
// the same block-local column are found with __match_any_sync and summed in entry order by the
// first of them (0 + v_first + ... ascending, as sp8_col_sum). Rows longer than 32 entries take
// the per-entry scans above (lanes striding over the row).
__device__ __forceinline__ float sp8_row_entry(const uint16_t* __restrict__ lcol, const float* __restrict__ val,
                                               int32_t beg, int32_t end, int lane, bool& first, int& col) {
    const int32_t e = beg + lane;
    const bool have = e < end;
    col = have ? (int)lcol[e] : -1 - lane;   // absent lanes match nobody
    const float v = have ? val[e] : 0.f;
    const unsigned peers = __match_any_sync(0xffffffffu, col);
    first = have && (__ffs(peers) - 1) == lane;
    if (__all_sync(0xffffffffu, peers == (1u << lane))) return v;   // no duplicates in this row
    float acc = 0.f;
    for (int src = 0; src < 32; ++src) {
        const float x = __shfl_sync(0xffffffffu, v, src);
        if ((peers >> src) & 1u) acc += x;
    }
    return acc;
}

__global__ void __launch_bounds__(128) k_sp8_build(int64_t n, int64_t nblk, const int32_t* __restrict__ rp,
                                                   const float* __restrict__ val, const uint16_t* __restrict__ lcol,
                                                   const int32_t* __restrict__ doff, const int64_t* __restrict__ ioff,
                                                   int8_t* __restrict__ img, int* __restrict__ escale,
                                                   unsigned int* __restrict__ rrange, const int32_t* __restrict__ brow0) {
    __shared__ float red[4], red2[4];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t B = blockIdx.x; B < nblk; B += gridDim.x) {
        const int64_t r0 = brow0[B];   // the block's rows [brow0[B], brow0[B + 1]): <= 128
        const int rows = (int)(brow0[B + 1] - r0);
        float m = 0.f, mn = INFINITY;   // block max |S|, smallest nonzero row max (this warp's rows)
        for (int r = wid; r < rows; r += 4) {
            const int32_t beg = rp[r0 + r], end = rp[r0 + r + 1];
            const bool longrow = end - beg > 32;   // (warp-uniform; the match runs on every lane)
            bool first;
            int col;
            const float v = sp8_row_entry(lcol, val, beg, longrow ? beg : end, lane, first, col);
            float rm = 0.f;
            if (!longrow) {
                if (first) rm = fabsf(v);
            } else {
                for (int32_t e = beg + lane; e < end; e += 32)
                    if (sp8_first_of_col(lcol, beg, e)) rm = fmaxf(rm, fabsf(sp8_col_sum(lcol, val, e, end)));
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) rm = fmaxf(rm, __shfl_xor_sync(0xffffffffu, rm, o));
            m = fmaxf(m, rm);
            if (rm > 0.f) mn = fminf(mn, rm);
        }
        __syncthreads();
        if (lane == 0) {
            red[wid] = m;
            red2[wid] = mn;
        }
        __syncthreads();
        const float bmax = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
        const float bmin = fminf(fminf(red2[0], red2[1]), fminf(red2[2], red2[3]));
        const int eS = i8_scale_exp(bmax);
        if (threadIdx.x == 0) {
            escale[B] = eS;
            // precision check: binades between the block's max and its smallest row maximum (a
            // row far below the block's scale keeps few significant bits in the shared quantum)
            if (bmax > 0.f && bmin < INFINITY) {
                int e1, e2;
                frexpf(bmax, &e1);
                frexpf(bmin, &e2);
                atomicMax(rrange, (unsigned)(e1 - e2));
            }
        }
        const int dp = sp8_dpad(doff[B + 1] - doff[B]);
        int8_t* out = img + ioff[B];
        auto put = [&](int r, int col, float v) {
            int d0, d1, d2;
            digits3(__float2int_rn(ldexpf(v, eS)), d0, d1, d2);
            const int o = sp8_off(r, col, kSp8RB / 8);
            out[o] = (int8_t)d0;
            out[kSp8RB * dp + o] = (int8_t)d1;
            out[2 * kSp8RB * dp + o] = (int8_t)d2;
        };
        for (int r = wid; r < rows; r += 4) {
            const int32_t beg = rp[r0 + r], end = rp[r0 + r + 1];
            const bool longrow = end - beg > 32;
            bool first;
            int col;
            const float v = sp8_row_entry(lcol, val, beg, longrow ? beg : end, lane, first, col);
            if (!longrow) {
                if (first) put(r, col, v);
            } else {
                for (int32_t e = beg + lane; e < end; e += 32)
                    if (sp8_first_of_col(lcol, beg, e)) put(r, (int)lcol[e], sp8_col_sum(lcol, val, e, end));
            }
        }
    }
}

// rs1[i] = (sum_j S_ij) - 1 (fp64 sum), the row-sum deviation the centred step adds back;
// norms[0] = max_i sum_j |S_ij|, norms[1] = max_i |rs1[i]| (bits of non-negative floats, zeroed
// by the caller): the step kernel's a-priori bound on |Y| (static scales of Y_B's digits)
__global__ void k_rowsum_m1(int64_t n, const int32_t* __restrict__ rp, const float* __restrict__ val,
                            float* __restrict__ rs1, unsigned int* __restrict__ norms) {
    float ma = 0.f, mr = 0.f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double a = 0.0, aa = 0.0;
        for (int32_t e = rp[i]; e < rp[i + 1]; ++e) {
            a += (double)val[e];
            aa += fabs((double)val[e]);
        }
        rs1[i] = (float)(a - 1.0);
        ma = fmaxf(ma, __double2float_ru(aa));
        mr = fmaxf(mr, fabsf(rs1[i]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ma = fmaxf(ma, __shfl_xor_sync(0xffffffffu, ma, o));
        mr = fmaxf(mr, __shfl_xor_sync(0xffffffffu, mr, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(norms, __float_as_uint(ma));
        atomicMax(norms + 1, __float_as_uint(mr));
    }
}

// pos[jlist[k]] = k: where the T drain stores the partial of dictionary slot d (landmark-major,
// so the landmark reduction reads each landmark's partials contiguously)
__global__ void k_inverse_perm(int32_t count, const int32_t* __restrict__ jlist, int32_t* __restrict__ pos) {
    for (int32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < count; k += gridDim.x * blockDim.x) pos[jlist[k]] = k;
}

__global__ void k_sp8_sizes(int64_t nblk, const int32_t* __restrict__ doff, int64_t* __restrict__ bytes) {
    for (int64_t B = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; B < nblk; B += (int64_t)gridDim.x * blockDim.x)
        bytes[B] = (int64_t)3 * kSp8RB * sp8_dpad(doff[B + 1] - doff[B]);
}

// column max / min keys of Y2 (for D paths whose reduction does not form them)
__global__ void __launch_bounds__(256) k_colminmax(int64_t l, int bp, const float* __restrict__ Y2,
                                                   unsigned int* __restrict__ y2mm) {
    __shared__ float m[256], n_[256];
    const int rb = 256 / bp, c = threadIdx.x % bp, r = threadIdx.x / bp;
    float v = -3.0e38f, w = 3.0e38f;
    for (int64_t k = (int64_t)blockIdx.x * rb + r; k < l; k += (int64_t)gridDim.x * rb) {
        v = fmaxf(v, Y2[k * bp + c]);
        w = fminf(w, Y2[k * bp + c]);
    }
    m[threadIdx.x] = v;
    n_[threadIdx.x] = w;
    __syncthreads();
    if (threadIdx.x < bp) {
        for (int q = 1; q < rb; ++q) {
            v = fmaxf(v, m[q * bp + threadIdx.x]);
            w = fminf(w, n_[q * bp + threadIdx.x]);
        }
        atomicMax(y2mm + threadIdx.x, f32_order_key(v));
        atomicMin(y2mm + 64 + threadIdx.x, f32_order_key(w));
    }
}

// centred Y2 -> its digit planes Yd[p][j][0..15] (p = 0, 1, 2: d0, d1, d2 of
// rint((Y2[j][c] - t_c) 2^ey_c), ey_c from the column maxima of |Y2 - t|), once per apply: the
// step kernel copies dictionary rows of these planes (16 bytes each) instead of digitising every
// landmark once per block it touches. Centring by t = w^T Y2 removes the large common part of
// Y2 that the second J cancels anyway (S Y2 - 1 t^T = S (Y2 - 1 t^T) + (S 1 - 1) t^T), so the 24
// bits of the digits cover what survives the centring.
// (max |Y2_c - t_c| = max(max_c - t_c, t_c - min_c) from the column max / min keys; block 0
// records the exponents for the step kernel)
// (pitch: floats per row of Y2; a 16-column half of a wider block passes Y2, t, y2mm, ey2_out
// offset by its first column)
template <int BP>
__device__ __forceinline__ void y2_digits_body(int64_t l, const float* __restrict__ Y2, const double* __restrict__ t,
                                               const unsigned int* __restrict__ y2mm, int* __restrict__ ey2_out,
                                               uint8_t* __restrict__ Yd, unsigned int* __restrict__ zero_next,
                                               int pitch = BP) {
    static_assert(BP == 16, "b = 16");
    // zero_next: the Y1f column maxima the next iteration's k_blk_reduce_fold accumulates (this
    // iteration's k_y8_split has read them)
    if (zero_next && blockIdx.x == 0 && threadIdx.x < 64) zero_next[threadIdx.x] = 0u;
    float sc[BP], tc[BP];
#pragma unroll
    for (int c = 0; c < BP; ++c) {
        tc[c] = (float)t[c];
        const float mx = fmaxf(f32_from_order_key(y2mm[c]) - tc[c], tc[c] - f32_from_order_key(y2mm[64 + c]));
        const int e = i8_scale_exp(mx);
        sc[c] = pow2f(e);
        if (blockIdx.x == 0 && threadIdx.x == c) ey2_out[c] = e;
    }
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < l; j += (int64_t)gridDim.x * blockDim.x) {
        float v[BP];
        const float4* src = reinterpret_cast<const float4*>(Y2 + j * pitch);
#pragma unroll
        for (int c4 = 0; c4 < BP / 4; ++c4) {
            const float4 x = src[c4];
            v[4 * c4] = x.x - tc[4 * c4];
            v[4 * c4 + 1] = x.y - tc[4 * c4 + 1];
            v[4 * c4 + 2] = x.z - tc[4 * c4 + 2];
            v[4 * c4 + 3] = x.w - tc[4 * c4 + 3];
        }
        uint4 w0, w1, w2;
        digit_rows16(v, sc, w0, w1, w2);
        reinterpret_cast<uint4*>(Yd)[j] = w0;
        reinterpret_cast<uint4*>(Yd)[l + j] = w1;
        reinterpret_cast<uint4*>(Yd)[2 * l + j] = w2;
    }
}

template <int BP>
__global__ void __launch_bounds__(256) k_y2_digits(int64_t l, const float* __restrict__ Y2, const double* __restrict__ t,
                                                   const unsigned int* __restrict__ y2mm, int* __restrict__ ey2_out,
                                                   uint8_t* __restrict__ Yd, unsigned int* __restrict__ zero_next,
                                                   int pitch) {
    pdl_trigger();
    pdl_wait();
    y2_digits_body<BP>(l, Y2, t, y2mm, ey2_out, Yd, zero_next, pitch);
}

// k_dreduce_pair's reduction at b = 16 with 16-byte loads: a thread owns four columns of one
// row and one half of its slots (8 in flight); Y2 = (first half + second half) in fp64, each
// half in slot order -- a fixed order, deterministic, not bitwise k_dreduce_pair's.
__device__ __forceinline__ void dreduce16_body(int64_t l, int b, const int* __restrict__ xptr,
                                               const float* __restrict__ P, const int* __restrict__ dexp,
                                               const int* __restrict__ yexp, const double* __restrict__ w,
                                               float* __restrict__ Y2, double* __restrict__ tpart,
                                               double* __restrict__ t, unsigned int* __restrict__ counter,
                                               unsigned int* __restrict__ y2mm) {
    // 8 threads per row: column quad cq, and the first / second half of the row tile's slots
    // (adjacent lanes, summed in slot order each, then first + second); 32 rows per block pass
    constexpr int BP = 16, RPB = 32, U = 8;
    __shared__ double red[RPB][BP + 1];
    __shared__ float cmx[RPB][BP + 1], cmn[RPB][BP + 1];
    const int tid = threadIdx.x, hh = tid & 1, cq = (tid >> 1) & 3, rloc = tid >> 3;
    double unscale[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) unscale[u] = ldexp(1.0, -(*dexp + yexp[4 * cq + u]));
    float m[4] = {-3.0e38f, -3.0e38f, -3.0e38f, -3.0e38f}, mn[4] = {3.0e38f, 3.0e38f, 3.0e38f, 3.0e38f};
    double acc_t[4] = {0.0, 0.0, 0.0, 0.0};
    const int64_t npass = (l + (int64_t)gridDim.x * RPB - 1) / ((int64_t)gridDim.x * RPB);
    for (int64_t ps = 0; ps < npass; ++ps) {   // (uniform trip count: the halves meet in shuffles)
        const int64_t r = (ps * gridDim.x + blockIdx.x) * RPB + rloc;
        double v[4] = {0.0, 0.0, 0.0, 0.0};
        if (r < l) {
            const int X = (int)(r >> 7), rr = (int)(r & 127);
            const int q0 = xptr[X], q1 = xptr[X + 1], qm = q0 + (q1 - q0 + 1) / 2;
            const int a0 = hh ? qm : q0, a1 = hh ? q1 : qm;
            const float4* base = reinterpret_cast<const float4*>(P) + (int64_t)rr * (BP / 4) + cq;
            int q = a0;
            for (; q + U <= a1; q += U) {
                float4 pv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) pv[u] = __ldcs(base + (int64_t)(q + u) * (128 * BP / 4));
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    v[0] += (double)pv[u].x;
                    v[1] += (double)pv[u].y;
                    v[2] += (double)pv[u].z;
                    v[3] += (double)pv[u].w;
                }
            }
            if (q < a1) {   // the remainder as one predicated batch (all loads in flight; slot order kept)
                float4 pv[U];
#pragma unroll
                for (int u = 0; u < U; ++u)
                    pv[u] = q + u < a1 ? __ldcs(base + (int64_t)(q + u) * (128 * BP / 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (q + u < a1) {
                        v[0] += (double)pv[u].x;
                        v[1] += (double)pv[u].y;
                        v[2] += (double)pv[u].z;
                        v[3] += (double)pv[u].w;
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double o = __shfl_xor_sync(0xffffffffu, v[u], 1);
            v[u] = hh ? o + v[u] : v[u] + o;   // first half + second half in both lanes
        }
        if (r < l && hh == 0) {
            float4 o;
            float* of = &o.x;
            const double wr = w[r];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double y = v[u] * unscale[u];
                of[u] = (float)y;
                m[u] = fmaxf(m[u], of[u]);
                mn[u] = fminf(mn[u], of[u]);
                if (4 * cq + u < b) acc_t[u] += wr * y;
            }
            reinterpret_cast<float4*>(Y2 + r * BP)[cq] = o;
        }
    }
    if (hh == 0) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            red[rloc][4 * cq + u] = acc_t[u];
            cmx[rloc][4 * cq + u] = m[u];
            cmn[rloc][4 * cq + u] = mn[u];
        }
    }
    __syncthreads();
    if (tid < BP) {
        float mm = -3.0e38f, mi = 3.0e38f;
        double a = 0.0;
        for (int q = 0; q < RPB; ++q) {
            mm = fmaxf(mm, cmx[q][tid]);
            mi = fminf(mi, cmn[q][tid]);
            a += red[q][tid];
        }
        atomicMax(y2mm + tid, f32_order_key(mm));
        atomicMin(y2mm + 64 + tid, f32_order_key(mi));
        tpart[blockIdx.x * kMaxB + tid] = a;
    }
    if (last_block_done(counter)) {
        ordered_colsum_block(tpart, gridDim.x, kMaxB, BP, t);
        if (tid == 0) *counter = 0;
    }
}

// k_dreduce_pair and k_y2_digits in one cooperative launch: the grid syncs once t = w^T Y2 and
// Y2's column max/min keys are complete, then digitises Y2 - 1 t^T (one launch fewer per
// iteration; the grid is the co-resident block count, so t's fixed partial order is per device).
template <int BP>
__global__ void __launch_bounds__(256, 4) k_dreduce_y2d(int64_t l, int b, const int* __restrict__ xptr,
                                                     const float* __restrict__ P, const int* __restrict__ dexp,
                                                     const int* __restrict__ yexp, const double* __restrict__ w,
                                                     float* __restrict__ Y2, double* __restrict__ tpart,
                                                     double* __restrict__ t, unsigned int* __restrict__ counter,
                                                     unsigned int* __restrict__ y2mm, int* __restrict__ ey2_out,
                                                     uint8_t* __restrict__ Yd, unsigned int* __restrict__ zero_next) {
    pdl_trigger();
    pdl_wait();
    dreduce16_body(l, b, xptr, P, dexp, yexp, w, Y2, tpart, t, counter, y2mm);
    __threadfence();
    cooperative_groups::this_grid().sync();
    y2_digits_body<BP>(l, Y2, t, y2mm, ey2_out, Yd, zero_next);
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
// arrive on `bar` once this thread's earlier cp.async copies have landed (counts as one of the
// barrier's expected arrivals)
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// ------------------------------------------------------------------ the step kernel
// GRAM8 (see k_sp8_step): no fp32 row buffers for the FP64 Gram warps. A fourth image stage then
// fits (NS = 4 with a B_N ring of 2 and an rs1 ring of 4) and was measured: no gain (0.185 vs
// 0.182 ms per launch at config 4) -- with the Gram off the epilogue's path the step is bound by
// shared-memory bandwidth (~220 KB per block: the image written once by the bulk copy and read
// once by each product's MMAs, ~75 B/clk per SM), not by the stages.
template <int BP, bool GRAM8 = false>
struct Sp8Cfg {
    static constexpr int NB = 3 * BP;                    // B rows [y0; y1; y2]
    static constexpr int IMG = 3 * kSp8RB * kSp8DK;      // 48 KB: largest image
    static constexpr int NS = 3;                         // image stages
    static constexpr int BN = NB * kSp8DK;               // B of N: d_pad x NB (MN-major)
    static constexpr int NBT = 64;                       // B of T: row width [y0 | y1 | y2 | ones chunk]
    static constexpr int BT = NBT * kSp8RB;              // B of T: 128 rows x NBT (MN-major)
    static constexpr int YR = kSp8RB * BP * 4;           // fp32 rows of a block
    static constexpr int OFF_BN = NS * IMG;
    static constexpr int NBN = 4;                        // B_N ring (staged NBN blocks ahead)
    static constexpr int OFF_BT = OFF_BN + NBN * BN;
    static constexpr int OFF_YR = OFF_BT + 2 * BT;       // (GRAM8: no Y rows, no Y_prev rows)
    static constexpr int OFF_YP = OFF_YR + (GRAM8 ? 0 : 2 * YR);
    static constexpr int OFF_BAR = OFF_YP + (GRAM8 ? 0 : 2 * YR);
    static constexpr int MAXNB = 192;                    // blocks per CTA (per-CTA metadata table)
    static constexpr int OFF_META = OFF_BAR + 512;       // int64 ioff[MAXNB], int32 doff[MAXNB + 1], int32 eS[MAXNB]
    // rs1 ring: slot i % NRS is rewritten when block i + NRS is staged, i.e. after N(i + NRS - NBN)
    // has completed, which needs the epilogue's release of N(i + NRS - NBN - 2): NRS >= NBN + 2
    static constexpr int NRS = 8;
    // int64 ioff[MAXNB], int32 doff[MAXNB + 1], int32 eS[MAXNB], int32 r0[MAXNB + 1] (+ 8: 16-byte aligned)
    static constexpr int OFF_RS = OFF_META + 8 * MAXNB + 4 * (MAXNB + 1) + 4 * MAXNB + 4 * (MAXNB + 1) + 8;
    static constexpr int SMEM = OFF_RS + NRS * kSp8RB * 4 + 128;   // + alignment slack (no swizzle: 128 B suffices)
    static_assert(OFF_RS % 16 == 0, "rs ring alignment");
    static_assert(NRS >= NBN + 2, "rs ring depth");
    static_assert(SMEM + 1024 <= 227 * 1024, "dynamic + the kernel's 1 KB of static shared memory");
    static constexpr int THREADS = 17 * 32;   // (<= 120 registers); warp 16 issues the T products
    static constexpr int NGW = 2;                        // Gram warps (group C)
    // TMEM columns: accumulators with four 16-column groups (c0 = d0 y0, c1, c2, c3 = d1 y2 + d2 y1):
    // N[2] and T[2] (double-buffered; one T accumulator per block, whose 128 rows share the
    // column scales of Y_B's digits), 256 of 512 columns
    static constexpr int ACCW = 4 * BP;
    static constexpr int ACCN = 0, ACCT = 2 * ACCW;
    static constexpr int ACCG = 4 * ACCW;                // int8 Gram accumulator (GRAM8): 3 BP columns
    static_assert(ACCG + 3 * BP <= 512, "tmem");
    static_assert(BP == 16, "the tensor-core sparse step is built for b = 16");
};

// GRAM8 (steps whose Gram only feeds the next Cholesky-QR, never a Rayleigh-Ritz step): G and
// 1^T Y are formed from Y_B's digits on the int8 tensor cores, Yd^T [Yd | 1] accumulated exactly
// in one TMEM accumulator over the CTA's blocks (the digits' scales are per launch), instead of
// the FP64 Gram of the fp32 rows: no Gram warps, no staging of Y for them.
// TONLY (the standalone apply's A2, S^T X): only the T products, on a block of rows given in
// global memory (Yprev = X, n x BP fp32, staged by bulk copies into the fp32 row buffers) with
// the column scales of `norms` (= the bits of max |X_c|, BP words): no N products, no Gram, no Y.
template <int BP, bool WITH_H, bool GRAM8, bool TONLY = false>
__global__ void __launch_bounds__(Sp8Cfg<BP, GRAM8>::THREADS, 1)
    k_sp8_step(int64_t n, int64_t l_rows, int64_t nblk, const int8_t* __restrict__ gimg, const int64_t* __restrict__ ioff,
               const int32_t* __restrict__ doff, const int32_t* __restrict__ dict, const int* __restrict__ escale,
               const uint8_t* __restrict__ Yd, const int* __restrict__ ey2in, const double* __restrict__ t,
               const float* __restrict__ rs1, const float* __restrict__ norms, const int32_t* __restrict__ ppos,
               float* __restrict__ Y, float* __restrict__ P1, const float* __restrict__ Yprev,
               double* __restrict__ part, double* __restrict__ G, double* __restrict__ H, double* __restrict__ cs,
               unsigned int* __restrict__ counter, unsigned long long* __restrict__ trace, int mode,
               double* __restrict__ Rinv_next, int* __restrict__ status, int defer_gram, int ypitch, int p1pitch,
               const int32_t* __restrict__ brow0) {
    using C = Sp8Cfg<BP, GRAM8>;
    static_assert(!(GRAM8 && WITH_H), "the int8 Gram has no H'");
    static_assert(!TONLY || (!GRAM8 && !WITH_H), "TONLY uses the row buffers of the plain layout");
    // (diagnostics) trace[ev * 64 + i] (ev < 12; 2048 + (ev - 12) * 64 + i for ev 12..19):
    // globaltimer of event ev for block i < 64 of CTA 0
#define SP8_TR(ev, i)                                                                          \
    if (trace && blockIdx.x == 0 && (i) < 64) {                                                \
        unsigned long long t_;                                                                 \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                 \
        trace[((ev) < 12 ? (ev) * 64 : 2048 + ((ev) - 12) * 64) + (i)] = t_;                    \
    }
    constexpr int NB = C::NB;
    constexpr int NCB = BP / 8;
    constexpr int NPG = NCB * (NCB + 1) / 2;
    constexpr int NPH = WITH_H ? NCB * NCB : 1;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + C::OFF_BAR);
    uint64_t* full_img = bars;          // [NS <= 4]
    uint64_t* empty_img = bars + 4;     // [NS <= 4]
    uint64_t* bn_full = bars + 30;      // [4]
    uint64_t* bn_empty = bars + 34;     // [4]
    uint64_t* an_full = bars + 10;
    uint64_t* an_empty = bars + 12;
    uint64_t* bt_full = bars + 14;
    uint64_t* bt_empty = bars + 16;
    uint64_t* at_full = bars + 18;
    uint64_t* at_empty = bars + 20;
    uint64_t* yr_full = bars + 22;
    uint64_t* yr_empty = bars + 24;
    uint64_t* yp_full = bars + 26;
    uint64_t* yp_empty = bars + 28;
    uint64_t* gram_full = bars + 8;     // (GRAM8) the CTA's last Gram MMA has completed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 42);
    int* ey2 = reinterpret_cast<int*>(bars + 44);          // [BP] scale exponents of Y2's columns
    int* eyb = ey2 + BP;                                   // [BP] scale exponents of Y_B's columns (static bound)

    pdl_trigger();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t b0 = blockIdx.x * nblk / gridDim.x, b1 = (blockIdx.x + 1) * nblk / gridDim.x;
    const int nb = (int)(b1 - b0);
    const bool want_t = P1 != nullptr;
    const bool stream_only = (mode & 1) != 0;    // (diagnostics) images streamed, no MMA
    const unsigned poll_ns = (unsigned)mode >> 8;   // MMA warp: back-off between unready polls
    const bool no_gram = (mode & 8) != 0;           // (GRAM8) a 16-column half of a wider block: no Gram here
    const int pf_ahead = (mode >> 4) & 15;          // producer: L2 prefetch of the image pf_ahead blocks ahead (0: off)

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::NS; ++s) {
            mbar_init(&full_img[s], 1);
            mbar_init(&empty_img[s], 1);
        }
        for (int a = 0; a < C::NBN; ++a) {
            mbar_init(&bn_full[a], 32);   // the producer warp's lanes
            mbar_init(&bn_empty[a], 1);
        }
        mbar_init(gram_full, 1);
        for (int a = 0; a < 2; ++a) {
            mbar_init(&an_full[a], 1);
            mbar_init(&an_empty[a], 256);
            mbar_init(&bt_full[a], 256);
            mbar_init(&bt_empty[a], 1);
            mbar_init(&at_full[a], 1);
            mbar_init(&at_empty[a], 128);
            mbar_init(&yr_full[a], TONLY ? (ypitch == BP ? 1 : 32) : 256);   // (TONLY: the producer's copy of X_B)
            mbar_init(&yr_empty[a], TONLY ? 256 : 32 * C::NGW);
            mbar_init(&yp_full[a], 32 * C::NGW);   // the Gram group's cp.async rows of Y_prev
        }
        fence_barrier_init();
    }
    // the CTA's block metadata, once: no role waits on an L2 round trip per block
    int64_t* m_ioff = reinterpret_cast<int64_t*>(base + C::OFF_META);
    int32_t* m_doff = reinterpret_cast<int32_t*>(m_ioff + C::MAXNB);
    int32_t* m_es = m_doff + C::MAXNB + 1;
    int32_t* m_r0 = m_es + C::MAXNB;   // first row of each block (blocks are <= 128 consecutive rows)
    for (int k = threadIdx.x; k <= nb; k += blockDim.x) {
        m_doff[k] = __ldg(doff + b0 + k);
        m_r0[k] = __ldg(brow0 + b0 + k);
        if (k < nb) {
            m_ioff[k] = __ldg(ioff + b0 + k);
            m_es[k] = __ldg(escale + b0 + k);
        }
    }
    if (threadIdx.x < 2 * kSp8RB) {   // the ones chunk of both B_T buffers' rows (byte 0 = 1): 1^T Yd for GRAM8
        uint8_t* bt = base + C::OFF_BT + (threadIdx.x >> 7) * C::BT;
        *reinterpret_cast<uint4*>(bt + sp8_boff<C::NBT>(threadIdx.x & 127, 3)) = make_uint4(1u, 0u, 0u, 0u);
        fence_proxy_async();
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
    pdl_wait();   // everything below reads what earlier kernels wrote (Y2 digits, exponents, t, P1 slots)
    // (diagnostics) trace[768 + c]: CTA c's start, trace[1024 + c]: its blocks done (c < 256),
    // trace[1279]: the last CTA's end (after the Gram sums and the Cholesky)
    auto tail_tr = [&](int slot) {
        if (trace && threadIdx.x == 0) {
            unsigned long long t_;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
            trace[slot] = t_;
        }
    };
    if (blockIdx.x < 256) tail_tr(768 + blockIdx.x);
    if (threadIdx.x < BP) {
        // Y_B's digits take one scale per column for the whole launch, from an a-priori bound:
        // |Y_rc| <= 1/2 (sum_j |S_rj|) max_j |Y2 - 1 t^T|_jc + 1/2 |rs1_r| |t_c|, the digitised
        // Y2 column being <= 2^(22 - ey2_c) (no per-block maxima, no exchange between the epilogue
        // warps; the quantum is the column's, as the D stream's Y1 digits)
        if constexpr (TONLY) {   // X's digits: one scale per column from max |X_c|
            ey2[threadIdx.x] = 0;
            eyb[threadIdx.x] = i8_scale_exp(__uint_as_float(reinterpret_cast<const unsigned int*>(norms)[threadIdx.x]));
        } else {
            const int e2 = ey2in[threadIdx.x];
            ey2[threadIdx.x] = e2;
            const float bound = 0.5f * (norms[0] * pow2f(22 - e2) + norms[1] * fabsf((float)t[threadIdx.x]));
            eyb[threadIdx.x] = i8_scale_exp(bound * 1.001f);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    auto dpad_of = [&](int64_t B) { return sp8_dpad(m_doff[B - b0 + 1] - m_doff[B - b0]); };
    auto rows_of = [&](int64_t B) { return (int)(m_r0[B - b0 + 1] - m_r0[B - b0]); };
    auto row0_of = [&](int64_t B) { return (int64_t)m_r0[B - b0]; };

    // Gram accumulators live in warps 10-11 (per-warp DMMA fragments, as k_fused.cuh)
    // two interleaved accumulator sets (even / odd 4-row steps) halve the DMMA dependency chains
    double gacc[NPG][2], hacc[NPH][2], csum[NCB], gacc1[NPG][2], hacc1[NPH][2];
#pragma unroll
    for (int i = 0; i < NPG; ++i) gacc[i][0] = gacc[i][1] = gacc1[i][0] = gacc1[i][1] = 0.0;
#pragma unroll
    for (int i = 0; i < NPH; ++i) hacc[i][0] = hacc[i][1] = hacc1[i][0] = hacc1[i][1] = 0.0;
#pragma unroll
    for (int c = 0; c < NCB; ++c) csum[c] = 0.0;

    if (warp == 0) {
        // ------------------------------------------------ producer: B operand of N (all lanes: the
        // dictionary's Y2 digit rows, cp.async, lane g owning entries g, g + 32, ...) and the image
        // (lane 0, one bulk copy, issued first) of each block. image(i) needs T(i - NS) done, B(i)
        // N(i - NBN) done (with NBN = 2 that comes later, and B(i) has the image's flight time to land).
        int32_t s_d0 = m_doff[0], s_du = nb > 0 ? m_doff[1] - s_d0 : 0;
        int32_t s_j[kSp8DK / 32];
#pragma unroll
        for (int u = 0; u < kSp8DK / 32; ++u) s_j[u] = (32 * u + lane < s_du) ? __ldg(dict + s_d0 + 32 * u + lane) : 0;
        for (int i = 0; i < nb; ++i) {
            const int64_t B = b0 + i;
            const int32_t du = s_du;
            int32_t j[kSp8DK / 32];
#pragma unroll
            for (int u = 0; u < kSp8DK / 32; ++u) j[u] = s_j[u];
            if (i + 1 < nb) {   // the next block's dictionary rows of this lane
                s_d0 = m_doff[i + 1];
                s_du = m_doff[i + 2] - s_d0;
#pragma unroll
                for (int u = 0; u < kSp8DK / 32; ++u) s_j[u] = (32 * u + lane < s_du) ? __ldg(dict + s_d0 + 32 * u + lane) : 0;
            }
            if (lane == 0) {
                const int s = i % C::NS;
                const uint32_t ph = (uint32_t)((i / C::NS) & 1);
                const uint32_t bytes = (uint32_t)(3 * kSp8RB * dpad_of(B));
                mbar_wait(&empty_img[s], ph ^ 1u, 141 * 65536 + (i & 0xFFFF));
                SP8_TR(8, i);
                mbar_arrive_expect_tx(&full_img[s], bytes);
                bulk_load(base + s * C::IMG, gimg + m_ioff[i], bytes, &full_img[s]);
                SP8_TR(0, i);
                // the image pf_ahead blocks on: HBM -> L2 now, so that its load into a freed stage
                // (three stages cover ~1.5 blocks of the ~2.2 us HBM latency) finds it in L2
                if (pf_ahead && i + pf_ahead < nb)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gimg + m_ioff[i + pf_ahead]),
                                 "r"((uint32_t)(3 * kSp8RB * dpad_of(B + pf_ahead))) : "memory");
            }
            __syncwarp();
            if constexpr (TONLY) {
                // the block's rows of X into the row buffers: one bulk copy where they are contiguous
                // (ypitch == BP), else 16-byte cp.async chunks (a 16-column half of a wider block)
                const int a = i & 1;
                const int xrows = rows_of(B);
                mbar_wait(&yr_empty[a], ((uint32_t)((i >> 1) & 1)) ^ 1u, 159 * 65536 + (i & 0xFFFF));
                if (ypitch == BP) {
                    if (lane == 0) {
                        const uint32_t xb = (uint32_t)(xrows * BP * 4);
                        mbar_arrive_expect_tx(&yr_full[a], xb);
                        bulk_load(base + C::OFF_YR + a * C::YR, Yprev + row0_of(B) * BP, xb, &yr_full[a]);
                    }
                } else {
                    for (int q = lane; q < xrows * (BP / 4); q += 32) {
                        const int rr = q / (BP / 4), ch = q % (BP / 4);
                        cp_async16(base + C::OFF_YR + a * C::YR + (rr * BP + 4 * ch) * 4,
                                   Yprev + (row0_of(B) + rr) * (int64_t)ypitch + 4 * ch);
                    }
                    cp_async_arrive_noinc(&yr_full[a]);
                }
            } else if (!stream_only) {
                const int sb = i % C::NBN;
                mbar_wait(&bn_empty[sb], ((uint32_t)((i / C::NBN) & 1)) ^ 1u, 154 * 65536 + (i & 0xFFFF));
                uint8_t* bn = base + C::OFF_BN + sb * C::BN;
#pragma unroll
                for (int u = 0; u < kSp8DK / 32; ++u) {
                    const int g = 32 * u + lane;
                    if (g < du) {
#pragma unroll
                        for (int pl = 0; pl < 3; ++pl) cp_async16(bn + sp8_boff<NB>(g, pl), Yd + (pl * l_rows + j[u]) * 16);
                    }
                }
                // the block's row-sum deviations (512 B, one 16-byte chunk per lane; rs1 is padded to
                // whole blocks) into their ring: the epilogue reads them from shared memory, with
                // no global load between the N accumulator and the digits
                cp_async16(base + C::OFF_RS + ((i % C::NRS) * kSp8RB + 4 * lane) * 4, rs1 + row0_of(B) + 4 * lane);
                cp_async_arrive_noinc(&bn_full[sb]);
                if (lane == 0) SP8_TR(7, i);
            }
            __syncwarp();
        }
    } else if (warp == 1 && stream_only) {
        // (diagnostics) consume the images without any MMA; the other roles idle
        for (int i = 0; i < nb; ++i) {
            mbar_wait(&full_img[i % C::NS], (uint32_t)((i / C::NS) & 1), 156 * 65536 + (i & 0xFFFF));
            if (lane == 0) SP8_TR(1, i);
            if (elect_one()) mbar_arrive(&empty_img[i % C::NS]);
            __syncwarp();
        }
    } else if (stream_only) {
    } else if (warp == 1 || warp == 16) {
        // ------------------------------------------------ MMA issue: warp 1 the N products, warp 16 the
        // T products. Each waits (blocking mbarrier waits, woken by the hardware) for its own
        // operands only, so T(i) never queues behind the issue of N(i + 1) and neither polls.
        // d0 x [y0|y1|y2] -> groups 0-2, d1 x [y0|y1|y2] -> 1-3, d2 x [y0|y1] -> 2-3
        constexpr uint32_t id1n = idesc_i8_bmn(128, NB, 0), id2n = idesc_i8_bmn(128, NB, 0),
                           id3n = idesc_i8_bmn(128, 2 * BP, 0), id0n = idesc_i8_bmn(128, BP, 0);
        constexpr uint32_t id1t = idesc_i8_bmn(128, NB, 1), id2t = idesc_i8_bmn(128, NB, 1),
                           id3t = idesc_i8_bmn(128, 2 * BP, 1), id0t = idesc_i8_bmn(128, BP, 1);
        constexpr uint32_t KG = NB / 16 * 128;        // B of N: bytes per 8-row K group (the LBO)
        constexpr uint32_t KGT = C::NBT / 16 * 128;   // B of T
        constexpr uint32_t idg = idesc_i8_bmn(128, NB, 1);   // Gram: A = B = Y_B's digit image (MN-major)
        (void)poll_ns;
        if (warp == 16) {
            for (int i = 0; want_t && i < nb; ++i) {
                const int64_t B = b0 + i;
                const int s = i % C::NS, a = i & 1;
                const uint32_t pa = (uint32_t)((i >> 1) & 1);
                const int dp = dpad_of(B);
                mbar_wait(&bt_full[a], pa, 145 * 65536 + (i & 0xFFFF));
                mbar_wait(&at_empty[a], pa ^ 1u, 146 * 65536 + (i & 0xFFFF));
                mbar_wait(&full_img[s], (uint32_t)((i / C::NS) & 1), 147 * 65536 + (i & 0xFFFF));   // (passed: N(i) is done)
                tc_fence_after();
                if (lane == 0) SP8_TR(2, i);
                const uint32_t sa = smem_u32(base + s * C::IMG), sb = smem_u32(base + C::OFF_BT + a * C::BT);
                const uint32_t plane = (uint32_t)(kSp8RB * dp);
                if (elect_one()) {
#pragma unroll
                    for (int j = 0; j < kSp8RB / 32; ++j) {   // K = 32 rows (epilogue quadrant j's) per MMA
                        const uint32_t d = tbase + (uint32_t)(C::ACCT + a * C::ACCW);   // one accumulator per block
                        const uint64_t bd = umma_desc_none(sb + 4 * KGT * j, KGT, 128);
                        const uint64_t a0 = umma_desc_none(sa + 512 * j, 128, 2048);
                        if (j > 0) {
                            tc_mma_i8(d, a0, bd, id1t, 1u);
                            tc_mma_i8(d + BP, umma_desc_none(sa + plane + 512 * j, 128, 2048), bd, id2t, 1u);
                        } else {   // chain start: every group initialised by an MMA (no TMEM zeroing)
                            tc_mma_i8(d + BP, umma_desc_none(sa + plane + 512 * j, 128, 2048), bd, id2t, 0u);
                            tc_mma_i8(d, a0, bd, id0t, 0u);
                            tc_mma_i8(d + BP, a0, umma_desc_none(sb + 4 * KGT * j + 128, KGT, 128), id3t, 1u);
                        }
                        tc_mma_i8(d + 2 * BP, umma_desc_none(sa + 2 * plane + 512 * j, 128, 2048), bd, id3t, 1u);
                    }
                    tc_commit(&at_full[a]);
                    if (GRAM8 && !no_gram) {
                        // Yd^T [Yd | 1]: M = the image's 16-byte chunks as rows (digit planes 0-2, the
                        // ones chunk: lanes 0-48 are used, the rest read the next K group), K = the
                        // block's rows, N = 3 BP; one accumulator for the whole CTA (exact in int32:
                        // <= 2^14 per product, <= 2^15 rows)
#pragma unroll
                        for (int j = 0; j < kSp8RB / 32; ++j) {
                            const uint64_t gd = umma_desc_none(sb + 4 * KGT * j, KGT, 128);
                            tc_mma_i8(tbase + (uint32_t)C::ACCG, gd, gd, idg, (i > 0 || j > 0) ? 1u : 0u);
                        }
                        if (i + 1 == nb) tc_commit(gram_full);
                    }
                    tc_commit(&bt_empty[a]);
                    tc_commit(&empty_img[s]);
                }
                __syncwarp();
                if (lane == 0) SP8_TR(10, i);
            }
        } else {
            for (int i = 0; !TONLY && i < nb; ++i) {
                const int64_t B = b0 + i;
                const int s = i % C::NS, a = i & 1;
                const int dp = dpad_of(B);
                mbar_wait(&full_img[s], (uint32_t)((i / C::NS) & 1), 142 * 65536 + (i & 0xFFFF));
                mbar_wait(&bn_full[i % C::NBN], (uint32_t)((i / C::NBN) & 1), 143 * 65536 + (i & 0xFFFF));
                mbar_wait(&an_empty[a], ((uint32_t)((i >> 1) & 1)) ^ 1u, 144 * 65536 + (i & 0xFFFF));
                fence_proxy_async();   // B_N arrived by cp.async (generic proxy) -> visible to the MMA (async proxy)
                tc_fence_after();
                if (lane == 0) SP8_TR(1, i);
                const uint32_t sa = smem_u32(base + s * C::IMG), sb = smem_u32(base + C::OFF_BN + (i % C::NBN) * C::BN);
                const uint32_t d = tbase + (uint32_t)(C::ACCN + a * C::ACCW);
                const uint32_t plane = (uint32_t)(kSp8RB * dp);
                if (elect_one()) {
                    for (int j = 0; j < dp / 32; ++j) {   // K = 32 dictionary entries per MMA
                        const uint64_t bd = umma_desc_none(sb + 4 * KG * j, KG, 128);
                        const uint64_t a0 = umma_desc_none(sa + 4096 * j, 2048, 128);
                        if (j > 0) {
                            tc_mma_i8(d, a0, bd, id1n, 1u);
                            tc_mma_i8(d + BP, umma_desc_none(sa + plane + 4096 * j, 2048, 128), bd, id2n, 1u);
                        } else {   // chain start: d1 [y0|y1|y2] initialises groups 1-3, d0 y0 group 0,
                                   // then d0 [y1|y2] accumulates into groups 1-2 (no TMEM zeroing)
                            tc_mma_i8(d + BP, umma_desc_none(sa + plane, 2048, 128), bd, id2n, 0u);
                            tc_mma_i8(d, a0, bd, id0n, 0u);
                            tc_mma_i8(d + BP, a0, umma_desc_none(sb + 128, KG, 128), id3n, 1u);
                        }
                        tc_mma_i8(d + 2 * BP, umma_desc_none(sa + 2 * plane + 4096 * j, 2048, 128), bd, id3n, 1u);
                    }
                    tc_commit(&an_full[a]);
                    tc_commit(&bn_empty[i % C::NBN]);
                    if (!want_t) tc_commit(&empty_img[s]);
                }
                __syncwarp();
                if (lane == 0) SP8_TR(9, i);
            }
        }
    } else if (warp < 10) {
        // ------------------------------------------------ epilogue A (warps 2-9, TMEM lane = row): two
        // halves of four warps, half hf owning columns 8 hf .. 8 hf + 7 of every row
        constexpr int HC = BP / 2;
        const int q = warp & 3;
        const int hf = (warp - 2) >> 2;
        const int cb = HC * hf;
        const int r = 32 * q + lane;
        const uint32_t lane_off = (uint32_t)(32 * q) << 16;
        float mht[HC];   // -t / 2
#pragma unroll
        for (int c = 0; c < HC; ++c) mht[c] = (float)(-0.5 * t[cb + c]);
        float ysc[HC];
#pragma unroll
        for (int c = 0; c < HC; ++c) ysc[c] = pow2f(eyb[cb + c]);
        const float* rs_ring = reinterpret_cast<const float*>(base + C::OFF_RS);
        for (int i = 0; i < nb; ++i) {
            const int64_t B = b0 + i;
            const int a = i & 1;
            const uint32_t pa = (uint32_t)((i >> 1) & 1);
            const int rows = rows_of(B);
            if constexpr (TONLY) {
                // X_B's rows from shared memory -> digits -> B operand of T
                mbar_wait(&yr_full[a], pa, 160 * 65536 + (i & 0xFFFF));
                const float4* xr = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(base + C::OFF_YR + a * C::YR) + r * BP + cb);
                const float4 x0 = xr[0], x1 = xr[1];
                mbar_arrive(&yr_empty[a]);
                const bool livex = r < rows;   // (rows past the block's end hold stale bytes)
                float xv[HC] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
                for (int c = 0; c < HC; ++c) xv[c] = livex ? xv[c] : 0.f;
                uint2 w0, w1, w2;
                digit_rows8(xv, ysc, w0, w1, w2);
                mbar_wait(&bt_empty[a], pa ^ 1u, 151 * 65536 + (i & 0xFFFF));
                uint8_t* bt = base + C::OFF_BT + a * C::BT;
                *reinterpret_cast<uint2*>(bt + sp8_boff<C::NBT>(r, 0) + cb) = w0;
                *reinterpret_cast<uint2*>(bt + sp8_boff<C::NBT>(r, 1) + cb) = w1;
                *reinterpret_cast<uint2*>(bt + sp8_boff<C::NBT>(r, 2) + cb) = w2;
                fence_proxy_async();
                mbar_arrive(&bt_full[a]);
                continue;
            }
            const int eS = m_es[i];
            float2 sce[HC];   // accumulator 2^(16 - eS - ey2_c) -> S Y2
#pragma unroll
            for (int c = 0; c < HC; ++c) sce[c] = pow2f2(16 - eS - ey2[cb + c]);
            if (r == 0 && hf == 0) SP8_TR(12, i);
            mbar_wait(&an_full[a], pa, 149 * 65536 + (i & 0xFFFF));
            tc_fence_after();
            if (r == 0 && hf == 0) SP8_TR(3, i);
            int g0[HC], g1[HC], g2[HC], g3[HC];
            {
                const uint32_t col = tbase + lane_off + (uint32_t)(C::ACCN + a * C::ACCW + cb);
                tmem_ld8_u(col, g0);
                tmem_ld8_u(col + BP, g1);
                tmem_ld8_u(col + 2 * BP, g2);
                tmem_ld8_u(col + 3 * BP, g3);
                tmem_wait_ld();
            }
            // (staged by the producer with the B operand of N(i): visible once N(i) has completed)
            const float rsm1 = rs_ring[(i % C::NRS) * kSp8RB + r];
            tc_fence_before();
            mbar_arrive(&an_empty[a]);
            if (r == 0 && hf == 0) SP8_TR(11, i);
            // Y = -1/2 (S Y2 - 1 t^T) = -1/2 (S (Y2 - 1 t^T) + (S 1 - 1) t^T) for this row
            float y[HC];
            const bool live = r < rows;
#pragma unroll
            for (int c = 0; c < HC; ++c)
                y[c] = live ? fmaf(-0.5f, acc4f(g0[c], g1[c], g2[c], g3[c], sce[c]), rsm1 * mht[c]) : 0.f;
            if (want_t) {
                // the digits of Y_B (B operand of T) on the launch's static column scales
                uint2 w0, w1, w2;
                digit_rows8(y, ysc, w0, w1, w2);
                mbar_wait(&bt_empty[a], pa ^ 1u, 151 * 65536 + (i & 0xFFFF));
                if (r == 0 && hf == 0) SP8_TR(14, i);
                uint8_t* bt = base + C::OFF_BT + a * C::BT;
                *reinterpret_cast<uint2*>(bt + sp8_boff<C::NBT>(r, 0) + cb) = w0;
                *reinterpret_cast<uint2*>(bt + sp8_boff<C::NBT>(r, 1) + cb) = w1;
                *reinterpret_cast<uint2*>(bt + sp8_boff<C::NBT>(r, 2) + cb) = w2;
                fence_proxy_async();
                mbar_arrive(&bt_full[a]);
                if (r == 0 && hf == 1) SP8_TR(18, i);
                if (r == 64 && hf == 1) SP8_TR(19, i);
                if (r == 0 && hf == 0) SP8_TR(4, i);
            }
            // (after the digits, which gate the T product and the image's release)
            if (live) {
                float4* dst = reinterpret_cast<float4*>(Y + (row0_of(B) + r) * (int64_t)ypitch + cb);
                dst[0] = make_float4(y[0], y[1], y[2], y[3]);
                dst[1] = make_float4(y[4], y[5], y[6], y[7]);
            }
            if (r == 0 && hf == 0) SP8_TR(15, i);
            if constexpr (!GRAM8) {   // the rows for the FP64 Gram warps
                mbar_wait(&yr_empty[a], pa ^ 1u, 150 * 65536 + (i & 0xFFFF));
                if (r == 0 && hf == 0) SP8_TR(16, i);
                float4* yr = reinterpret_cast<float4*>(reinterpret_cast<float*>(base + C::OFF_YR + a * C::YR) + r * BP + cb);
                yr[0] = make_float4(y[0], y[1], y[2], y[3]);
                yr[1] = make_float4(y[4], y[5], y[6], y[7]);
                mbar_arrive(&yr_full[a]);
            }
        }
    } else if (warp < 14) {
        // ------------------------------------------------ group B (warps 10-13): T accumulator -> P1
        const int gt = threadIdx.x - 320;   // 0..127 (T accumulator: TMEM lane = dictionary entry gt)
        const uint32_t lane_off = (uint32_t)(32 * (warp & 3)) << 16;
        // T accumulator of block i -> P1 partials, scaled by Y_B's column exponents; the P1 slot
        // of this thread, du and eS of that block are passed in
        auto drain_t = [&](int i, int32_t pos, int32_t du, int eS) {
            const int a = i & 1;
            const uint32_t pa = (uint32_t)((i >> 1) & 1);
            mbar_wait(&at_full[a], pa, 148 * 65536 + (i & 0xFFFF));
            tc_fence_after();
            if (threadIdx.x == 320) SP8_TR(17, i);
            const int lrow = 32 * (warp & 3) + lane;   // the TMEM lane (dictionary entry) this thread drains
            float out[BP];
            if (mode & 4) {   // (diagnostics: drain arithmetic skipped)
#pragma unroll
                for (int c = 0; c < BP; ++c) out[c] = 0.f;
            } else {
                int g0[BP], g1[BP], g2[BP], g3[BP];
                const uint32_t col = (uint32_t)(C::ACCT + a * C::ACCW);
#pragma unroll
                for (int c0 = 0; c0 < BP; c0 += 8) {
                    tmem_ld8_u(tbase + lane_off + col + c0, *reinterpret_cast<int(*)[8]>(&g0[c0]));
                    tmem_ld8_u(tbase + lane_off + col + BP + c0, *reinterpret_cast<int(*)[8]>(&g1[c0]));
                    tmem_ld8_u(tbase + lane_off + col + 2 * BP + c0, *reinterpret_cast<int(*)[8]>(&g2[c0]));
                    tmem_ld8_u(tbase + lane_off + col + 3 * BP + c0, *reinterpret_cast<int(*)[8]>(&g3[c0]));
                }
                tmem_wait_ld();
                const int* ey = eyb;
#pragma unroll
                for (int c = 0; c < BP; ++c) out[c] = acc4f(g0[c], g1[c], g2[c], g3[c], pow2f2(16 - eS - ey[c]));
            }
            tc_fence_before();
            mbar_arrive(&at_empty[a]);
            if (lrow < du) {
                float4* dst = reinterpret_cast<float4*>(P1 + (int64_t)pos * p1pitch);
#pragma unroll
                for (int c = 0; c < BP; c += 4) dst[c / 4] = make_float4(out[c], out[c + 1], out[c + 2], out[c + 3]);
            }
        };
        int32_t p_d0 = nb > 0 ? m_doff[0] : 0, p_du = nb > 0 ? m_doff[1] - p_d0 : 0;
        int p_eS = nb > 0 ? m_es[0] : 0;
        const int lrow = 32 * (warp & 3) + lane;
        int32_t p_pos = (nb > 0 && lrow < p_du) ? __ldg(ppos + p_d0 + lrow) : 0;
        for (int i = 0; i < nb; ++i) {
            const int32_t du = p_du, pos = p_pos;
            const int eS = p_eS;
            if (i + 1 < nb) {   // the next block's P1 slot of this thread, one block ahead
                p_d0 = m_doff[i + 1];
                p_du = m_doff[i + 2] - p_d0;
                p_eS = m_es[i + 1];
                p_pos = (lrow < p_du) ? __ldg(ppos + p_d0 + lrow) : 0;
            }
            if (want_t) drain_t(i, pos, du, eS);
            if (lane == 0 && warp == 10) SP8_TR(6, i);
        }
        if constexpr (GRAM8) {
            // the CTA's Gram accumulator -> fp64 in shared memory (image stage 0: every MMA and load
            // of the CTA has completed once gram_full has): TMEM lane 16 p + i, column 16 q + j holds
            // sum_r d_p[r][i] d_q[r][j] (p <= 2), lane 48 the column sums of the digit planes
            if ((warp == 12 || warp == 13) && nb > 0 && want_t && !no_gram) {   // (no T products: no Gram, standalone A5)
                mbar_wait(gram_full, 0u, 158 * 65536);
                tc_fence_after();
                const int L = 32 * (warp & 3) + lane;
                int g[3 * BP];
#pragma unroll
                for (int c0 = 0; c0 < 3 * BP; c0 += 8)
                    tmem_ld8_u(tbase + lane_off + (uint32_t)(C::ACCG + c0), *reinterpret_cast<int(*)[8]>(&g[c0]));
                tmem_wait_ld();
                tc_fence_before();
                double* dbuf = reinterpret_cast<double*>(base);   // [3][BP][BP], then cs[BP]
                if (L <= 3 * BP) {
                    const int p = L / BP, ii = L % BP;
                    const double place = p == 0 ? 65536.0 : (p == 1 ? 256.0 : 1.0);   // 2^(16 - 8 p); the sums row: 1
#pragma unroll
                    for (int j = 0; j < BP; ++j) {
                        const double v = ((double)g[j] * 65536.0 + (double)g[BP + j] * 256.0 + (double)g[2 * BP + j]) * place;
                        if (p < 3) dbuf[(p * BP + ii) * BP + j] = v;
                        else if (ii == 0) dbuf[3 * BP * BP + j] = v;
                    }
                }
            }
        }
    } else if constexpr (GRAM8 || TONLY) {
        // (group C idles: the Gram runs on the int8 tensor cores, or there is none)
    } else {
        // ------------------------------------------------ group C (warps 14-15): the Grams on the FP64 tensor cores
        const int gt = threadIdx.x - 448;   // 0..63: rows gt, gt + 64 of Y_prev this thread stages
        const int gw = warp - 14;           // 0..1
        const int kr = lane & 3, cc = lane >> 2;
        auto gram = [&](int i) {
            const int64_t B = b0 + i;
            const int a = i & 1;
            const uint32_t pa = (uint32_t)((i >> 1) & 1);
            const int rows = rows_of(B);
            mbar_wait(&yr_full[a], pa, 152 * 65536 + (i & 0xFFFF));
            if constexpr (WITH_H) mbar_wait(&yp_full[a], pa, 153 * 65536 + (i & 0xFFFF));
            const float* yr = reinterpret_cast<const float*>(base + C::OFF_YR + a * C::YR);
            const float* yp = reinterpret_cast<const float*>(base + C::OFF_YP + a * C::YR);
            auto step = [&](int s4, double (&ga)[NPG][2], double (&ha)[NPH][2]) {
                const int rr = 64 * gw + 4 * s4 + kr;
                double yv[NCB], xv[NCB];
#pragma unroll
                for (int c = 0; c < NCB; ++c) {
                    const int col = 8 * c + cc;
                    yv[c] = (double)yr[rr * BP + col];
                    csum[c] += yv[c];
                    if constexpr (WITH_H) xv[c] = rr < rows ? (double)yp[rr * BP + col] : 0.0;
                }
                int pi = 0;
#pragma unroll
                for (int c = 0; c < NCB; ++c)
#pragma unroll
                    for (int c2 = c; c2 < NCB; ++c2) dmma_8x8x4(ga[pi++], yv[c], yv[c2]);
                if constexpr (WITH_H) {
#pragma unroll
                    for (int c = 0; c < NCB; ++c)
#pragma unroll
                        for (int c2 = 0; c2 < NCB; ++c2) dmma_8x8x4(ha[c * NCB + c2], xv[c], yv[c2]);
                }
            };
            if (!(mode & 2)) {   // (mode & 2: diagnostics, Gram skipped)
#pragma unroll 2
                for (int s4 = 0; s4 < 16; s4 += 2) {
                    step(s4, gacc, hacc);
                    step(s4 + 1, gacc1, hacc1);
                }
            }
            mbar_arrive(&yr_empty[a]);
        };
        // Y_prev rows of block k (Rayleigh-Ritz steps) -> yp[k & 1], cp.async, thread g = row g
        auto stage_yp = [&](int k) {
            if constexpr (WITH_H) {
                const int64_t B = b0 + k;
                uint8_t* yp = base + C::OFF_YP + (k & 1) * C::YR;
                const int rows = rows_of(B);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int rr = gt + 64 * h;
                    if (rr < rows) {
                        const uint8_t* src = reinterpret_cast<const uint8_t*>(Yprev + (row0_of(B) + rr) * BP);
#pragma unroll
                        for (int u = 0; u < BP / 4; ++u) cp_async16(yp + rr * BP * 4 + 16 * u, src + 16 * u);
                    }
                }
                cp_async_arrive_noinc(&yp_full[k & 1]);
            }
        };
        stage_yp(0);
        if (nb > 1) stage_yp(1);
        for (int i = 0; i < nb; ++i) {
            gram(i);
            if (gt == 0) SP8_TR(5, i);
            if (WITH_H && i + 2 < nb) {
                named_bar(5, 32 * C::NGW);   // every row of yp[i & 1] has been read by gram(i)
                stage_yp(i + 2);
            }
        }
    }

#undef SP8_TR
    __syncthreads();
    if (blockIdx.x < 256) tail_tr(1024 + blockIdx.x);
    // ---- CTA partial of the Grams (fixed warp order), then the last CTA sums them in CTA order
    tc_fence_before();
    __syncthreads();
    if (blockIdx.x < 256) tail_tr(1536 + blockIdx.x);
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
    }
    auto red = reinterpret_cast<double (*)[NCB * 8][NCB * 8 + 1]>(base);   // the image stages are free now
    auto cred = reinterpret_cast<double (*)[NCB * 8]>(reinterpret_cast<double*>(base) + 4 * (NCB * 8) * (NCB * 8 + 1));
    const int gw = warp - 14;
    const int kr = lane & 3, cc = lane >> 2, fr = lane >> 2, fc = 2 * (lane & 3);
#pragma unroll
    for (int i = 0; i < NPG; ++i) {
        gacc[i][0] += gacc1[i][0];
        gacc[i][1] += gacc1[i][1];
    }
#pragma unroll
    for (int i = 0; i < NPH; ++i) {
        hacc[i][0] += hacc1[i][0];
        hacc[i][1] += hacc1[i][1];
    }
    if (!GRAM8 && (warp == 14 || warp == 15)) {
#pragma unroll
        for (int c = 0; c < NCB; ++c) {
            double v = csum[c];
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            if (kr == 0) cred[gw][8 * c + cc] = v;
        }
        int pi = 0;
#pragma unroll
        for (int c = 0; c < NCB; ++c)
#pragma unroll
            for (int c2 = c; c2 < NCB; ++c2) {
                red[gw][8 * c + fr][8 * c2 + fc] = gacc[pi][0];
                red[gw][8 * c + fr][8 * c2 + fc + 1] = gacc[pi][1];
                red[gw][8 * c2 + fc][8 * c + fr] = gacc[pi][0];
                red[gw][8 * c2 + fc + 1][8 * c + fr] = gacc[pi][1];
                ++pi;
            }
    }
    __syncthreads();
    if (blockIdx.x < 256) tail_tr(1792 + blockIdx.x);
    double* pg = part + (int64_t)blockIdx.x * kGramPart;
    if constexpr (TONLY) {
        (void)pg;   // no Gram
    } else if constexpr (GRAM8) {
        // G_ij = 2^-(e_i + e_j) sum_p dbuf[p][i][j] (= sum_pq 2^(32 - 8p - 8q) c_pq[i][j]; the upper
        // triangle, mirrored), 1^T Y_j = 2^-e_j cs[j]; a CTA without blocks contributes zeros
        const double* dbuf = reinterpret_cast<const double*>(base);
        for (int pq = threadIdx.x; pq < BP * BP; pq += blockDim.x) {
            const int p = pq / BP, qq = pq % BP, i = p < qq ? p : qq, j = p < qq ? qq : p;
            const double v = (dbuf[(0 * BP + i) * BP + j] + dbuf[(1 * BP + i) * BP + j]) + dbuf[(2 * BP + i) * BP + j];
            pg[pq] = nb > 0 && want_t && !no_gram ? ldexp(v, -(eyb[i] + eyb[j])) : 0.0;
        }
        for (int qq = threadIdx.x; qq < BP; qq += blockDim.x)
            pg[2 * kMaxB * kMaxB + qq] = nb > 0 && want_t && !no_gram ? ldexp(dbuf[3 * BP * BP + qq], -eyb[qq]) : 0.0;
    } else {
        for (int pq = threadIdx.x; pq < BP * BP; pq += blockDim.x) {
            const int p = pq / BP, qq = pq % BP;
            pg[pq] = red[0][p][qq] + red[1][p][qq];
        }
        for (int qq = threadIdx.x; qq < BP; qq += blockDim.x)
            pg[2 * kMaxB * kMaxB + qq] = cred[0][qq] + cred[1][qq];
    }
    if constexpr (WITH_H) {
        __syncthreads();
        if (warp == 14 || warp == 15) {
#pragma unroll
            for (int c = 0; c < NCB; ++c)
#pragma unroll
                for (int c2 = 0; c2 < NCB; ++c2) {
                    red[gw][8 * c + fr][8 * c2 + fc] = hacc[c * NCB + c2][0];
                    red[gw][8 * c + fr][8 * c2 + fc + 1] = hacc[c * NCB + c2][1];
                }
        }
        __syncthreads();
        for (int pq = threadIdx.x; pq < BP * BP; pq += blockDim.x) {
            const int p = pq / BP, qq = pq % BP;
            pg[kMaxB * kMaxB + pq] = red[0][p][qq] + red[1][p][qq];
        }
    }
    if (blockIdx.x < 256) tail_tr(1280 + blockIdx.x);
    // defer_gram: the next k_blk_reduce_fold sums these partials and factors G (FoldGram)
    if (!defer_gram && last_block_done(counter)) {
        tail_tr(1277);
        for (int qq = threadIdx.x; qq < BP; qq += blockDim.x)
            cs[qq] = ordered_sum<32>(part + 2 * kMaxB * kMaxB + qq, gridDim.x, kGramPart);
        for (int pq = threadIdx.x; pq < BP * BP; pq += blockDim.x) {
            G[pq] = ordered_sum<32>(part + pq, gridDim.x, kGramPart);
            if constexpr (WITH_H) H[pq] = ordered_sum<32>(part + kMaxB * kMaxB + pq, gridDim.x, kGramPart);
        }
        if (threadIdx.x == 0) *counter = 0;
        __syncthreads();
        tail_tr(1278);
        if (Rinv_next) {   // E3 here too: G = R^T R and R^-1 for the next iteration (no extra launch)
            __syncthreads();
            auto A = reinterpret_cast<double (*)[kMaxB + 1]>(base);
            int* fail = reinterpret_cast<int*>(base + kMaxB * (kMaxB + 1) * sizeof(double));
            double* shift = reinterpret_cast<double*>(base + kMaxB * (kMaxB + 1) * sizeof(double) + 16);
            chol_block(BP, G, Rinv_next, status, A, fail, shift);
        }
        __syncthreads();
        tail_tr(1279);
    }
}

// ------------------------------------------------------------------ the int8 Gram at width 32
// G = Y^T Y and 1^T Y of an n x 32 block from Y's 24-bit digits (reading R18: eigs steps at
// block = 32 that feed no Rayleigh-Ritz step; the two 16-column passes of the sparse step share no
// Gram). Per 128-row block: the rows (16 KB, contiguous) by cp.async into one of two buffers;
// thread (row r, half h) digitises its 16 columns on the same per-column scales as the sparse
// step's Y_B digits into image h (rows of [y0 | y1 | y2 | ones chunk], the B_T layout); one
// elected thread issues Yd_a^T [Yd_a | 1], Yd_a^T [Yd_b | 1], Yd_b^T [Yd_b | 1] (4 K steps each)
// into three TMEM accumulators that live for the CTA's whole block list (exact int32 sums:
// <= 2^14 per product, <= 2^17 rows per CTA). Two image sets: block k + 1 is digitised while
// block k's MMAs run; two CTAs per SM hide the rest. At the end accumulator lane 16 p + i,
// column 16 q + j = sum_r d_p[r][i] d_q[r][j] is combined in fp64 into the CTA's partial, and
// the last CTA sums the partials in CTA order (fixed order: bitwise reproducible).
struct Gram8Cfg {
    static constexpr int ROWS = kSp8RB * 32 * 4;          // 16 KB: a block's fp32 rows
    static constexpr int IMG = 64 * kSp8RB;               // 8 KB: one half's digit image
    static constexpr int OFF_IMG = 2 * ROWS;              // [set][half]
    static constexpr int OFF_BAR = OFF_IMG + 4 * IMG;
    static constexpr int SMEM = OFF_BAR + 64 + 128;
    static constexpr int THREADS = 256;
    static constexpr int TCOLS = 256;                     // 3 accumulators of 48 columns
};

__global__ void __launch_bounds__(Gram8Cfg::THREADS, 2)
    k_gram8_32(int64_t n, const float* __restrict__ Y, const int* __restrict__ ey2in, const double* __restrict__ t,
               const float* __restrict__ norms, double* __restrict__ part, double* __restrict__ G,
               double* __restrict__ cs, unsigned int* __restrict__ counter) {
    using C = Gram8Cfg;
    constexpr int BW = 32, NB = 48;
    extern __shared__ __align__(128) uint8_t g8_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(g8_raw) + 127) & ~uintptr_t(127));
    uint64_t* mma_done = reinterpret_cast<uint64_t*>(base + C::OFF_BAR);   // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mma_done + 2);
    __shared__ int ecol[BW];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t nblk = (n + kSp8RB - 1) / kSp8RB;
    if (tid == 0) {
        mbar_init(&mma_done[0], 1);
        mbar_init(&mma_done[1], 1);
        fence_barrier_init();
    }
    if (tid < BW) {   // the sparse step's scales of Y's digits (k_sp8_step, same bound)
        const float bound = 0.5f * (norms[0] * pow2f(22 - ey2in[tid]) + norms[1] * fabsf((float)t[tid]));
        ecol[tid] = i8_scale_exp(bound * 1.001f);
    }
    // the ones chunk of all four images' rows (byte 0 = 1)
    for (int q = tid; q < 4 * kSp8RB; q += C::THREADS)
        *reinterpret_cast<uint4*>(base + C::OFF_IMG + (q >> 7) * C::IMG + sp8_boff<64>(q & 127, 3)) = make_uint4(1u, 0u, 0u, 0u);
    fence_proxy_async();
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(C::TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;
    const int r = tid & 127, hf = tid >> 7;
    float sc[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) sc[c] = pow2f(ecol[16 * hf + c]);
    auto stage = [&](int64_t B, int bufi) {   // rows of block B -> buffer bufi (16-byte chunks, 4 per thread)
        const int64_t r0 = B * kSp8RB;
        const int nrow = (int)min((int64_t)kSp8RB, n - r0);
        for (int q = tid; q < nrow * (BW / 4); q += C::THREADS)
            cp_async16(base + bufi * C::ROWS + q * 16, Y + r0 * BW + q * 4);
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    constexpr uint32_t KGT = 64 / 16 * 128;
    constexpr uint32_t idg = idesc_i8_bmn(128, NB, 1);
    int k = 0;
    if ((int64_t)blockIdx.x < nblk) stage(blockIdx.x, 0);
    for (int64_t B = blockIdx.x; B < nblk; B += gridDim.x, ++k) {
        const int bufi = k & 1, set = k & 1;
        if (B + gridDim.x < nblk) {
            stage(B + gridDim.x, bufi ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();   // block B's rows have landed (every thread's copies)
        if (k >= 2) mbar_wait(&mma_done[set], (uint32_t)(((k - 2) >> 1) & 1), 161 * 65536 + (k & 0xFFFF));
        {
            const bool live = B * kSp8RB + r < n;
            const float4* src = reinterpret_cast<const float4*>(base + bufi * C::ROWS + (r * BW + 16 * hf) * 4);
            float v[16];
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
                const float4 x = live ? src[c4] : make_float4(0.f, 0.f, 0.f, 0.f);
                v[4 * c4] = x.x; v[4 * c4 + 1] = x.y; v[4 * c4 + 2] = x.z; v[4 * c4 + 3] = x.w;
            }
            uint4 w0, w1, w2;
            digit_rows16(v, sc, w0, w1, w2);
            uint8_t* img = base + C::OFF_IMG + (2 * set + hf) * C::IMG;
            *reinterpret_cast<uint4*>(img + sp8_boff<64>(r, 0)) = w0;
            *reinterpret_cast<uint4*>(img + sp8_boff<64>(r, 1)) = w1;
            *reinterpret_cast<uint4*>(img + sp8_boff<64>(r, 2)) = w2;
        }
        fence_proxy_async();
        __syncthreads();   // both images complete; the row buffer may be refilled
        if (warp == 0) {
            tc_fence_after();
            const uint32_t ia = smem_u32(base + C::OFF_IMG + (2 * set) * C::IMG), ib = ia + C::IMG;
            if (elect_one()) {
#pragma unroll
                for (int j = 0; j < kSp8RB / 32; ++j) {   // K = 32 rows per MMA
                    const uint64_t da = umma_desc_none(ia + 4 * KGT * j, KGT, 128), db = umma_desc_none(ib + 4 * KGT * j, KGT, 128);
                    const uint32_t acc = (k > 0 || j > 0) ? 1u : 0u;
                    tc_mma_i8(tbase, da, da, idg, acc);            // Yd_a^T [Yd_a | 1]
                    tc_mma_i8(tbase + NB, da, db, idg, acc);       // Yd_a^T Yd_b (lane 48: 1^T Yd_b)
                    tc_mma_i8(tbase + 2 * NB, db, db, idg, acc);   // Yd_b^T [Yd_b | 1]
                }
                tc_commit(&mma_done[set]);
            }
            __syncwarp();
        }
    }
    // every MMA of this CTA has completed: the last commit of each set
    for (int set = 0; set < 2; ++set) {
        const int uses = (k + 1 - set) / 2;   // blocks k' < k with k' & 1 == set
        if (uses > 0) mbar_wait(&mma_done[set], (uint32_t)((uses - 1) & 1), 162 * 65536 + set);
    }
    tc_fence_after();
    // accumulators -> fp64: dbuf[a][p][i][j] (a = aa, ab, bb; p < 3), sums[a][j] from lane 48
    double* dbuf = reinterpret_cast<double*>(base);   // 3 * 3 * 16 * 16 + 3 * 16 doubles = 18.8 KB (the row buffers)
    if (warp < 2 && k > 0) {
        const int L = 32 * warp + lane;
        const uint32_t lane_off = (uint32_t)(32 * warp) << 16;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            int g[NB];
#pragma unroll
            for (int c0 = 0; c0 < NB; c0 += 8) tmem_ld8_u(tbase + lane_off + (uint32_t)(a * NB + c0), *reinterpret_cast<int(*)[8]>(&g[c0]));
            tmem_wait_ld();
            if (L <= 48) {
                const int p = L / 16, ii = L % 16;
                const double place = p == 0 ? 65536.0 : (p == 1 ? 256.0 : 1.0);
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const double v = ((double)g[j] * 65536.0 + (double)g[16 + j] * 256.0 + (double)g[32 + j]) * place;
                    if (p < 3) dbuf[((a * 3 + p) * 16 + ii) * 16 + j] = v;
                    else if (ii == 0) dbuf[3 * 3 * 256 + a * 16 + j] = v;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(C::TCOLS));
    }
    // the CTA's partial: G (32 x 32, row-major at pitch 32), then the column sums
    double* pg = part + (int64_t)blockIdx.x * kGramPart;
    for (int pq = tid; pq < BW * BW; pq += C::THREADS) {
        const int p_ = pq / BW, q_ = pq % BW, i = p_ < q_ ? p_ : q_, j = p_ < q_ ? q_ : p_;   // i <= j
        const int a = (i < 16 ? 0 : 2) + ((i < 16 && j >= 16) ? 1 : 0), ii = i & 15, jj = j & 15;
        double v = 0.0;
        if (k > 0) {
            v = (dbuf[((a * 3 + 0) * 16 + ii) * 16 + jj] + dbuf[((a * 3 + 1) * 16 + ii) * 16 + jj]) +
                dbuf[((a * 3 + 2) * 16 + ii) * 16 + jj];
            v = ldexp(v, -(ecol[i] + ecol[j]));
        }
        pg[pq] = v;
    }
    for (int q = tid; q < BW; q += C::THREADS)
        pg[2 * kMaxB * kMaxB + q] = k > 0 ? ldexp(dbuf[3 * 3 * 256 + (q < 16 ? 0 : 2) * 16 + (q & 15)], -ecol[q]) : 0.0;
    if (counter && last_block_done(counter)) {   // (counter == NULL: k_gram_sum follows)
        if (cs)
            for (int q = tid; q < BW; q += C::THREADS) cs[q] = ordered_sum(part + 2 * kMaxB * kMaxB + q, gridDim.x, kGramPart);
        double o[4];
        ordered_sum_x4(part, tid, BW * BW, gridDim.x, kGramPart, o);
#pragma unroll
        for (int e = 0; e < 4; ++e) G[tid + 256 * e] = o[e];
        if (tid == 0) *counter = 0;
    }
}

}  // namespace sbmds
