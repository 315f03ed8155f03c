// Row-blocked S with per-block landmark dictionaries (SURVEY.md §7 hard part 3).
//
// The interpolation operator is local ("the number of data points influenced
// by each landmark will shrink"; the sparse P keeps the few large entries),
// so RB = 256 consecutive vertices touch only u_B ~ 200 landmarks at config 4 (40x reuse).
// Both SpMMs therefore stage the touched rows in shared memory instead of gathering them
// through L1/L2 (the CSR/CSC kernels of k_sparse.cuh are L1- resp. L2-latency bound):
//
//   S Y2  (A5):  block B loads Y2[dict_B] (u_B x bp) into smem; each nnz carries a 16-bit
//                local column; rows are formed from smem gathers.             k_blk_spmm
//   S^T X (A2):  block B loads its 256 X rows into smem and forms, for each dictionary
//                entry d of B, the partial P1[d] = sum over the block's nnz in column
//                dict[d] (a block-local CSC: 8-bit local row, value), in fixed order;
//                k_blk_reduce sums the partials of landmark j over blocks in ascending
//                block order and applies the rank-one centring.               k_blk_spmmt
// Every sum has a fixed order: results are bitwise reproducible.
#pragma once
#include "common.cuh"
#include "k_dstream_sym8.cuh"   // digits3, i8_scale_exp (the fused Y1 digit split)
#include "k_small.cuh"          // chol_block, ordered_sum (the deferred Gram of the fold)

#include <cooperative_groups.h>

namespace sbmds {

constexpr int kRB = 256;   // rows per block (local row fits in 8 bits)

// ------------------------------------------------------------------ create-time build
// Blocks are rb consecutive rows each, or (brow0 != NULL) the row ranges [brow0[B], brow0[B + 1])
// with blkof[row] = B (the tensor-core sparse step splits a 128-row block whose dictionary
// exceeds its image into shorter ones).
__global__ void k_blk_offsets(int64_t n, int64_t nblk, int rb, const int32_t* __restrict__ rp, int32_t* __restrict__ off,
                              const int32_t* __restrict__ brow0) {
    for (int64_t B = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; B <= nblk; B += (int64_t)gridDim.x * blockDim.x)
        off[B] = rp[brow0 ? (int64_t)brow0[B] : min(B * rb, n)];
}

__global__ void k_blk_fill_blkof(int64_t nblk, const int32_t* __restrict__ brow0, int32_t* __restrict__ blkof) {
    for (int64_t B = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; B < nblk; B += (int64_t)gridDim.x * blockDim.x)
        for (int32_t r = brow0[B]; r < brow0[B + 1]; ++r) blkof[r] = (int32_t)B;
}

// flag[p] = 1 where a new (block, column) pair starts in the block-segmented col sort.
__global__ void k_blk_flags(int32_t nnz, int rb, const int32_t* __restrict__ scol, const int32_t* __restrict__ perm,
                            const int32_t* __restrict__ rowof, const int32_t* __restrict__ off,
                            int32_t* __restrict__ flag, const int32_t* __restrict__ blkof) {
    for (int32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += gridDim.x * blockDim.x) {
        const int32_t B = blkof ? blkof[rowof[perm[p]]] : rowof[perm[p]] / rb;
        flag[p] = (p == off[B] || scol[p] != scol[p - 1]) ? 1 : 0;
    }
}

// incl = inclusive scan of flags: dictionary slot of sorted entry p is incl[p] - 1.
__global__ void k_blk_dictoff(int64_t nblk, int32_t nnz, const int32_t* __restrict__ off,
                              const int32_t* __restrict__ flag, const int32_t* __restrict__ incl, int32_t total_u,
                              int32_t* __restrict__ dict_off) {
    for (int64_t B = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; B <= nblk; B += (int64_t)gridDim.x * blockDim.x) {
        const int32_t p = off[B];
        dict_off[B] = (p < nnz) ? incl[p] - flag[p] : total_u;
    }
}

__global__ void k_blk_umax(int64_t nblk, const int32_t* __restrict__ dict_off, unsigned int* __restrict__ umax) {
    unsigned int m = 0;
    for (int64_t B = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; B < nblk; B += (int64_t)gridDim.x * blockDim.x)
        m = max(m, (unsigned int)(dict_off[B + 1] - dict_off[B]));
    atomicMax(umax, m);
}

// (rb: rows per block; lcp, lrow, lval may be NULL when the block-local CSC is not wanted)
__global__ void k_blk_scatter(int32_t nnz, int rb, const int32_t* __restrict__ scol, const int32_t* __restrict__ perm,
                              const int32_t* __restrict__ rowof, const float* __restrict__ val,
                              const int32_t* __restrict__ flag, const int32_t* __restrict__ incl,
                              const int32_t* __restrict__ dict_off, int32_t* __restrict__ dict,
                              int32_t* __restrict__ lcp, uint16_t* __restrict__ lcol, uint8_t* __restrict__ lrow,
                              float* __restrict__ lval, const int32_t* __restrict__ blkof,
                              const int32_t* __restrict__ brow0) {
    for (int32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += gridDim.x * blockDim.x) {
        const int32_t e = perm[p];
        const int32_t row = rowof[e];
        const int32_t B = blkof ? blkof[row] : row / rb;
        const int32_t d = incl[p] - 1;
        if (flag[p]) {
            dict[d] = scol[p];
            if (lcp) lcp[d] = p;
        }
        lcol[e] = (uint16_t)(d - dict_off[B]);
        if (lrow) {
            lrow[p] = (uint8_t)(row - (brow0 ? brow0[B] : B * rb));
            lval[p] = val[e];
        }
    }
}

// ------------------------------------------------------------------ A5: Y = -1/2 (S Y2 - 1 t^T)
// One CTA per 256-row block: Y2[dict_B] -> smem, then LPR lanes per row (float4 each);
// a row's nnz metadata is read LPR entries at a time (one coalesced load per lane) and
// broadcast within the lane group by shuffles.
// Sum over one row of S of val * Y2[dict[lcol]] (staged in shared memory as float4 rows), LPR
// lanes per row (lane q owns float4 q of the b values). The loop is warp-uniform (maxlen = the
// warp's longest row) so the shuffles are full-warp; each lane first loads 8 of the row's
// (column, value) pairs with independent loads, then the group consumes them in entry order
// (beg, beg + 1, ...): the summation order is fixed, so results are bitwise reproducible.
template <int LPR>
__device__ __forceinline__ float4 blk_row_sum(int32_t beg, int32_t end, int maxlen, int q,
                                              const uint16_t* __restrict__ lcol, const float* __restrict__ val,
                                              const float4* __restrict__ ys4, int nv) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int c0 = 0; c0 < maxlen; c0 += 8 * LPR) {
        int lc[8];
        float vv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int32_t e = beg + c0 + u * LPR + q;
            const bool ok = e < end;
            lc[u] = ok ? (int)__ldg(lcol + e) : 0;
            vv[u] = ok ? __ldg(val + e) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (c0 + u * LPR >= maxlen) break;   // (warp-uniform) the rest of the chunk is padding in every row
#pragma unroll
            for (int tq = 0; tq < LPR; ++tq) {
                const int c = __shfl_sync(0xffffffffu, lc[u], tq, LPR);
                const float v = __shfl_sync(0xffffffffu, vv[u], tq, LPR);
                const float4 y = ys4[c * nv + q];
                acc.x = fmaf(v, y.x, acc.x);
                acc.y = fmaf(v, y.y, acc.y);
                acc.z = fmaf(v, y.z, acc.z);
                acc.w = fmaf(v, y.w, acc.w);
            }
        }
    }
    return acc;
}

template <int LPR>
__global__ void __launch_bounds__(256) k_blk_spmm(int64_t n, int b, int bp, const int32_t* __restrict__ rp,
                                                  const uint16_t* __restrict__ lcol, const float* __restrict__ val,
                                                  const int32_t* __restrict__ dict, const int32_t* __restrict__ dict_off,
                                                  const float* __restrict__ Y2, const double* __restrict__ t,
                                                  float* __restrict__ Y) {
    constexpr int G = 32 / LPR;
    extern __shared__ float4 ys4[];
    const int64_t B = blockIdx.x;
    const int32_t d0 = dict_off[B], u = dict_off[B + 1] - d0;
    const int nv = bp / 4;
    for (int e = threadIdx.x; e < u * nv; e += blockDim.x) {
        const int i = e / nv, q = e % nv;
        ys4[e] = __ldg(reinterpret_cast<const float4*>(Y2 + (int64_t)dict[d0 + i] * bp) + q);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / LPR, q = lane % LPR;
    const unsigned gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (g * LPR));
    const double t0 = t[4 * q], t1 = t[4 * q + 1], t2 = t[4 * q + 2], t3 = t[4 * q + 3];
    for (int r = warp * G + g; r < kRB; r += 8 * G) {   // the same trip count for every lane
        const int64_t i = B * kRB + r;
        const bool live = i < n;
        const int32_t beg = live ? rp[i] : 0, end = live ? rp[i + 1] : 0;
        const int maxlen = __reduce_max_sync(0xffffffffu, (unsigned)(end - beg));
        const float4 acc = blk_row_sum<LPR>(beg, end, maxlen, q, lcol, val, ys4, nv);
        if (!live) continue;
        float4 out;
        out.x = (float)(-0.5 * ((double)acc.x - t0));
        out.y = (float)(-0.5 * ((double)acc.y - t1));
        out.z = (float)(-0.5 * ((double)acc.z - t2));
        out.w = (float)(-0.5 * ((double)acc.w - t3));
        reinterpret_cast<float4*>(Y + i * b)[q] = out;
    }
}

// ------------------------------------------------------------------ A2 part 1: block partials
// One CTA per 256-row block: its X rows -> smem. Each group of LPR lanes owns one dictionary
// entry d of the block (32/LPR entries per warp in flight) and walks the entry's block-local
// column list in row order: metadata is read LPR entries at a time (one load per lane) and
// broadcast within the group; P1[d] = the fp32 partial (bp wide), fixed summation order.
template <int LPR>
__global__ void __launch_bounds__(256) k_blk_spmmt(int64_t n, int b, int bp, const float* __restrict__ X,
                                                   const int32_t* __restrict__ dict_off, const int32_t* __restrict__ lcp,
                                                   const uint8_t* __restrict__ lrow, const float* __restrict__ lval,
                                                   float* __restrict__ P1) {
    constexpr int G = 32 / LPR;
    extern __shared__ float4 xs4[];   // kRB x bp/4 (dynamic: up to 64 KB at bp = 64)
    const int64_t B = blockIdx.x;
    const int nv = bp / 4;
    const int64_t r0 = B * kRB;
    const int rows = (int)((n - r0) < kRB ? (n - r0) : kRB);
    for (int e = threadIdx.x; e < rows * nv; e += blockDim.x)
        xs4[e] = __ldg(reinterpret_cast<const float4*>(X + (r0 + e / nv) * b) + (e % nv));
    __syncthreads();
    const int32_t d0 = dict_off[B], u = dict_off[B + 1] - d0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / LPR, q = lane % LPR;
    const unsigned gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (g * LPR));
    for (int di = warp * G + g; di < u; di += 8 * G) {
        const int32_t d = d0 + di;
        const int32_t beg = lcp[d], end = lcp[d + 1];
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int32_t p0 = beg; p0 < end; p0 += LPR) {
            const int32_t p = p0 + q;
            const int r_l = (p < end) ? (int)lrow[p] : 0;
            const float v_l = (p < end) ? lval[p] : 0.f;
#pragma unroll
            for (int tq = 0; tq < LPR; ++tq) {
                const int r = __shfl_sync(gmask, r_l, tq, LPR);
                const float v = __shfl_sync(gmask, v_l, tq, LPR);
                const float4 x = xs4[r * nv + q];
                acc.x = fmaf(v, x.x, acc.x);
                acc.y = fmaf(v, x.y, acc.y);
                acc.z = fmaf(v, x.z, acc.z);
                acc.w = fmaf(v, x.w, acc.w);
            }
        }
        reinterpret_cast<float4*>(P1 + (int64_t)d * bp)[q] = acc;
    }
}

// ------------------------------------------------------------------ A2 part 2: Y1 = sum_B P1 - w s^T
// One warp per landmark j: the dictionary slots holding j (ascending block order) are
// summed in fp64 (jlist == NULL: the partials are already stored landmark-major, slot k = k), LPR lanes per slot row, a fixed shuffle tree across the G slot groups.
template <int LPR>
__global__ void __launch_bounds__(256) k_blk_reduce(int64_t l, int b, int bp, const int32_t* __restrict__ jptr,
                                                    const int32_t* __restrict__ jlist, const float* __restrict__ P1,
                                                    const double* __restrict__ w, const double* __restrict__ s,
                                                    float* __restrict__ Y1) {
    constexpr int G = 32 / LPR;
    const int lane = threadIdx.x & 31;
    const int g = lane / LPR, q = lane % LPR;
    const int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (j >= l) return;
    const int32_t beg = jptr[j], end = jptr[j + 1];
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int32_t k = beg + g;
    for (; k + 3 * G < end; k += 4 * G) {   // four loads in flight, added in slot order
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            v[u] = __ldg(reinterpret_cast<const float4*>(P1 + (int64_t)(jlist ? jlist[k + u * G] : k + u * G) * bp) + q);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a0 += v[u].x; a1 += v[u].y; a2 += v[u].z; a3 += v[u].w;
        }
    }
    for (; k < end; k += G) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(P1 + (int64_t)(jlist ? jlist[k] : k) * bp) + q);
        a0 += v.x; a1 += v.y; a2 += v.z; a3 += v.w;
    }
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, o);
        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        a2 += __shfl_xor_sync(0xffffffffu, a2, o);
        a3 += __shfl_xor_sync(0xffffffffu, a3, o);
    }
    if (g == 0) {
        const double wj = w[j];
        const int c = 4 * q;
        float4 out;
        out.x = (float)(a0 - wj * s[c + 0]);
        out.y = (float)(a1 - wj * s[c + 1]);
        out.z = (float)(a2 - wj * s[c + 2]);
        out.w = (float)(a3 - wj * s[c + 3]);
        reinterpret_cast<float4*>(Y1 + j * bp)[q] = out;
    }
}

// Deferred E2/E3 of the previous tensor-core sparse step (k_sp8_step with defer_gram): its CTA
// Gram partials, summed here in CTA order by block 0 (s = 1^T Y, G = Y^T Y) and factored
// (chol_block -> R^-1, status) while the other blocks sum the landmark partials into `scratch`
// (fp64); a grid sync, then the fold reads s and R^-1. Off the step's critical path: its last CTA
// no longer sums and factors after every other CTA has finished.
struct FoldGram {
    const double* part = nullptr;   // nullptr: s and Rinv are given (no deferred Gram)
    int nparts = 0;
    double* G = nullptr;
    double* s_out = nullptr;
    double* Rinv_out = nullptr;
    int* status = nullptr;
    double* scratch = nullptr;      // lpad x 16 fp64 landmark sums
    unsigned int* counter = nullptr;   // zero; the last of the Gram blocks factors
};
constexpr int kFoldGramBlocks = 5;   // blocks summing the Gram partials (4 threads per entry)

// A2 part 2 fused with the R^-1 fold of the eigs iteration (b = 16): Y1[j] = (sum of landmark
// j's partials, landmark-major, in slot order, fp64) - w_j s^T, then Y1f[j] = (Y1[j] R^-1) exactly
// as k_y16_prep forms it (fp64 fma over p <= c in order), the per-column max |Y1f| (atomicMax on
// the float bits; cmax zeroed by the caller) and zero pad rows l..lpad; block 0 also resets the Y2
// max / min keys of the pair reduce (zero64, as k_y16_prep). A thread owns four columns of one
// landmark (16-byte partial loads, 8 slots in flight); the four threads of a landmark exchange
// their sums by shuffles for the fold.
__global__ void __launch_bounds__(256, 4) k_blk_reduce_fold(int64_t l, int64_t lpad, const int32_t* __restrict__ jptr,
                                                         const float* __restrict__ P1, const double* __restrict__ w,
                                                         const double* s, const double* Rinv,
                                                         float* __restrict__ Y1f, unsigned int* __restrict__ cmax,
                                                         unsigned int* __restrict__ zero64, int8_t* __restrict__ Y8T,
                                                         int* __restrict__ yexp, FoldGram fg) {
    pdl_trigger();
    pdl_wait();
    constexpr int BP = 16, JPB = 64, U = 8;
    __shared__ double Ms[BP * BP];
    __shared__ float mxs[JPB][BP + 1];
    if (zero64 && blockIdx.x == 0 && threadIdx.x < 128) zero64[threadIdx.x] = threadIdx.x < 64 ? 0u : 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31, cq = threadIdx.x & 3, jl = threadIdx.x >> 2;
    // fp64 sum of landmark j's partials (columns 4 cq .. 4 cq + 3), in slot order
    auto landmark_sum = [&](int64_t j, double (&a)[4]) {
        const int32_t b0 = __ldg(jptr + j), e0 = __ldg(jptr + j + 1);
        const float4* base = reinterpret_cast<const float4*>(P1) + cq;
        a[0] = a[1] = a[2] = a[3] = 0.0;
        int32_t k = b0;
        for (; k + U <= e0; k += U) {
            float4 pv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) pv[u] = __ldcs(base + (int64_t)(k + u) * (BP / 4));
#pragma unroll
            for (int u = 0; u < U; ++u) {
                a[0] += pv[u].x; a[1] += pv[u].y; a[2] += pv[u].z; a[3] += pv[u].w;
            }
        }
        if (k < e0) {   // the remainder as one predicated batch (slot order kept)
            float4 pv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) pv[u] = k + u < e0 ? __ldcs(base + (int64_t)(k + u) * (BP / 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (k + u < e0) { a[0] += pv[u].x; a[1] += pv[u].y; a[2] += pv[u].z; a[3] += pv[u].w; }
        }
    };
    const bool deferred = fg.part != nullptr;
    if (deferred) {
        if (blockIdx.x < kFoldGramBlocks) {
            // entry e < 272 (G row-major, then s), quarter qt of the CTA range: 4 consecutive lanes,
            // each sums its quarter in CTA order, the first adds the four in quarter order
            __shared__ double Ach[BP][kMaxB + 1];
            __shared__ int chfail;
            __shared__ double chshift;
            const int task = blockIdx.x * blockDim.x + threadIdx.x, e = task >> 2, qt = task & 3;
            const int per = (fg.nparts + 3) / 4, q0 = min(fg.nparts, qt * per), q1 = min(fg.nparts, q0 + per);
            const int off = e < BP * BP ? e : 2 * kMaxB * kMaxB + (e - BP * BP);
            double v = 0.0;
            if (e < BP * BP + BP) v = ordered_sum<32>(fg.part + (int64_t)q0 * kGramPart + off, q1 - q0, kGramPart);
            const double v1 = __shfl_down_sync(0xffffffffu, v, 1), v2 = __shfl_down_sync(0xffffffffu, v, 2),
                         v3 = __shfl_down_sync(0xffffffffu, v, 3);
            if (qt == 0 && e < BP * BP + BP) {
                const double tot = ((v + v1) + v2) + v3;
                if (e < BP * BP) fg.G[e] = tot;
                else fg.s_out[e - BP * BP] = tot;
            }
            if (last_block_of(fg.counter, kFoldGramBlocks)) {
                chol_block(BP, fg.G, fg.Rinv_out, fg.status, Ach, &chfail, &chshift);
                if (threadIdx.x == 0) *fg.counter = 0;
            }
        } else {
            // 8 threads per landmark here: column quad and the first / second half of its slots
            // (each half in slot order, then first + second), 32 landmarks per block pass
            const int hh = threadIdx.x & 1, cq2 = (threadIdx.x >> 1) & 3, jl2 = threadIdx.x >> 3;
            const int64_t nlb = gridDim.x - kFoldGramBlocks, npass = (l + nlb * 32 - 1) / (nlb * 32);
            for (int64_t ps = 0; ps < npass; ++ps) {
                const int64_t j = (ps * nlb + (blockIdx.x - kFoldGramBlocks)) * 32 + jl2;
                double a[4] = {0.0, 0.0, 0.0, 0.0};
                if (j < l) {
                    const int32_t b0 = __ldg(jptr + j), e0 = __ldg(jptr + j + 1), bm = b0 + (e0 - b0 + 1) / 2;
                    const int32_t k0 = hh ? bm : b0, k1 = hh ? e0 : bm;
                    const float4* base = reinterpret_cast<const float4*>(P1) + cq2;
                    int32_t k = k0;
                    for (; k + U <= k1; k += U) {
                        float4 pv[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) pv[u] = __ldcs(base + (int64_t)(k + u) * (BP / 4));
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            a[0] += pv[u].x; a[1] += pv[u].y; a[2] += pv[u].z; a[3] += pv[u].w;
                        }
                    }
                    if (k < k1) {   // the remainder as one predicated batch (slot order kept)
                        float4 pv[U];
#pragma unroll
                        for (int u = 0; u < U; ++u)
                            pv[u] = k + u < k1 ? __ldcs(base + (int64_t)(k + u) * (BP / 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                        for (int u = 0; u < U; ++u)
                            if (k + u < k1) { a[0] += pv[u].x; a[1] += pv[u].y; a[2] += pv[u].z; a[3] += pv[u].w; }
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const double o = __shfl_xor_sync(0xffffffffu, a[u], 1);
                    a[u] = hh ? o + a[u] : a[u] + o;
                }
                if (j < l && hh == 0) {
                    double2* dst = reinterpret_cast<double2*>(fg.scratch + j * BP + 4 * cq2);
                    dst[0] = make_double2(a[0], a[1]);
                    dst[1] = make_double2(a[2], a[3]);
                }
            }
        }
        __threadfence();
        cooperative_groups::this_grid().sync();
        s = fg.s_out;
        Rinv = fg.Rinv_out;
    }
    for (int e = threadIdx.x; e < BP * BP; e += blockDim.x) Ms[e] = __ldcg(Rinv + e);
    __syncthreads();
    float cm[4] = {0.f, 0.f, 0.f, 0.f};
    double sc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) sc[u] = __ldcg(s + 4 * cq + u);
    for (int64_t j0 = (int64_t)blockIdx.x * JPB; j0 < lpad; j0 += (int64_t)gridDim.x * JPB) {
        const int64_t j = j0 + jl;
        float y[4] = {0.f, 0.f, 0.f, 0.f};
        if (j < l) {
            double a[4];
            if (deferred) {
                const double2* src = reinterpret_cast<const double2*>(fg.scratch + j * BP + 4 * cq);
                const double2 a01 = __ldcg(src), a23 = __ldcg(src + 1);
                a[0] = a01.x; a[1] = a01.y; a[2] = a23.x; a[3] = a23.y;
            } else {
                landmark_sum(j, a);
            }
            const double wj = w[j];
#pragma unroll
            for (int u = 0; u < 4; ++u) y[u] = (float)(a[u] - wj * sc[u]);
        }
        // the landmark's 16 values in each of its four lanes, then columns 4 cq .. 4 cq + 3 of
        // the folded row (fp64 fma over p <= c, in order)
        float yr[BP];
#pragma unroll
        for (int p = 0; p < BP; ++p) yr[p] = __shfl_sync(0xffffffffu, y[p & 3], (lane & ~3) | (p >> 2));
        if (j < lpad) {
            float4 o;
            float* of = &o.x;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int c = 4 * cq + u;
                double acc = 0.0;
#pragma unroll
                for (int p = 0; p < BP; ++p)
                    if (p <= c) acc = fma((double)yr[p], Ms[p * BP + c], acc);
                of[u] = (float)acc;
                cm[u] = fmaxf(cm[u], fabsf(of[u]));
            }
            reinterpret_cast<float4*>(Y1f + j * BP)[cq] = o;
        }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) mxs[jl][4 * cq + u] = cm[u];
    __syncthreads();
    if (threadIdx.x < BP) {
        float m = 0.f;
        for (int q = 0; q < JPB; ++q) m = fmaxf(m, mxs[q][threadIdx.x]);
        atomicMax(cmax + threadIdx.x, __float_as_uint(m));
    }
    if (Y8T) {
        // (cooperative launch) every block's maxima are in: the int8 D stream's digits of Y1f
        // (k_y8_split's work) right here, from L2-hot Y1f, without another launch
        cooperative_groups::this_grid().sync();
        const int rb = 256 / BP;
        const int r = threadIdx.x % rb, c = threadIdx.x / rb;
        const int e = i8_scale_exp(__uint_as_float(((volatile unsigned int*)cmax)[c]));
        if (blockIdx.x == 0 && r == 0) yexp[c] = e;
        for (int64_t k = (int64_t)blockIdx.x * rb + r; k < lpad; k += (int64_t)gridDim.x * rb) {
            int d0, d1, d2;
            digits3(__float2int_rn(ldexpf(__ldcg(Y1f + k * BP + c), e)), d0, d1, d2);
            Y8T[(int64_t)c * lpad + k] = (int8_t)d0;
            Y8T[(int64_t)(BP + c) * lpad + k] = (int8_t)d1;
            Y8T[(int64_t)(2 * BP + c) * lpad + k] = (int8_t)d2;
        }
    }
}

}  // namespace sbmds
