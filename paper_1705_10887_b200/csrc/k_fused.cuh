// Fused A5 + (next apply's) A2 + E2 for the eigensolver ("fused sparse step").
//
// Inside sbmds_eigs the block Y = B~ X produced by A5 is consumed by exactly two things before
// the next apply: the Gram step (G = Y^T Y, column sums s = 1^T Y, and at Rayleigh-Ritz steps
// H' = Y_prev^T Y) and the next apply's A2 (S^T Y, centred with s). Both are linear in the rows
// of Y, and S is row-blocked (k_blocked.cuh): the 256 rows a CTA forms for A5 are exactly the
// rows of its block-local CSC. So one persistent kernel, per 256-row block B:
//   1. stages Y2[dict_B] (and, at RR steps, the block's rows of Y_prev) in shared memory,
//   2. forms the block's rows of Y = -1/2 (S Y2 - 1 t^T) (as k_blk_spmm), writes them to HBM
//      once and keeps them in shared memory,
//   3. writes the S^T partials P1[d] for the block's dictionary entries d (as k_blk_spmmt,
//      fixed order over the block-local CSC) -- k_blk_reduce later sums each landmark's
//      partials over blocks in ascending block order and subtracts w s^T,
//   4. accumulates Y_B^T Y_B, 1^T Y_B (and Y_prev,B^T Y_B) on the FP64 tensor cores into
//      per-warp fragments (as k_gram_tc: products of fp32 values are exact in fp64).
// After its last block a CTA reduces its warps in fixed order into one partial, and the last
// CTA to finish sums the CTA partials in CTA order: G, H', s are bitwise reproducible, as are Y
// and P1. This replaces the CSC SpMM pass (3.6 GB of L2 gathers at config 4) and the Gram's
// separate read of Y.
#pragma once
#include "common.cuh"
#include "k_blocked.cuh"
#include "k_small.cuh"

namespace sbmds {

template <int LPR, bool WITH_H>
__global__ void __launch_bounds__(256) k_blk_spmm_fused(
    int64_t n, int64_t nblk, int b, const int32_t* __restrict__ rp, const uint16_t* __restrict__ lcol,
    const float* __restrict__ val, const int32_t* __restrict__ dict, const int32_t* __restrict__ dict_off,
    uint32_t umax, const float* __restrict__ Y2, const double* __restrict__ t, float* __restrict__ Y,
    const int32_t* __restrict__ lcp, const uint8_t* __restrict__ lrow, const float* __restrict__ lval,
    float* __restrict__ P1, const float* __restrict__ Yprev, double* __restrict__ part, double* __restrict__ G,
    double* __restrict__ H, double* __restrict__ cs, unsigned int* __restrict__ counter) {
    constexpr int BP = 4 * LPR;                  // b == bp (power of two, multiple of 4)
    constexpr int NCB = BP < 8 ? 1 : BP / 8;     // 8-column blocks of the Gram
    constexpr int NPG = NCB * (NCB + 1) / 2;
    constexpr int NPH = WITH_H ? NCB * NCB : 0;
    constexpr int G_ = 32 / LPR;                 // row / entry groups per warp
    constexpr int NV = BP / 4;
    extern __shared__ float4 fsm[];
    float4* ys4 = fsm;                                   // [umax][NV]   Y2[dict_B]
    float* yrow = reinterpret_cast<float*>(fsm + (size_t)umax * NV);   // [kRB][BP]
    float* yprv = yrow + kRB * BP;                       // [kRB][BP]   (WITH_H)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / LPR, q = lane % LPR;
    const unsigned gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (g * LPR));
    const double t0 = t[4 * q], t1 = t[4 * q + 1], t2 = t[4 * q + 2], t3 = t[4 * q + 3];
    const int kr = lane & 3, cc = lane >> 2;     // DMMA fragment row-in-k, column-in-block

    double gacc[NPG][2], hacc[NPH > 0 ? NPH : 1][2], csum[NCB];
#pragma unroll
    for (int i = 0; i < NPG; ++i) gacc[i][0] = gacc[i][1] = 0.0;
#pragma unroll
    for (int i = 0; i < (NPH > 0 ? NPH : 1); ++i) hacc[i][0] = hacc[i][1] = 0.0;
#pragma unroll
    for (int c = 0; c < NCB; ++c) csum[c] = 0.0;

    for (int64_t B = blockIdx.x; B < nblk; B += gridDim.x) {
        const int32_t d0 = dict_off[B], u = dict_off[B + 1] - d0;
        const int64_t r0 = B * kRB;
        const int rows = (int)((n - r0) < kRB ? (n - r0) : kRB);
        // 1. stage Y2[dict_B] (and Y_prev rows)
        for (int e = threadIdx.x; e < u * NV; e += blockDim.x) {
            const int i = e / NV, qq = e % NV;
            ys4[e] = __ldg(reinterpret_cast<const float4*>(Y2 + (int64_t)dict[d0 + i] * BP) + qq);
        }
        if constexpr (WITH_H) {
            for (int e = threadIdx.x; e < kRB * NV; e += blockDim.x) {
                const int r = e / NV;
                reinterpret_cast<float4*>(yprv)[e] =
                    r < rows ? __ldg(reinterpret_cast<const float4*>(Yprev + (r0 + r) * b) + e % NV)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        __syncthreads();
        // 2. rows of Y = -1/2 (S Y2 - 1 t^T): HBM once, shared memory for 3 and 4
        for (int r = warp * G_ + g; r < kRB; r += 8 * G_) {   // the same trip count for every lane
            const bool live = r < rows;
            const int64_t i = r0 + r;
            const int32_t beg = live ? rp[i] : 0, end = live ? rp[i + 1] : 0;
            const int maxlen = __reduce_max_sync(0xffffffffu, (unsigned)(end - beg));
            const float4 acc = blk_row_sum<LPR>(beg, end, maxlen, q, lcol, val, ys4, NV);
            float4 out = make_float4(0.f, 0.f, 0.f, 0.f);
            if (live) {
                out.x = (float)(-0.5 * ((double)acc.x - t0));
                out.y = (float)(-0.5 * ((double)acc.y - t1));
                out.z = (float)(-0.5 * ((double)acc.z - t2));
                out.w = (float)(-0.5 * ((double)acc.w - t3));
                reinterpret_cast<float4*>(Y + i * b)[q] = out;
            }
            reinterpret_cast<float4*>(yrow + r * BP)[q] = out;
        }
        __syncthreads();
        // 3. S^T partials of the block's dictionary entries (next apply's A2)
        if (P1) {
            for (int di = warp * G_ + g; di < u; di += 8 * G_) {
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
                        const float4 x = reinterpret_cast<const float4*>(yrow + r * BP)[q];
                        acc.x = fmaf(v, x.x, acc.x);
                        acc.y = fmaf(v, x.y, acc.y);
                        acc.z = fmaf(v, x.z, acc.z);
                        acc.w = fmaf(v, x.w, acc.w);
                    }
                }
                reinterpret_cast<float4*>(P1 + (int64_t)d * BP)[q] = acc;
            }
        }
        // 4. Gram fragments: warp w takes rows 32w .. 32w+31, 4 at a time
#pragma unroll 2
        for (int s4 = 0; s4 < 8; ++s4) {
            const int r = 32 * warp + 4 * s4 + kr;
            double y[NCB], x[NCB];
#pragma unroll
            for (int c = 0; c < NCB; ++c) {
                const int col = 8 * c + cc;
                y[c] = col < BP ? (double)yrow[r * BP + col] : 0.0;
                csum[c] += y[c];
                if constexpr (WITH_H) x[c] = col < BP ? (double)yprv[r * BP + col] : 0.0;
            }
            int pi = 0;
#pragma unroll
            for (int c = 0; c < NCB; ++c)
#pragma unroll
                for (int c2 = c; c2 < NCB; ++c2) dmma_8x8x4(gacc[pi++], y[c], y[c2]);
            if constexpr (WITH_H) {
#pragma unroll
                for (int c = 0; c < NCB; ++c)
#pragma unroll
                    for (int c2 = 0; c2 < NCB; ++c2) dmma_8x8x4(hacc[c * NCB + c2], x[c], y[c2]);
            }
        }
        __syncthreads();   // shared memory is restaged by the next block
    }

    // ---- CTA partial (fixed warp order), then the last CTA sums the partials in CTA order
    auto red = reinterpret_cast<double (*)[NCB * 8][NCB * 8 + 1]>(fsm);
    auto cred = reinterpret_cast<double (*)[NCB * 8]>(reinterpret_cast<double*>(fsm) + 8 * (NCB * 8) * (NCB * 8 + 1));
#pragma unroll
    for (int c = 0; c < NCB; ++c) {
        double v = csum[c];
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        if (kr == 0) cred[warp][8 * c + cc] = v;
    }
    const int fr = lane >> 2, fc = 2 * (lane & 3);
    {
        int pi = 0;
#pragma unroll
        for (int c = 0; c < NCB; ++c)
#pragma unroll
            for (int c2 = c; c2 < NCB; ++c2) {
                red[warp][8 * c + fr][8 * c2 + fc] = gacc[pi][0];
                red[warp][8 * c + fr][8 * c2 + fc + 1] = gacc[pi][1];
                red[warp][8 * c2 + fc][8 * c + fr] = gacc[pi][0];
                red[warp][8 * c2 + fc + 1][8 * c + fr] = gacc[pi][1];
                ++pi;
            }
    }
    __syncthreads();
    double* pg = part + (int64_t)blockIdx.x * kGramPart;
    for (int pq = threadIdx.x; pq < b * b; pq += 256) {
        const int p = pq / b, qq = pq % b;
        double a = 0.0;
        for (int w = 0; w < 8; ++w) a += red[w][p][qq];
        pg[pq] = a;
    }
    for (int qq = threadIdx.x; qq < b; qq += 256) {
        double a = 0.0;
        for (int w = 0; w < 8; ++w) a += cred[w][qq];
        pg[2 * kMaxB * kMaxB + qq] = a;
    }
    if constexpr (WITH_H) {
        __syncthreads();
#pragma unroll
        for (int c = 0; c < NCB; ++c)
#pragma unroll
            for (int c2 = 0; c2 < NCB; ++c2) {
                red[warp][8 * c + fr][8 * c2 + fc] = hacc[c * NCB + c2][0];
                red[warp][8 * c + fr][8 * c2 + fc + 1] = hacc[c * NCB + c2][1];
            }
        __syncthreads();
        for (int pq = threadIdx.x; pq < b * b; pq += 256) {
            const int p = pq / b, qq = pq % b;
            double a = 0.0;
            for (int w = 0; w < 8; ++w) a += red[w][p][qq];
            pg[kMaxB * kMaxB + pq] = a;
        }
    }
    if (last_block_done(counter)) {
        for (int qq = threadIdx.x; qq < b; qq += 256) cs[qq] = ordered_sum(part + 2 * kMaxB * kMaxB + qq, gridDim.x, kGramPart);
        for (int pq = threadIdx.x; pq < b * b; pq += 256) {
            G[pq] = ordered_sum(part + pq, gridDim.x, kGramPart);
            if constexpr (WITH_H) H[pq] = ordered_sum(part + kMaxB * kMaxB + pq, gridDim.x, kGramPart);
        }
        if (threadIdx.x == 0) *counter = 0;
    }
}

// dynamic shared memory of k_blk_spmm_fused (also holds the final reduction scratch)
inline size_t fused_smem_bytes(uint32_t umax, int bp, bool with_h) {
    const size_t stage = (size_t)umax * bp * 4 + (size_t)kRB * bp * 4 * (with_h ? 2 : 1);
    const int ncb = bp < 8 ? 1 : bp / 8;
    const size_t redb = (size_t)8 * (ncb * 8) * (ncb * 8 + 1) * 8 + (size_t)8 * ncb * 8 * 8;
    return stage > redb ? stage : redb;
}

}  // namespace sbmds
