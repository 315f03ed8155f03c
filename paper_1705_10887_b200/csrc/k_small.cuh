// Block subspace iteration kernels (BASELINE.json north_star:
// "block subspace iteration with Cholesky-QR and Rayleigh-Ritz ... a tall-skinny Gram
// X^T X kernel for Cholesky-QR; a single-block Jacobi kernel for the p x p Ritz problem,
// so nothing falls back to the CPU").
//
//   k_gram        G = Y^T Y (and H = X^T Y), fp64 accumulation, deterministic        E2/E5
//   k_chol        G = R^T R (shifted retry on breakdown), Rinv = R^-1, single CTA      E3
//   k_rr          cyclic parallel Jacobi of H, Ritz values/vectors, residuals, conv.  E5
//   k_rotate      out = in * M  (n x b times b x mo, fp64 arithmetic)                  E4/E6
//   k_init_philox X0 ~ N(0,1), counter-based Philox4x32-10 + Box-Muller               E1
//   k_col_argmax, k_finalize   sign canonicalisation and Z = V diag(sqrt(max θ, 0))  E6
#pragma once
#include "common.cuh"

namespace sbmds {

// ------------------------------------------------------------------ E2: tall-skinny Gram
constexpr int kGramPart = 2 * kMaxB * kMaxB + kMaxB;   // per-block partial: G, H, column sums
__host__ __device__ inline int gram_tile_rows(int b) {  // ~32 KB of fp64 per staged tile
    const int b4 = (b + 3) & ~3;
    const int r = 4096 / b4;
    return r > 256 ? 256 : r;
}

// Rows are cut into gridDim.x contiguous ranges. A block stages 64-row tiles of Y (and X)
// in shared memory as fp64 (fp32 -> fp64 is exact, so every product is exact) and splits
// the b4 x b4 output (b4 = b rounded up to 4) into 4x4 micro-tiles; the 256 threads are
// (micro-tile, row-group) pairs, each accumulating 16 (or 32 with H) fp64 FMAs per row.
// Row-group partials are summed in fixed order, then the last block sums the block
// partials in block order: bitwise deterministic.
// cs (optional): column sums 1^T Y (fp64), same fixed-order reductions.
template <bool WITH_H>
__global__ void __launch_bounds__(256) k_gram(int64_t n, int b, const float* __restrict__ Y,
                                              const float* __restrict__ X, double* __restrict__ part,
                                              double* __restrict__ G, double* __restrict__ H,
                                              double* __restrict__ cs, unsigned int* __restrict__ counter) {
    extern __shared__ double gsm[];
    const int b4 = (b + 3) & ~3;
    const int TR = gram_tile_rows(b);
    const int nt = b4 / 4;                 // micro-tiles per side
    const int ntiles = nt * nt;            // <= 256
    const int groups = 256 / ntiles;       // row groups (>= 1)
    double* Ys = gsm;                      // [TR][b4]
    double* Xs = gsm + TR * b4;            // [TR][b4] (WITH_H)
    const int tid = threadIdx.x;
    const int tile = tid % ntiles, grp = tid / ntiles;
    const int ti = tile / nt, tj = tile % nt;
    const bool active = grp < groups;
    double g[4][4], h[4][4], csum[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        csum[i] = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) g[i][j] = h[i][j] = 0.0;
    }
    const int64_t rows_per_blk = (n + gridDim.x - 1) / gridDim.x;
    const int64_t beg = blockIdx.x * rows_per_blk, end = min(n, beg + rows_per_blk);
    for (int64_t r0 = beg; r0 < end; r0 += TR) {
        const int rows = (int)((end - r0) < TR ? (end - r0) : TR);
        __syncthreads();
        for (int e = tid; e < TR * b4; e += 256) {
            const int r = e / b4, c = e % b4;
            const bool ok = r < rows && c < b;
            Ys[e] = ok ? (double)Y[(r0 + r) * b + c] : 0.0;
            if constexpr (WITH_H) Xs[e] = ok ? (double)X[(r0 + r) * b + c] : 0.0;
        }
        __syncthreads();
        if (active) {
            for (int r = grp; r < rows; r += groups) {
                const double* yr = Ys + r * b4;
                double a[4], c[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) { a[i] = yr[4 * ti + i]; c[i] = yr[4 * tj + i]; }
#pragma unroll
                for (int i = 0; i < 4; ++i) csum[i] += c[i];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) g[i][j] = fma(a[i], c[j], g[i][j]);
                if constexpr (WITH_H) {
                    const double* xr = Xs + r * b4;
                    double xa[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) xa[i] = xr[4 * ti + i];
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) h[i][j] = fma(xa[i], c[j], h[i][j]);
                }
            }
        }
    }
    // reduce the row groups in fixed order through shared memory
    __syncthreads();
    double* red = gsm;  // [groups][b4*b4] (+ same for H), then [groups][b4] column sums
    const int bb4 = b4 * b4;
    double* cred = gsm + 2 * groups * bb4;
    if (active && ti == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) cred[grp * b4 + 4 * tj + i] = csum[i];
    }
    if (active) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int pq = (4 * ti + i) * b4 + 4 * tj + j;
                red[grp * bb4 + pq] = g[i][j];
                if constexpr (WITH_H) red[(groups + grp) * bb4 + pq] = h[i][j];
            }
    }
    __syncthreads();
    double* pg = part + (int64_t)blockIdx.x * kGramPart;
    for (int pq = tid; pq < b * b; pq += 256) {
        const int p = pq / b, q = pq % b, e = p * b4 + q;
        double a = 0.0, ah = 0.0;
        for (int k = 0; k < groups; ++k) {
            a += red[k * bb4 + e];
            if constexpr (WITH_H) ah += red[(groups + k) * bb4 + e];
        }
        pg[pq] = a;
        if constexpr (WITH_H) pg[kMaxB * kMaxB + pq] = ah;
    }
    for (int q = tid; q < b; q += 256) {
        double a = 0.0;
        for (int k = 0; k < groups; ++k) a += cred[k * b4 + q];
        pg[2 * kMaxB * kMaxB + q] = a;
    }
    if (last_block_done(counter)) {
        if (cs)
            for (int q = tid; q < b; q += 256) cs[q] = ordered_sum(part + 2 * kMaxB * kMaxB + q, gridDim.x, kGramPart);
        for (int pq = tid; pq < b * b; pq += 256) {
            G[pq] = ordered_sum(part + pq, gridDim.x, kGramPart);
            if constexpr (WITH_H) H[pq] = ordered_sum(part + kMaxB * kMaxB + pq, gridDim.x, kGramPart);
        }
        if (tid == 0) *counter = 0;
    }
}
// Gram on the FP64 tensor cores: mma.sync.m8n8k4.f64 (fp32 -> fp64 is exact, so every product
// is exact and only the fp64 accumulation rounds). A warp walks a contiguous row range 4 rows at
// a time; lane t holds Y[r0 + (t & 3)][8c + (t >> 2)] for each 8-column block c, which is at the
// same time the A fragment of (Y^T)_c (8 x 4, row-major) and the B fragment of Y_c (4 x 8,
// col-major). G (symmetric) needs the NCB(NCB+1)/2 blocks c <= c'; H = X^T Y needs all NCB^2.
// Warp fragments -> shared memory (fixed warp order) -> block partial -> last block, like k_gram.
__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void gtc_cp16(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}

template <int NCB, bool WITH_H>
__global__ void __launch_bounds__(256) k_gram_tc(int64_t n, int b, const float* __restrict__ Y,
                                                 const float* __restrict__ X, double* __restrict__ part,
                                                 double* __restrict__ G, double* __restrict__ H,
                                                 double* __restrict__ cs, unsigned int* __restrict__ counter) {
    constexpr int NPG = NCB * (NCB + 1) / 2;
    constexpr int NPH = WITH_H ? NCB * NCB : 0;
    extern __shared__ double gtc_smem[];   // per-warp G (H reuses it after) + column sums
    auto red = reinterpret_cast<double (*)[NCB * 8][NCB * 8 + 1]>(gtc_smem);
    auto cred = reinterpret_cast<double (*)[NCB * 8]>(gtc_smem + 8 * (NCB * 8) * (NCB * 8 + 1));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int kr = lane & 3, cc = lane >> 2;   // fragment row-in-k and column-in-block
    double g[NPG][2], h[NPH > 0 ? NPH : 1][2], csum[NCB];
#pragma unroll
    for (int i = 0; i < NPG; ++i) g[i][0] = g[i][1] = 0.0;
#pragma unroll
    for (int i = 0; i < (NPH > 0 ? NPH : 1); ++i) h[i][0] = h[i][1] = 0.0;
#pragma unroll
    for (int c = 0; c < NCB; ++c) csum[c] = 0.0;
    const int64_t nw = (int64_t)gridDim.x * 8;
    const int64_t wid = (int64_t)blockIdx.x * 8 + warp;
    const int64_t rows_per_warp = ((n + nw - 1) / nw + 15) & ~int64_t(15);
    const int64_t beg = wid * rows_per_warp, end = min(n, beg + rows_per_warp);
    constexpr int U = 4;   // 4-row groups whose loads are issued together (memory-level parallelism)
    // one 16-row chunk of fragments: y / x values of 4-row group u for this lane
    auto consume = [&](const float (&yf)[U][NCB], const float (&xf)[U][NCB]) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            double y[NCB], x[NCB];
#pragma unroll
            for (int c = 0; c < NCB; ++c) {
                y[c] = (double)yf[u][c];
                csum[c] += y[c];
                if constexpr (WITH_H) x[c] = (double)xf[u][c];
            }
            int pi = 0;
#pragma unroll
            for (int c = 0; c < NCB; ++c)
#pragma unroll
                for (int c2 = c; c2 < NCB; ++c2) dmma_8x8x4(g[pi++], y[c], y[c2]);
            if constexpr (WITH_H) {
#pragma unroll
                for (int c = 0; c < NCB; ++c)
#pragma unroll
                    for (int c2 = 0; c2 < NCB; ++c2) dmma_8x8x4(h[c * NCB + c2], x[c], y[c2]);
            }
        }
    };
    const bool vec = (b % 4 == 0) && ((reinterpret_cast<uintptr_t>(Y) & 15) == 0) &&
                     (!WITH_H || (reinterpret_cast<uintptr_t>(X) & 15) == 0);
    if (vec) {
        // Rows staged through shared memory: a warp copies its next 16 rows (16 b floats, contiguous in
        // Y) with 16-byte cp.async while it works on the current ones (two stages; row pitch b + 8
        // floats: the fragment reads of a 4-row group then hit 32 distinct banks), instead of 4-byte
        // gathers in the fragment layout (0.9 TB/s at b = 32).
        const int pitch = b + 8, cpr = b / 4;   // floats per staged row, 16-byte chunks per row
        float* stg = reinterpret_cast<float*>(gtc_smem) + (size_t)warp * (WITH_H ? 4 : 2) * 16 * pitch;
        auto stage = [&](int64_t r0, int sidx) {
            const int nrow = (int)min((int64_t)16, end - r0);
            for (int q = lane; q < nrow * cpr; q += 32) {
                const int rr = q / cpr, ch = q % cpr;
                gtc_cp16(stg + (sidx * 16 + rr) * pitch + 4 * ch, Y + (r0 + rr) * b + 4 * ch);
                if constexpr (WITH_H) gtc_cp16(stg + ((2 + sidx) * 16 + rr) * pitch + 4 * ch, X + (r0 + rr) * b + 4 * ch);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        if (beg < end) stage(beg, 0);
        int sidx = 0;
        for (int64_t r0 = beg; r0 < end; r0 += 16, sidx ^= 1) {
            if (r0 + 16 < end) {
                stage(r0 + 16, sidx ^ 1);
                asm volatile("cp.async.wait_group 1;" ::: "memory");
            } else {
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            }
            __syncwarp();
            float yf[U][NCB], xf[U][NCB];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const bool ok = r0 + 4 * u + kr < end;
#pragma unroll
                for (int c = 0; c < NCB; ++c) {
                    const int col = 8 * c + cc;
                    const int o = (sidx * 16 + 4 * u + kr) * pitch + col;
                    yf[u][c] = (ok && col < b) ? stg[o] : 0.f;
                    if constexpr (WITH_H) xf[u][c] = (ok && col < b) ? stg[o + 2 * 16 * pitch] : 0.f;
                    else xf[u][c] = 0.f;
                }
            }
            consume(yf, xf);
            __syncwarp();   // every lane has read stage sidx before it is refilled two chunks on
        }
        __syncthreads();   // the staging area is reused for the fragment reduction below
    } else {
    for (int64_t r0 = beg; r0 < end; r0 += 4 * U) {
        float yf[U][NCB], xf[U][NCB];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t r = r0 + 4 * u + kr;
            const bool ok = r < end;
#pragma unroll
            for (int c = 0; c < NCB; ++c) {
                const int col = 8 * c + cc;
                yf[u][c] = (ok && col < b) ? __ldg(Y + r * b + col) : 0.f;
                if constexpr (WITH_H) xf[u][c] = (ok && col < b) ? __ldg(X + r * b + col) : 0.f;
                else xf[u][c] = 0.f;
            }
        }
        consume(yf, xf);
    }
    }
    // column sums: lanes with the same cc hold the same columns
#pragma unroll
    for (int c = 0; c < NCB; ++c) {
        double v = csum[c];
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        if (kr == 0) cred[warp][8 * c + cc] = v;
    }
    // C fragment: lane t holds (row t >> 2, cols 2(t & 3), 2(t & 3) + 1) of each 8 x 8 block
    const int fr = lane >> 2, fc = 2 * (lane & 3);
    {
        int pi = 0;
#pragma unroll
        for (int c = 0; c < NCB; ++c)
#pragma unroll
            for (int c2 = c; c2 < NCB; ++c2) {
                red[warp][8 * c + fr][8 * c2 + fc] = g[pi][0];
                red[warp][8 * c + fr][8 * c2 + fc + 1] = g[pi][1];
                red[warp][8 * c2 + fc][8 * c + fr] = g[pi][0];          // mirror (symmetric)
                red[warp][8 * c2 + fc + 1][8 * c + fr] = g[pi][1];
                ++pi;
            }
    }
    __syncthreads();
    double* pg = part + (int64_t)blockIdx.x * kGramPart;
    for (int pq = threadIdx.x; pq < b * b; pq += 256) {
        const int p = pq / b, q = pq % b;
        double a = 0.0;
        for (int w = 0; w < 8; ++w) a += red[w][p][q];
        pg[pq] = a;
    }
    for (int q = threadIdx.x; q < b; q += 256) {
        double a = 0.0;
        for (int w = 0; w < 8; ++w) a += cred[w][q];
        pg[2 * kMaxB * kMaxB + q] = a;
    }
    if constexpr (WITH_H) {
        __syncthreads();
#pragma unroll
        for (int c = 0; c < NCB; ++c)
#pragma unroll
            for (int c2 = 0; c2 < NCB; ++c2) {
                red[warp][8 * c + fr][8 * c2 + fc] = h[c * NCB + c2][0];
                red[warp][8 * c + fr][8 * c2 + fc + 1] = h[c * NCB + c2][1];
            }
        __syncthreads();
        for (int pq = threadIdx.x; pq < b * b; pq += 256) {
            const int p = pq / b, q = pq % b;
            double a = 0.0;
            for (int w = 0; w < 8; ++w) a += red[w][p][q];
            pg[kMaxB * kMaxB + pq] = a;
        }
    }
    // (counter == NULL: the caller sums the partials with k_gram_sum)
    if (counter && last_block_done(counter)) {
        if (cs)
            for (int q = threadIdx.x; q < b; q += 256) cs[q] = ordered_sum(part + 2 * kMaxB * kMaxB + q, gridDim.x, kGramPart);
        {   // this thread's entries tid + 256 e (b <= 32: at most 4), their partial loads batched together
            double o[4];
            ordered_sum_x4(part, (int)threadIdx.x, b * b, gridDim.x, kGramPart, o);
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if ((int)threadIdx.x + 256 * e < b * b) G[threadIdx.x + 256 * e] = o[e];
            if constexpr (WITH_H) {
                ordered_sum_x4(part + kMaxB * kMaxB, (int)threadIdx.x, b * b, gridDim.x, kGramPart, o);
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if ((int)threadIdx.x + 256 * e < b * b) H[threadIdx.x + 256 * e] = o[e];
            }
        }
        if (threadIdx.x == 0) *counter = 0;
    }
}

// the per-warp fragment reduction, or the row staging (8 warps x 2 stages x 16 rows x (8 NCB + 8) floats,
// twice with H), whichever is larger
template <int NCB>
constexpr size_t gram_tc_smem(bool with_h = true) {
    const size_t red = (size_t)8 * (NCB * 8) * (NCB * 8 + 1 + 1) * sizeof(double);
    const size_t stg = (size_t)8 * (with_h ? 4 : 2) * 16 * (NCB * 8 + 8) * sizeof(float);
    return red > stg ? red : stg;
}

// The block partials of a Gram kernel summed by several blocks instead of the kernel's last block
// (b = 32: 1056 entries over ~300 partials were ~35 us of a 90 us launch in one block): four
// consecutive lanes per entry, each summing a quarter of the partials in order, the first adding
// the four in quarter order -- a fixed order, bitwise reproducible. Entries: G (b x b), H (with_h)
// and the column sums (cs != NULL), at their offsets in a partial.
__global__ void __launch_bounds__(256) k_gram_sum(int b, int nparts, const double* __restrict__ part,
                                                  double* __restrict__ G, double* __restrict__ H,
                                                  double* __restrict__ cs) {
    const int nG = b * b, nH = H ? b * b : 0, nC = cs ? b : 0;
    const int task = blockIdx.x * blockDim.x + threadIdx.x, e = task >> 2, qt = task & 3;
    const int per = (nparts + 3) / 4, q0 = min(nparts, qt * per), q1 = min(nparts, q0 + per);
    const bool live = e < nG + nH + nC;
    int off = 0;
    double* dst = nullptr;
    if (e < nG) { off = e; dst = G + e; }
    else if (e < nG + nH) { off = kMaxB * kMaxB + (e - nG); dst = H + (e - nG); }
    else if (live) { off = 2 * kMaxB * kMaxB + (e - nG - nH); dst = cs + (e - nG - nH); }
    double v = 0.0;
    if (live) v = ordered_sum<16>(part + (int64_t)q0 * kGramPart + off, q1 - q0, kGramPart);
    const double v1 = __shfl_down_sync(0xffffffffu, v, 1), v2 = __shfl_down_sync(0xffffffffu, v, 2),
                 v3 = __shfl_down_sync(0xffffffffu, v, 3);
    if (live && qt == 0) *dst = ((v + v1) + v2) + v3;
}

// dynamic smem: max(2 tiles of TR x b4, 2*groups*b4^2 + groups*b4) doubles
inline size_t gram_smem_bytes(int b) {
    const int b4 = (b + 3) & ~3;
    const int nt = b4 / 4, groups = 256 / (nt * nt);
    const size_t a = (size_t)2 * gram_tile_rows(b) * b4, c = (size_t)2 * groups * b4 * b4 + groups * b4;
    return (a > c ? a : c) * sizeof(double);
}

// ------------------------------------------------------------------ E3: Cholesky + R^-1
// status: 0 ok, 1 ok after the shifted retry, 2 breakdown. G, Rinv are b x b row-major.
// G = R^T R in one thread block (any blockDim >= b; every thread of the block calls it): the
// body of k_chol, also run by the last CTA of the tensor-core sparse step (k_sp8.cuh) right
// after it forms G. A: b x (kMaxB + 1) doubles of shared memory; fail / shift: shared scalars.
__device__ void chol_block(int b, const double* __restrict__ G, double* __restrict__ Rinv, int* __restrict__ status,
                           double (*A)[kMaxB + 1], int* fail_s, double* shift_s) {
    // Warp 0 factors in shared memory with __syncwarp between the b steps (no block barriers);
    // the loops stay rolled -- this runs once per iteration from a cold instruction cache, where
    // a fully unrolled register version measured 2x slower than its hot time. One reciprocal per
    // pivot, products instead of per-element divisions.
    int& fail = *fail_s;
    double& shift = *shift_s;
    const int tid = threadIdx.x;
    for (int attempt = 0; attempt < 2; ++attempt) {
        for (int e = tid; e < b * b; e += blockDim.x) {
            const int i = e / b, j = e % b;
            A[i][j] = 0.5 * (G[i * b + j] + G[j * b + i]);
        }
        if (tid == 0) {
            fail = 0;
            double tr = 0.0;
            for (int i = 0; i < b; ++i) tr += fabs(G[i * b + i]);
            shift = attempt == 0 ? 0.0 : 1e-13 * tr;   // (an all-zero G stays a breakdown)
        }
        __syncthreads();
        if (attempt == 1 && tid < b) A[tid][tid] += shift;
        __syncthreads();
        if (tid < 32) {
            const int lane = tid;
            int f = 0;
#pragma unroll 1
            for (int k = 0; k < b; ++k) {
                const double d = A[k][k];
                if (!(d > 0.0) || !isfinite(d)) {   // (the same value in every lane)
                    f = 1;
                    break;
                }
                const double r = sqrt(d), ri = 1.0 / r;
                __syncwarp();
                for (int j = k + 1 + lane; j < b; j += 32) A[k][j] *= ri;   // row k of R
                if (lane == 0) A[k][k] = r;
                __syncwarp();
                // trailing update A[i][j] -= R[k][i] R[k][j], k < i <= j < b: element e of the
                // m (m + 1) / 2 upper entries, row-major
                const int m = b - k - 1;
                for (int e = lane; e < m * (m + 1) / 2; e += 32) {
                    int i = 0, rem = e;
                    while (rem >= m - i) {
                        rem -= m - i;
                        ++i;
                    }
                    const int ii = k + 1 + i, jj = ii + rem;
                    A[ii][jj] = fma(-A[k][ii], A[k][jj], A[ii][jj]);
                }
                __syncwarp();
            }
            if (lane == 0) fail = f;
        }
        __syncthreads();
        if (!fail) break;
        __syncthreads();
    }
    if (fail) {
        if (tid == 0) *status = 2;
        return;
    }
    // R upper triangular in A (i <= j). Column c of R^-1 by back substitution; thread c keeps its
    // column in row c of A's unused lower triangle (x_i at A[c][i], i < c) and x_c at A[c][kMaxB].
    if (tid < b) {
        const int c = tid;
        A[c][kMaxB] = 1.0 / A[c][c];
        for (int i = c - 1; i >= 0; --i) {
            double sacc = 0.0;
            for (int k = i + 1; k <= c; ++k) sacc = fma(A[i][k], k == c ? A[c][kMaxB] : A[c][k], sacc);
            A[c][i] = -sacc / A[i][i];
        }
        for (int i = 0; i < b; ++i) Rinv[i * b + c] = i < c ? A[c][i] : (i == c ? A[c][kMaxB] : 0.0);
    }
    if (tid == 0) *status = (shift > 0.0) ? 1 : 0;
}

__global__ void __launch_bounds__(256) k_chol(int b, const double* __restrict__ G, double* __restrict__ Rinv,
                                              int* __restrict__ status) {
    __shared__ double A[kMaxB][kMaxB + 1];
    __shared__ int fail;
    __shared__ double shift;
    chol_block(b, G, Rinv, status, A, &fail, &shift);
}

// k_chol for wider blocks (b > 16; round 2): the whole block factors, one barrier-separated
// step per pivot (the trailing update spread over all threads), and R^{-1} row by row from the
// bottom (row i of X = R^{-1} is final once the rows below it are; each step then adds
// R[j][i] X[i][c] into the rows j < i, all (j, c) in parallel). Same status and shifted retry as
// chol_block; deterministic (one thread per element and step). At b = 32 the warp-0 form of
// chol_block took ~0.07 ms (its triangular index decode is O(b) per element per step).
constexpr int kCholParSmem = 2 * kMaxB * (kMaxB + 1) * sizeof(double);
__global__ void __launch_bounds__(256) k_chol_par(int b, const double* __restrict__ G, double* __restrict__ Rinv,
                                                  int* __restrict__ status) {
    extern __shared__ double chol_smem[];
    double (*A)[kMaxB + 1] = reinterpret_cast<double (*)[kMaxB + 1]>(chol_smem);
    double (*X)[kMaxB + 1] = reinterpret_cast<double (*)[kMaxB + 1]>(chol_smem + kMaxB * (kMaxB + 1));
    __shared__ int fail;
    __shared__ double shift;
    const int tid = threadIdx.x;
    for (int attempt = 0; attempt < 2; ++attempt) {
        for (int e = tid; e < b * b; e += blockDim.x) {
            const int i = e / b, j = e % b;
            A[i][j] = 0.5 * (G[i * b + j] + G[j * b + i]);
        }
        if (tid == 0) {
            fail = 0;
            double tr = 0.0;
            for (int i = 0; i < b; ++i) tr += fabs(G[i * b + i]);
            shift = attempt == 0 ? 0.0 : 1e-13 * tr;
        }
        __syncthreads();
        if (attempt == 1 && tid < b) A[tid][tid] += shift;
        __syncthreads();
        for (int k = 0; k < b; ++k) {
            const double d = A[k][k];
            if (!(d > 0.0) || !isfinite(d)) {   // (every thread reads the same value)
                if (tid == 0) fail = 1;
                break;
            }
            const double r = sqrt(d), ri = 1.0 / r;
            __syncthreads();   // A[k][k] read by all
            for (int j = k + 1 + tid; j < b; j += blockDim.x) A[k][j] *= ri;
            if (tid == 0) A[k][k] = r;
            __syncthreads();
            const int m = b - k - 1;
            for (int e = tid; e < m * m; e += blockDim.x) {
                const int i = k + 1 + e / m, j = k + 1 + e % m;
                if (j >= i) A[i][j] = fma(-A[k][i], A[k][j], A[i][j]);
            }
            __syncthreads();
        }
        __syncthreads();
        if (!fail) break;
        __syncthreads();
    }
    if (fail) {
        if (tid == 0) *status = 2;
        return;
    }
    for (int e = tid; e < b * b; e += blockDim.x) X[e / b][e % b] = 0.0;
    __syncthreads();
    for (int i = b - 1; i >= 0; --i) {
        const double rii = 1.0 / A[i][i];
        for (int c = i + tid; c < b; c += blockDim.x) X[i][c] = ((c == i ? 1.0 : 0.0) - X[i][c]) * rii;
        __syncthreads();
        const int w = b - i;   // columns c in [i, b)
        for (int e = tid; e < i * w; e += blockDim.x) {
            const int j = e / w, c = i + e % w;
            X[j][c] = fma(A[j][i], X[i][c], X[j][c]);
        }
        __syncthreads();
    }
    for (int e = tid; e < b * b; e += blockDim.x) {
        const int i = e / b, c = e % b;
        Rinv[e] = c >= i ? X[i][c] : 0.0;
    }
    if (tid == 0) *status = (shift > 0.0) ? 1 : 0;
}

// ------------------------------------------------------------------ E5: Rayleigh-Ritz
constexpr int kRrSmem = 2 * kMaxB * (kMaxB + 1) * sizeof(double);

struct RrOut {
    double theta[kMaxB];     // Ritz values, descending algebraic
    double U[kMaxB * kMaxB]; // U[p*b + j]: component p of Ritz vector j (sorted)
    double resid[kMaxB];     // ||B~ v_j - θ_j v_j|| for all j
    double maxres;           // max_j<m resid_j / max_i |θ_i|
    int converged;
    int n_negative;          // among the top m
    int sweeps;
};

// E6 selection (one block): the top-m algebraic Ritz pairs with the exact null pair (0, 1/sqrt(n))
// merged in (it enters when fewer than m Ritz values are >= 0; reading R10), the R^-1 fold of
// the Ritz vectors V = Y_k (R_k^{-1} U) as the b x m selection matrix Msel, the added constant
// column addc (1/sqrt(n) for the null pair) and the selected eigenvalues theta_out.
__global__ void __launch_bounds__(256) k_select(int b, int m, int64_t n, const RrOut* __restrict__ rr,
                                                const double* __restrict__ Rinv, double* __restrict__ Msel,
                                                double* __restrict__ addc, double* __restrict__ theta_out) {
    __shared__ int src[kMaxB];
    if (threadIdx.x == 0) {
        int r = 0;
        bool zero_used = false;
        for (int j = 0; j < m; ++j) {
            if (!zero_used && (r >= b || rr->theta[r] < 0.0)) {
                zero_used = true;
                src[j] = -1;
            } else {
                src[j] = r++;
            }
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < b * m; e += blockDim.x) {
        const int p = e / m, j = e % m;
        double acc = 0.0;
        if (src[j] >= 0)
            for (int q = p; q < b; ++q) acc += Rinv[p * b + q] * rr->U[q * b + src[j]];
        Msel[p * m + j] = acc;
    }
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
        addc[j] = src[j] < 0 ? 1.0 / sqrt((double)n) : 0.0;
        theta_out[j] = src[j] < 0 ? 0.0 : rr->theta[src[j]];
    }
}


// Parallel cyclic Jacobi (round-robin pair ordering) on sym(H); residuals from the Gram
// G = Y^T Y with Y = B~ X: r_j^2 = u_j^T G u_j - θ_j^2 for orthonormal X.
// With Rinv != null the iterate is X = Y_prev Rinv and Hg holds Y_prev^T (B~X), so
// H = Rinv^T Hg (the R^-1 fold of the eigs loop).
__global__ void __launch_bounds__(256) k_rr(int b, int m, double tol, const double* __restrict__ Hg,
                                            const double* __restrict__ Gg, const double* __restrict__ Rinv,
                                            RrOut* __restrict__ out) {
    extern __shared__ double rr_smem[];
    double (*A)[kMaxB + 1] = reinterpret_cast<double (*)[kMaxB + 1]>(rr_smem);
    double (*V)[kMaxB + 1] = reinterpret_cast<double (*)[kMaxB + 1]>(rr_smem + kMaxB * (kMaxB + 1));
    __shared__ double cs[kMaxB / 2 + 1], sn[kMaxB / 2 + 1];
    __shared__ int pp[kMaxB / 2 + 1], qq[kMaxB / 2 + 1];
    __shared__ double offn, nrm;
    __shared__ int order[kMaxB];
    const int tid = threadIdx.x;
    const int be = b + (b & 1);
    const int np = be / 2;
    if (Rinv) {
        // V <- Hg, then A <- Rinv^T V (V reused as scratch)
        for (int e = tid; e < b * b; e += blockDim.x) V[e / b][e % b] = Hg[e];
        __syncthreads();
        for (int e = tid; e < b * b; e += blockDim.x) {
            const int i = e / b, j = e % b;
            double acc = 0.0;
            for (int p = 0; p <= i; ++p) acc += Rinv[p * b + i] * V[p][j];   // Rinv upper triangular
            A[i][j] = acc;
        }
        __syncthreads();
        for (int e = tid; e < b * b; e += blockDim.x) {
            const int i = e / b, j = e % b;
            V[i][j] = 0.5 * (A[i][j] + A[j][i]);
        }
        __syncthreads();
        for (int e = tid; e < b * b; e += blockDim.x) {
            const int i = e / b, j = e % b;
            A[i][j] = V[i][j];
            V[i][j] = (i == j) ? 1.0 : 0.0;
        }
    } else {
        for (int e = tid; e < b * b; e += blockDim.x) {
            const int i = e / b, j = e % b;
            A[i][j] = 0.5 * (Hg[i * b + j] + Hg[j * b + i]);
            V[i][j] = (i == j) ? 1.0 : 0.0;
        }
    }
    __syncthreads();
    __shared__ double red_o[8], red_f[8];
    int sweep = 0;
    for (; sweep < 40; ++sweep) {
        {   // off-diagonal and total squared norms: every thread, then fixed-order warp / block sums
            double o = 0.0, f = 0.0;
            for (int e = tid; e < b * b; e += blockDim.x) {
                const int i = e / b, j = e % b;
                const double v = A[i][j] * A[i][j];
                f += v;
                if (i != j) o += v;
            }
#pragma unroll
            for (int w = 16; w > 0; w >>= 1) {
                o += __shfl_xor_sync(0xffffffffu, o, w);
                f += __shfl_xor_sync(0xffffffffu, f, w);
            }
            if ((tid & 31) == 0) {
                red_o[tid >> 5] = o;
                red_f[tid >> 5] = f;
            }
            __syncthreads();
            if (tid == 0) {
                double so = 0.0, sf = 0.0;
                for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
                    so += red_o[w];
                    sf += red_f[w];
                }
                offn = so;
                nrm = sf;
            }
            __syncthreads();
        }
        if (!(offn > 1e-30 * nrm) || nrm == 0.0) break;
        for (int round = 0; round < be - 1; ++round) {
            if (tid < np) {
                // round-robin tournament in closed form: player be-1 is fixed, the others rotate
                int p, q;
                if (tid == 0) {
                    p = round;
                    q = be - 1;
                } else {
                    p = (round + tid) % (be - 1);
                    q = (round - tid + be - 1) % (be - 1);
                }
                if (p > q) { const int t = p; p = q; q = t; }
                pp[tid] = p;
                qq[tid] = q;
                double c = 1.0, s = 0.0;
                if (q < b) {
                    const double apq = A[p][q];
                    if (fabs(apq) > 1e-300) {
                        const double th = (A[q][q] - A[p][p]) / (2.0 * apq);
                        const double t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
                        c = 1.0 / sqrt(t * t + 1.0);
                        s = t * c;
                    }
                }
                cs[tid] = c;
                sn[tid] = s;
            }
            __syncthreads();
            // rows: A <- J^T A
            for (int e = tid; e < np * b; e += blockDim.x) {
                const int pr = e / b, k = e % b;
                const int p = pp[pr], q = qq[pr];
                if (q < b) {
                    const double c = cs[pr], s = sn[pr];
                    const double ap = A[p][k], aq = A[q][k];
                    A[p][k] = c * ap - s * aq;
                    A[q][k] = s * ap + c * aq;
                }
            }
            __syncthreads();
            // columns: A <- A J, V <- V J
            for (int e = tid; e < np * b; e += blockDim.x) {
                const int pr = e / b, k = e % b;
                const int p = pp[pr], q = qq[pr];
                if (q < b) {
                    const double c = cs[pr], s = sn[pr];
                    const double ap = A[k][p], aq = A[k][q];
                    A[k][p] = c * ap - s * aq;
                    A[k][q] = s * ap + c * aq;
                    const double vp = V[k][p], vq = V[k][q];
                    V[k][p] = c * vp - s * vq;
                    V[k][q] = s * vp + c * vq;
                }
            }
            __syncthreads();
        }
    }
    if (tid == 0) {
        for (int i = 0; i < b; ++i) order[i] = i;
        for (int i = 0; i < b; ++i) {  // selection sort, descending θ, ties -> lower index
            int best = i;
            for (int j = i + 1; j < b; ++j)
                if (A[order[j]][order[j]] > A[order[best]][order[best]]) best = j;
            const int t = order[i]; order[i] = order[best]; order[best] = t;
        }
        out->sweeps = sweep;
    }
    __syncthreads();
    for (int e = tid; e < b * b; e += blockDim.x) {
        const int p = e / b, j = e % b;
        out->U[p * b + j] = V[p][order[j]];
    }
    if (tid < b) out->theta[tid] = A[order[tid]][order[tid]];
    // residuals: thread j computes u_j^T G u_j
    if (tid < b) {
        const int j = order[tid];
        double s = 0.0;
        for (int p = 0; p < b; ++p) {
            double gp = 0.0;
            for (int q = 0; q < b; ++q) gp += Gg[p * b + q] * V[q][j];
            s += V[p][j] * gp;
        }
        const double th = A[j][j];
        out->resid[tid] = sqrt(fmax(s - th * th, 0.0));
    }
    __syncthreads();
    if (tid == 0) {
        double tmax = 0.0;
        for (int i = 0; i < b; ++i) tmax = fmax(tmax, fabs(A[i][i]));
        double mr = 0.0;
        int neg = 0;
        for (int j = 0; j < m; ++j) {
            mr = fmax(mr, out->resid[j]);
            if (out->theta[j] < 0.0) ++neg;
        }
        out->maxres = tmax > 0.0 ? mr / tmax : 0.0;
        out->converged = (tol > 0.0 && out->maxres <= tol) ? 1 : 0;
        out->n_negative = neg;
    }
}

// ------------------------------------------------------------------ E4/E6: out = in * M
// in: n x b (row stride b, b <= BT), M: b x mo fp64 row-major (leading dim ldm), out: n x mo.
// One thread per row, fp64 arithmetic in column chunks of 16; M is broadcast from shared
// memory. addc (optional, mo): a constant added to column c (the exact null eigenvector
// 1/sqrt(n) of B~, "J 1 = 0", when it belongs to the top m).
// cs_part (optional): also produce s = 1^T out (fp64: warp sums -> per-warp smem rows ->
// block partial -> last block, fixed order) = A1 of the next apply, so the eigs loop never
// re-reads X for its column sums.
// (CW: output columns formed together; 4 for the final V = Y (R^-1 U) with m <= 4 columns, where
// 16 predicated accumulators per row made the kernel instruction-bound)
template <int BT, int CW = 16>
__global__ void __launch_bounds__(256) k_rotate(int64_t n, int b, int mo, int ldm, const float* __restrict__ in,
                                                const double* __restrict__ M, float* __restrict__ out,
                                                const double* __restrict__ addc, double* __restrict__ cs_part,
                                                double* __restrict__ cs_out, unsigned int* __restrict__ counter) {
    __shared__ double Ms[kMaxB * kMaxB];
    __shared__ double As[kMaxB];
    __shared__ double red[8][kMaxB];
    for (int e = threadIdx.x; e < b * mo; e += blockDim.x) Ms[e] = M[(e / mo) * ldm + (e % mo)];
    for (int e = threadIdx.x; e < mo; e += blockDim.x) As[e] = addc ? addc[e] : 0.0;
    for (int e = threadIdx.x; e < 8 * kMaxB; e += blockDim.x) (&red[0][0])[e] = 0.0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool want_cs = cs_part != nullptr;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
        const int64_t i = base + threadIdx.x;
        const bool act = i < n;
        float y[BT];
        const float* row = in + (act ? i : 0) * b;
        if ((b & 3) == 0) {
#pragma unroll
            for (int p4 = 0; p4 < BT / 4; ++p4) {
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (act && 4 * p4 < b) v = __ldg(reinterpret_cast<const float4*>(row) + p4);
                y[4 * p4] = v.x; y[4 * p4 + 1] = v.y; y[4 * p4 + 2] = v.z; y[4 * p4 + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int p = 0; p < BT; ++p) y[p] = (act && p < b) ? __ldg(row + p) : 0.f;
        }
        for (int c0 = 0; c0 < mo; c0 += CW) {
            double acc[CW];
#pragma unroll
            for (int c = 0; c < CW; ++c) acc[c] = (c0 + c < mo) ? As[c0 + c] : 0.0;
#pragma unroll
            for (int p = 0; p < BT; ++p) {
                if (p < b) {
                    const double yp = (double)y[p];
                    const double* mr = Ms + p * mo + c0;
#pragma unroll
                    for (int c = 0; c < CW; ++c)
                        if (c0 + c < mo) acc[c] = fma(yp, mr[c], acc[c]);
                }
            }
            float* orow = out + i * mo + c0;
#pragma unroll
            for (int c = 0; c < CW; ++c) {
                float v = 0.f;
                if (c0 + c < mo) {
                    v = (float)acc[c];
                    if (act) orow[c] = v;
                }
                if (want_cs && c0 + c < mo) {
                    const double sv = warp_sum(act ? (double)v : 0.0);
                    if (lane == 0) red[warp][c0 + c] += sv;
                }
            }
        }
    }
    if (!want_cs) return;
    __syncthreads();
    if (threadIdx.x < mo) {
        double v = 0.0;
        for (int w = 0; w < 8; ++w) v += red[w][threadIdx.x];
        cs_part[blockIdx.x * kMaxB + threadIdx.x] = v;
    }
    if (last_block_done(counter)) {
        if (threadIdx.x < mo) cs_out[threadIdx.x] = ordered_sum(cs_part + threadIdx.x, gridDim.x, kMaxB);
        if (threadIdx.x == 0) *counter = 0;
    }
}

// Y1 (l x bp, first b columns) <- Y1 Rinv: the R^-1 fold (S^T (Y R^-1) - w (1^T Y R^-1)^T
// = (S^T Y - w (1^T Y)^T) R^-1), so the orthonormal iterate X = Y R^-1 is never formed.
// Element-parallel: a block stages 256/bp rows in shared memory, each thread forms one
// output entry in fp64 (R^-1 upper triangular) and writes it back in place.
__global__ void __launch_bounds__(256) k_y1_rot(int64_t l, int b, int bp, const double* __restrict__ Rinv,
                                                float* __restrict__ Y1) {
    __shared__ double Ms[kMaxB * kMaxB];
    __shared__ float ys[256];
    for (int e = threadIdx.x; e < b * b; e += blockDim.x) Ms[e] = Rinv[e];
    const int rb = 256 / bp;
    const int r = threadIdx.x / bp, c = threadIdx.x % bp;
    for (int64_t j0 = (int64_t)blockIdx.x * rb; j0 < l; j0 += (int64_t)gridDim.x * rb) {
        __syncthreads();
        const int64_t j = j0 + r;
        ys[threadIdx.x] = (j < l) ? Y1[j * bp + c] : 0.f;
        __syncthreads();
        if (j < l && c < b) {
            double acc = 0.0;
            for (int p = 0; p <= c; ++p) acc = fma((double)ys[r * bp + p], Ms[p * b + c], acc);
            Y1[j * bp + c] = (float)acc;
        }
    }
}

// ------------------------------------------------------------------ E1: Philox N(0,1)
__device__ __forceinline__ void philox4x32_10(uint32_t ctr[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * ctr[0];
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * ctr[2];
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ ctr[1] ^ k0;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ ctr[3] ^ k1;
        ctr[1] = (uint32_t)p1;
        ctr[3] = (uint32_t)p0;
        ctr[0] = n0;
        ctr[2] = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

// Element ge of the global n x b block is output (ge & 3) of the Philox call with counter ge >> 2:
// the four 32-bit words of a call give two Box-Muller pairs (r cos, r sin), in fp32 (the initial
// block only has to be generic). A thread forms one call's four normals and stores those inside
// [e0, e0 + total) (e0: the global index of X's first element -- a shard's rows continue the
// global sequence, so the sharded and the unsharded solve start from the same block).
__global__ void k_init_philox(int64_t n, int b, uint64_t seed, float* __restrict__ X, int64_t e0) {
    const int64_t total = n * b;
    const int64_t q0 = e0 >> 2, q1 = (e0 + total + 3) >> 2;
    const bool vec = (e0 & 3) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0;
    for (int64_t q = q0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < q1; q += (int64_t)gridDim.x * blockDim.x) {
        uint32_t ctr[4] = {(uint32_t)q, (uint32_t)(q >> 32), 0x5eed5eedu, 0u};
        philox4x32_10(ctr, (uint32_t)seed, (uint32_t)(seed >> 32));
        float z[4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float u1 = (float)((ctr[2 * h] >> 8) + 1u) * (1.0f / 16777216.0f);   // (0, 1], exact
            const float u2 = (float)(ctr[2 * h + 1] >> 8) * (1.0f / 16777216.0f);        // [0, 1)
            const float r = sqrtf(-2.0f * logf(u1));
            float sn, cs;
            sincospif(2.0f * u2, &sn, &cs);
            z[2 * h] = r * cs;
            z[2 * h + 1] = r * sn;
        }
        const int64_t e = 4 * q - e0;   // local index of z[0]
        if (vec && e + 3 < total) {
            *reinterpret_cast<float4*>(X + e) = make_float4(z[0], z[1], z[2], z[3]);
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (e + i >= 0 && e + i < total) X[e + i] = z[i];
        }
    }
}

// ------------------------------------------------------------------ E6: signs and Z
// Per column the entry of largest |v| (ties -> lowest row); sign[c] = its sign.
__global__ void __launch_bounds__(256) k_col_argmax(int64_t n, int mo, const float* __restrict__ V,
                                                    float* __restrict__ pval, long long* __restrict__ pidx,
                                                    float* __restrict__ sign, unsigned int* __restrict__ counter) {
    __shared__ float bv[256];
    __shared__ long long bi[256];
    const int tid = threadIdx.x;
    const int rps = 256 / mo;
    const int c = tid % mo, r0 = tid / mo;
    const int64_t rows_per_blk = (n + gridDim.x - 1) / gridDim.x;
    const int64_t beg = blockIdx.x * rows_per_blk, end = min(n, beg + rows_per_blk);
    float best = -1.f;
    long long bidx = -1;
    if (r0 < rps)
        for (int64_t i = beg + r0; i < end; i += rps) {
            const float a = fabsf(V[i * mo + c]);
            if (a > best) { best = a; bidx = i; }   // rows visited in increasing order
        }
    bv[tid] = best;
    bi[tid] = bidx;
    __syncthreads();
    if (tid < mo) {
        for (int q = 1; q < rps; ++q) {
            const float a = bv[q * mo + tid];
            const long long ii = bi[q * mo + tid];
            if (ii >= 0 && (a > best || (a == best && (bidx < 0 || ii < bidx)))) { best = a; bidx = ii; }
        }
        pval[blockIdx.x * kMaxB + tid] = best;
        pidx[blockIdx.x * kMaxB + tid] = bidx;
    }
    if (last_block_done(counter)) {
        if (tid < mo) {
            float bb = -1.f;
            long long ii = -1;
            for (unsigned int q = 0; q < gridDim.x; ++q) {
                const float a = pval[q * kMaxB + tid];
                const long long j = pidx[q * kMaxB + tid];
                if (j >= 0 && (a > bb || (a == bb && (ii < 0 || j < ii)))) { bb = a; ii = j; }
            }
            sign[tid] = (ii >= 0 && V[ii * mo + tid] < 0.f) ? -1.f : 1.f;
        }
        if (tid == 0) *counter = 0;
    }
}

// Sharded E6 (sbmds.cu eigs_shard): per column the key (|v| bits << 32 | (2^31 - 1 - global row))
// of this rank's rows -- its max over the ranks is the global largest |v|, ties to the lowest
// row -- and then the sign of V at that row from the rank that holds it (0 elsewhere).
__global__ void __launch_bounds__(256) k_col_key(int64_t n, int mo, const float* __restrict__ V, int64_t row0,
                                                 unsigned long long* __restrict__ key) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * mo; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / mo;
        const int c = (int)(e % mo);
        const unsigned long long k = ((unsigned long long)__float_as_uint(fabsf(V[e])) << 32) |
                                     (unsigned long long)(0x7FFFFFFFll - (row0 + r));
        atomicMax(key + c, k);
    }
}

__global__ void k_key_sign(int64_t n, int mo, const float* __restrict__ V, int64_t row0,
                           const unsigned long long* __restrict__ key, float* __restrict__ sgn) {
    const int c = threadIdx.x;
    if (c >= mo) return;
    const int64_t r = 0x7FFFFFFFll - (int64_t)(key[c] & 0xFFFFFFFFull) - row0;
    sgn[c] = (r >= 0 && r < n) ? (V[r * mo + c] < 0.f ? -1.f : 1.f) : 0.f;
}

__global__ void k_vec_rinv(int b, const double* __restrict__ v, const double* __restrict__ Rinv, double* __restrict__ t) {
    const int c = threadIdx.x;
    if (c >= b) return;
    double acc = 0.0;
    for (int p = 0; p <= c; ++p) acc = fma(v[p], Rinv[p * b + c], acc);   // Rinv upper triangular
    t[c] = acc;
}

__global__ void k_finalize(int64_t n, int mo, const float* __restrict__ sign, const double* __restrict__ theta,
                           float* __restrict__ V, float* __restrict__ Z) {
    const int64_t total = n * mo;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(e % mo);
        const float v = V[e] * sign[c];
        V[e] = v;
        if (Z) Z[e] = (float)((double)v * sqrt(fmax(theta[c], 0.0)));
    }
}

}  // namespace sbmds
