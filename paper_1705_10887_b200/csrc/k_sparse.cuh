// Sparse stages of the sBMDS operator apply.
//
//   B~ X = -1/2 J S D S^T J X with J S = S - 1 w^T, w = S^T 1 / n, so
//     s  = 1^T X                          k_colsum        (A1, "J ... rank-one")
//     Y1 = S^T X - w s^T                   k_spmm_csc_*    (A2, right-multiply by P^T)
//     Y2 = D Y1,  t = w^T Y2               k_dstream.cuh   (A3, A4)
//     Y  = -1/2 (S Y2 - 1 t^T)             k_spmm_csr_*    (A5, left-multiply by P)
// No n-length centred copy is formed; every reduction has a fixed order (no atomics on
// values), so results are bitwise deterministic.
#pragma once
#include "common.cuh"

namespace sbmds {

// ------------------------------------------------------------------ create-time helpers
__global__ void k_rowptr_to_i32(int64_t n, const int64_t* __restrict__ rp64, int32_t* __restrict__ rp32,
                                int64_t nnz, int* __restrict__ bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = rp64[i];
        const bool ok = v >= 0 && v <= nnz && (i == 0 ? v == 0 : true) && (i == n ? v == nnz : true) &&
                        (i == 0 || rp64[i - 1] <= v);
        if (!ok) atomicOr(bad, 1);
        rp32[i] = (int32_t)v;
    }
}

// rowof[e] = row of stored entry e; checks 0 <= col < l and finite values.
__global__ void k_expand_rows(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                              const float* __restrict__ val, int64_t l, int32_t* __restrict__ rowof,
                              int* __restrict__ bad) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        for (int32_t e = rp[i] + lane; e < rp[i + 1]; e += 32) {
            rowof[e] = (int32_t)i;
            const int32_t c = col[e];
            if (c < 0 || c >= l || !isfinite(val[e])) atomicOr(bad, 2);
        }
    }
}

__global__ void k_iota(int32_t n, int32_t* __restrict__ out) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = i;
}

// After a stable sort of (col, entry) pairs: CSC row index / value gathers.
__global__ void k_gather_csc(int32_t nnz, const int32_t* __restrict__ perm, const int32_t* __restrict__ rowof,
                             const float* __restrict__ val, int32_t* __restrict__ row_idx,
                             float* __restrict__ cval) {
    for (int32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += gridDim.x * blockDim.x) {
        const int32_t e = perm[p];
        row_idx[p] = rowof[e];
        cval[p] = val[e];
    }
}

// col_ptr[c] = first position of column >= c in the sorted column keys (binary search).
__global__ void k_col_ptr(int64_t l, int32_t nnz, const int32_t* __restrict__ keys,
                          int32_t* __restrict__ col_ptr) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= l;
         c += (int64_t)gridDim.x * blockDim.x) {
        int32_t lo = 0, hi = nnz;
        while (lo < hi) {
            const int32_t mid = lo + ((hi - lo) >> 1);
            if (keys[mid] < c) lo = mid + 1; else hi = mid;
        }
        col_ptr[c] = lo;
    }
}

// w_j = (1/n) Σ_i S_ij  (column sums, fixed order) and the spatial key of column j
// (median row of its support) used to order the CSC SpMM for L2 locality.
__global__ void k_colstats(int64_t l, int64_t n, const int32_t* __restrict__ col_ptr,
                           const int32_t* __restrict__ row_idx, const float* __restrict__ cval,
                           double* __restrict__ w, int32_t* __restrict__ key) {
    const int lane = threadIdx.x & 31;
    for (int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; j < l;
         j += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int32_t b = col_ptr[j], e = col_ptr[j + 1];
        double s = 0.0;
        for (int32_t p = b + lane; p < e; p += 32) s += (double)cval[p];
        s = warp_sum(s);
        if (lane == 0) {
            w[j] = s / (double)n;
            key[j] = (e > b) ? row_idx[b + ((e - b) >> 1)] : 0;
        }
    }
}

// max |Σ_j S_ij - 1| over rows (diagnostic: PoU S has rows summing to 1).
__global__ void k_rowsum_dev(int64_t n, const int32_t* __restrict__ rp, const float* __restrict__ val,
                             unsigned long long* __restrict__ out_bits) {
    const int lane = threadIdx.x & 31;
    double dmax = 0.0;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        double s = 0.0;
        for (int32_t e = rp[i] + lane; e < rp[i + 1]; e += 32) s += (double)val[e];
        s = warp_sum(s);
        dmax = fmax(dmax, fabs(s - 1.0));
    }
    if (lane == 0) atomicMax(out_bits, (unsigned long long)__double_as_longlong(dmax));
}

// |D_ij - D_ji| max and a finiteness check (SBMDS_VALIDATE). Order-free max -> atomic ok.
__global__ void k_check_sym(int64_t l, int64_t ld, const float* __restrict__ D,
                            unsigned int* __restrict__ maxdiff_bits, unsigned int* __restrict__ maxabs_bits,
                            int* __restrict__ bad) {
    __shared__ float tile[32][33];
    const int64_t bi = blockIdx.y * 32, bj = blockIdx.x * 32;
    if (bj > bi) return;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    float md = 0.f, ma = 0.f;
    for (int r = ty; r < 32; r += 8) {
        const int64_t i = bj + r, j = bi + tx;
        tile[r][tx] = (i < l && j < l) ? D[i * ld + j] : 0.f;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int64_t i = bi + r, j = bj + tx;
        if (i < l && j < l) {
            const float a = D[i * ld + j], b = tile[tx][r];
            if (!isfinite(a)) atomicOr(bad, 4);
            md = fmaxf(md, fabsf(a - b));
            ma = fmaxf(ma, fabsf(a));
        }
    }
    atomicMax(maxdiff_bits, __float_as_uint(md));
    atomicMax(maxabs_bits, __float_as_uint(ma));
}

// ------------------------------------------------------------------ A1: s = 1^T X  (fp64)
// Block partials over row ranges, then the last block sums them in block order.
__global__ void __launch_bounds__(256) k_colsum(int64_t n, int b, const float* __restrict__ X, double* __restrict__ part,
                                                double* __restrict__ s, unsigned int* __restrict__ counter) {
    __shared__ double red[256];
    const int rps = blockDim.x / b;                 // rows per step (b <= 64 -> >= 4)
    const int t = threadIdx.x;
    const int c = t % b, r0 = t / b;
    const int64_t rows_per_blk = (n + gridDim.x - 1) / gridDim.x;
    const int64_t beg = blockIdx.x * rows_per_blk, end = min(n, beg + rows_per_blk);
    // four independent partial sums (rows i, i + rps, i + 2 rps, i + 3 rps of each step of
    // 4 rps) keep four loads in flight; they are combined in a fixed order
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (r0 < rps) {
        int64_t i = beg + r0;
        for (; i + 3 * rps < end; i += 4 * rps) {
            const float x0 = X[i * b + c], x1 = X[(i + rps) * b + c];
            const float x2 = X[(i + 2 * rps) * b + c], x3 = X[(i + 3 * rps) * b + c];
            a0 += (double)x0; a1 += (double)x1; a2 += (double)x2; a3 += (double)x3;
        }
        for (; i < end; i += rps) a0 += (double)X[i * b + c];
    }
    red[t] = (r0 < rps) ? (a0 + a1) + (a2 + a3) : 0.0;
    __syncthreads();
    if (t < b) {
        double v = 0.0;
        for (int q = 0; q < rps; ++q) v += red[q * b + t];
        part[blockIdx.x * kMaxB + t] = v;
    }
    if (last_block_done(counter)) {
        ordered_colsum_block(part, gridDim.x, kMaxB, b, s);
        if (t == 0) *counter = 0;
    }
}

// k_colsum for b % 4 == 0 and 16-byte aligned X: a thread owns a column quad (float4 loads)
// and keeps eight rows in flight in four fixed-order partial sums (round 2: the scalar form ran
// at ~2.3 TB/s on config 4's 115 MB block).
// STAT: also the per-column max |x| (atomicMax on the float bits) and sum of squares (atomicAdd)
// into stat[0, 64) / the 64 doubles after them (zeroed by the caller), for the check and the
// scales of the standalone apply's tensor-core A2 (as k_ycheck's for Y1).
template <bool STAT>
__global__ void __launch_bounds__(256) k_colsum4(int64_t n, int b, const float* __restrict__ X, double* __restrict__ part,
                                                 double* __restrict__ s, unsigned int* __restrict__ counter,
                                                 unsigned int* __restrict__ stat) {
    __shared__ double red[256][4];
    float mx[4] = {0.f, 0.f, 0.f, 0.f};
    double sq[4] = {0.0, 0.0, 0.0, 0.0};
    const int nq = b / 4, rps = blockDim.x / nq;
    const int t = threadIdx.x, cq = t % nq, r0 = t / nq;
    const int64_t rows_per_blk = (n + gridDim.x - 1) / gridDim.x;
    const int64_t beg = blockIdx.x * rows_per_blk, end = min(n, beg + rows_per_blk);
    double a[4][4] = {};
    const float4* X4 = reinterpret_cast<const float4*>(X);
    if (r0 < rps) {
        int64_t i = beg + r0;
        for (; i + 7 * rps < end; i += 8 * rps) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcs(X4 + (i + u * rps) * nq + cq);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                a[u & 3][0] += (double)v[u].x;
                a[u & 3][1] += (double)v[u].y;
                a[u & 3][2] += (double)v[u].z;
                a[u & 3][3] += (double)v[u].w;
            }
            if constexpr (STAT) {
                float q[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    mx[0] = fmaxf(mx[0], fabsf(v[u].x)); q[0] = fmaf(v[u].x, v[u].x, q[0]);
                    mx[1] = fmaxf(mx[1], fabsf(v[u].y)); q[1] = fmaf(v[u].y, v[u].y, q[1]);
                    mx[2] = fmaxf(mx[2], fabsf(v[u].z)); q[2] = fmaf(v[u].z, v[u].z, q[2]);
                    mx[3] = fmaxf(mx[3], fabsf(v[u].w)); q[3] = fmaf(v[u].w, v[u].w, q[3]);
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) sq[k] += (double)q[k];
            }
        }
        for (; i < end; i += rps) {
            const float4 v = __ldcs(X4 + i * nq + cq);
            a[0][0] += (double)v.x;
            a[0][1] += (double)v.y;
            a[0][2] += (double)v.z;
            a[0][3] += (double)v.w;
            if constexpr (STAT) {
                mx[0] = fmaxf(mx[0], fabsf(v.x)); sq[0] += (double)v.x * v.x;
                mx[1] = fmaxf(mx[1], fabsf(v.y)); sq[1] += (double)v.y * v.y;
                mx[2] = fmaxf(mx[2], fabsf(v.z)); sq[2] += (double)v.z * v.z;
                mx[3] = fmaxf(mx[3], fabsf(v.w)); sq[3] += (double)v.w * v.w;
            }
        }
    }
    if constexpr (STAT) {   // block-level first: one atomic pair per column per block
        __shared__ float smx[256][4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            smx[t][k] = (r0 < rps) ? mx[k] : 0.f;
            red[t][k] = (r0 < rps) ? sq[k] : 0.0;
        }
        __syncthreads();
        if (t < b) {
            float m = 0.f;
            double v = 0.0;
            for (int q = 0; q < rps; ++q) {
                m = fmaxf(m, smx[q * nq + t / 4][t % 4]);
                v += red[q * nq + t / 4][t % 4];
            }
            atomicMax(stat + t, __float_as_uint(m));
            atomicAdd(reinterpret_cast<double*>(stat + 64) + t, v);
        }
        __syncthreads();
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) red[t][k] = (r0 < rps) ? (a[0][k] + a[1][k]) + (a[2][k] + a[3][k]) : 0.0;
    __syncthreads();
    if (t < b) {
        double v = 0.0;
        for (int q = 0; q < rps; ++q) v += red[q * nq + t / 4][t % 4];
        part[blockIdx.x * kMaxB + t] = v;
    }
    if (last_block_done(counter)) {
        ordered_colsum_block(part, gridDim.x, kMaxB, b, s);
        if (t == 0) *counter = 0;
    }
}

// ------------------------------------------------------------------ A2: Y1 = S^T X - w s^T
// Transposed SpMM through the device CSC copy: one warp per column (processed in the
// spatial `order`), LPR lanes per gathered X row (float4 each), G = 32/LPR rows in
// flight; the G partial sums are combined with shuffles (fixed order). Y1 is l x bp
// (bp = padded width; columns >= b are written as 0).
template <int LPR>
__global__ void __launch_bounds__(256) k_spmm_csc_vec4(
    int64_t l, int b, int bp, const int32_t* __restrict__ col_ptr, const int32_t* __restrict__ row_idx,
    const float* __restrict__ cval, const int32_t* __restrict__ order, const float* __restrict__ X,
    const double* __restrict__ w, const double* __restrict__ s, float* __restrict__ Y1) {
    constexpr int G = 32 / LPR;
    const int lane = threadIdx.x & 31;
    const int g = lane / LPR, q = lane % LPR;
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (wid >= l) return;
    const int64_t j = order ? order[wid] : wid;
    const int32_t beg = col_ptr[j], end = col_ptr[j + 1];
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    // software-pipelined: the next 32 (row, value) pairs load while this chunk's gathers run
    int32_t r_n = beg + lane < end ? row_idx[beg + lane] : 0;
    float v_n = beg + lane < end ? cval[beg + lane] : 0.f;
    for (int32_t base = beg; base < end; base += 32) {
        const int32_t r_l = r_n;
        const float v_l = v_n;
        const int32_t en = base + 32 + lane;
        r_n = en < end ? row_idx[en] : 0;
        v_n = en < end ? cval[en] : 0.f;
        const int cnt = min(32, end - base);
#pragma unroll
        for (int tq = g; tq < 32; tq += G) {
            const int32_t r = __shfl_sync(0xffffffffu, r_l, tq);
            const float v = __shfl_sync(0xffffffffu, v_l, tq);
            if (tq < cnt) {
                const float4 x = __ldg(reinterpret_cast<const float4*>(X + (int64_t)r * b) + q);
                acc.x = fmaf(v, x.x, acc.x);
                acc.y = fmaf(v, x.y, acc.y);
                acc.z = fmaf(v, x.z, acc.z);
                acc.w = fmaf(v, x.w, acc.w);
            }
        }
    }
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
        acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
        acc.w += __shfl_xor_sync(0xffffffffu, acc.w, o);
    }
    if (g == 0) {
        const double wj = w[j];
        const int c = 4 * q;
        float4 out;
        out.x = (float)((double)acc.x - wj * s[c + 0]);
        out.y = (float)((double)acc.y - wj * s[c + 1]);
        out.z = (float)((double)acc.z - wj * s[c + 2]);
        out.w = (float)((double)acc.w - wj * s[c + 3]);
        reinterpret_cast<float4*>(Y1 + j * bp)[q] = out;
    }
}

// Generic width: LPR = nextpow2(b) (<= 32) lanes per row, NC columns per lane.
template <int LPR, int NC>
__global__ void __launch_bounds__(256) k_spmm_csc_gen(
    int64_t l, int b, int bp, const int32_t* __restrict__ col_ptr, const int32_t* __restrict__ row_idx,
    const float* __restrict__ cval, const int32_t* __restrict__ order, const float* __restrict__ X,
    const double* __restrict__ w, const double* __restrict__ s, float* __restrict__ Y1) {
    constexpr int G = 32 / LPR;
    const int lane = threadIdx.x & 31;
    const int g = lane / LPR, q = lane % LPR;
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (wid >= l) return;
    const int64_t j = order ? order[wid] : wid;
    const int32_t beg = col_ptr[j], end = col_ptr[j + 1];
    float acc[NC];
#pragma unroll
    for (int u = 0; u < NC; ++u) acc[u] = 0.f;
    int32_t r_n = beg + lane < end ? row_idx[beg + lane] : 0;   // software-pipelined (as vec4)
    float v_n = beg + lane < end ? cval[beg + lane] : 0.f;
    for (int32_t base = beg; base < end; base += 32) {
        const int32_t r_l = r_n;
        const float v_l = v_n;
        const int32_t en = base + 32 + lane;
        r_n = en < end ? row_idx[en] : 0;
        v_n = en < end ? cval[en] : 0.f;
        const int cnt = min(32, end - base);
#pragma unroll 4
        for (int tq = g; tq < 32; tq += G) {
            const int32_t r = __shfl_sync(0xffffffffu, r_l, tq);
            const float v = __shfl_sync(0xffffffffu, v_l, tq);
            if (tq < cnt) {
#pragma unroll
                for (int u = 0; u < NC; ++u) {
                    const int c = q + u * LPR;
                    if (c < b) acc[u] = fmaf(v, __ldg(X + (int64_t)r * b + c), acc[u]);
                }
            }
        }
    }
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
        for (int u = 0; u < NC; ++u) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
    if (g == 0) {
        const double wj = w[j];
#pragma unroll
        for (int u = 0; u < NC; ++u) {
            const int c = q + u * LPR;
            if (c < b) Y1[j * bp + c] = (float)((double)acc[u] - wj * s[c]);
            else if (c < bp) Y1[j * bp + c] = 0.f;
        }
    }
}

// ------------------------------------------------------------------ A5: Y = -1/2 (S Y2 - 1 t^T)
// CSR SpMM: LPR lanes per row (float4 gathers of the L1/L2-resident Y2 rows), G rows per warp.
// The G rows of a warp are consecutive, so their (column, value) pairs are contiguous: each lane
// loads one pair per chunk of LPR (four chunks in flight), and the group broadcasts them in entry
// order with shuffles. One lane per pair instead of every lane of a group re-reading its row's
// pair cuts the L1 wavefronts per step from ~16 (4 + 4 for the strided column and value words,
// 8 for the gathered rows) to ~10; the sums keep the entry order (beg, beg + 1, ...), so results
// are bitwise those of the plain loop. The trip count is warp-uniform (full-warp shuffles).
// SHF = false: the plain loop (every lane of a group reads its row's pairs itself; measured faster for
// wide rows, LPR >= 8, where a warp holds few rows and the pair loads are few lines anyway).
template <int LPR, bool SHF>
__global__ void __launch_bounds__(256) k_spmm_csr_vec4(
    int64_t n, int b, int bp, const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
    const float* __restrict__ val, const float* __restrict__ Y2, const double* __restrict__ t,
    float* __restrict__ Y) {
    constexpr int G = 32 / LPR;
    constexpr int U = 4;   // chunks of LPR entries loaded ahead
    const int lane = threadIdx.x & 31;
    const int g = lane / LPR, q = lane % LPR;
    const int64_t i = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * G + g;
    const bool live = i < n;
    const int32_t beg = live ? rp[i] : 0, end = live ? rp[i + 1] : 0;
    const int len = end - beg;
    const float4* __restrict__ Y24 = reinterpret_cast<const float4*>(Y2);
    const int nv = bp / 4;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if constexpr (!SHF) {
#pragma unroll 4
        for (int32_t e = beg; e < end; ++e) {
            const int32_t c = __ldg(col + e);
            const float v = __ldg(val + e);
            const float4 y = __ldg(Y24 + (int64_t)c * nv + q);
            acc.x = fmaf(v, y.x, acc.x);
            acc.y = fmaf(v, y.y, acc.y);
            acc.z = fmaf(v, y.z, acc.z);
            acc.w = fmaf(v, y.w, acc.w);
        }
    }
    const int maxlen = SHF ? (int)__reduce_max_sync(0xffffffffu, (unsigned)len) : 0;
    for (int c0 = 0; c0 < maxlen; c0 += U * LPR) {
        int lc[U];
        float lv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t e = beg + c0 + u * LPR + q;
            const bool ok = e < end;
            lc[u] = ok ? __ldg(col + e) : 0;
            lv[u] = ok ? __ldg(val + e) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (c0 + u * LPR >= maxlen) break;   // (warp-uniform)
#pragma unroll
            for (int tq = 0; tq < LPR; ++tq) {
                const int c = __shfl_sync(0xffffffffu, lc[u], tq, LPR);
                const float v = __shfl_sync(0xffffffffu, lv[u], tq, LPR);
                if (c0 + u * LPR + tq < len) {
                    const float4 y = __ldg(Y24 + (int64_t)c * nv + q);
                    acc.x = fmaf(v, y.x, acc.x);
                    acc.y = fmaf(v, y.y, acc.y);
                    acc.z = fmaf(v, y.z, acc.z);
                    acc.w = fmaf(v, y.w, acc.w);
                }
            }
        }
    }
    if (!live) return;
    const int c0 = 4 * q;
    float4 out;
    out.x = (float)(-0.5 * ((double)acc.x - t[c0 + 0]));
    out.y = (float)(-0.5 * ((double)acc.y - t[c0 + 1]));
    out.z = (float)(-0.5 * ((double)acc.z - t[c0 + 2]));
    out.w = (float)(-0.5 * ((double)acc.w - t[c0 + 3]));
    reinterpret_cast<float4*>(Y + i * b)[q] = out;
}

template <int LPR, int NC>
__global__ void __launch_bounds__(256) k_spmm_csr_gen(
    int64_t n, int b, int bp, const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
    const float* __restrict__ val, const float* __restrict__ Y2, const double* __restrict__ t,
    float* __restrict__ Y) {
    constexpr int G = 32 / LPR;
    const int lane = threadIdx.x & 31;
    const int g = lane / LPR, q = lane % LPR;
    const int64_t i = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * G + g;
    if (i >= n) return;
    const int32_t beg = rp[i], end = rp[i + 1];
    float acc[NC];
#pragma unroll
    for (int u = 0; u < NC; ++u) acc[u] = 0.f;
#pragma unroll 4
    for (int32_t e = beg; e < end; ++e) {
        const int32_t c = __ldg(col + e);
        const float v = __ldg(val + e);
#pragma unroll
        for (int u = 0; u < NC; ++u) {
            const int cc = q + u * LPR;
            if (cc < b) acc[u] = fmaf(v, __ldg(Y2 + (int64_t)c * bp + cc), acc[u]);
        }
    }
#pragma unroll
    for (int u = 0; u < NC; ++u) {
        const int cc = q + u * LPR;
        if (cc < b) Y[i * b + cc] = (float)(-0.5 * ((double)acc[u] - t[cc]));
    }
}

// Narrow blocks (bp <= 4): L lanes per row stride over the row's nonzeros, so the col / val
// reads of a warp are contiguous (one lane per row would read 32 rows' entries with a
// stride of the row length), then a fixed shuffle tree adds the L partial sums (bitwise
// reproducible). L ~ the mean row length (4 .. 32), BW = bp values per gathered Y2 row.
template <int L, int BW>
__global__ void __launch_bounds__(256) k_spmm_csr_sub(
    int64_t n, int b, int bp, const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
    const float* __restrict__ val, const float* __restrict__ Y2, const double* __restrict__ t,
    float* __restrict__ Y) {
    constexpr int G = 32 / L;
    const int lane = threadIdx.x & 31;
    const int g = lane / L, q = lane % L;
    const int64_t i = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * G + g;
    const bool live = i < n;
    float acc[BW];
#pragma unroll
    for (int u = 0; u < BW; ++u) acc[u] = 0.f;
    if (live) {
        const int32_t beg = rp[i], end = rp[i + 1];
#pragma unroll 2
        for (int32_t e = beg + q; e < end; e += L) {
            const int32_t c = __ldg(col + e);
            const float v = __ldg(val + e);
            if constexpr (BW == 4) {
                const float4 y = __ldg(reinterpret_cast<const float4*>(Y2 + (int64_t)c * 4));
                acc[0] = fmaf(v, y.x, acc[0]);
                acc[1] = fmaf(v, y.y, acc[1]);
                acc[2] = fmaf(v, y.z, acc[2]);
                acc[3] = fmaf(v, y.w, acc[3]);
            } else if constexpr (BW == 2) {
                const float2 y = __ldg(reinterpret_cast<const float2*>(Y2 + (int64_t)c * 2));
                acc[0] = fmaf(v, y.x, acc[0]);
                acc[1] = fmaf(v, y.y, acc[1]);
            } else {
                acc[0] = fmaf(v, __ldg(Y2 + c), acc[0]);
            }
        }
    }
#pragma unroll
    for (int off = L / 2; off > 0; off >>= 1)
#pragma unroll
        for (int u = 0; u < BW; ++u) acc[u] += __shfl_down_sync(0xffffffffu, acc[u], off, L);
    if (live && q == 0) {
#pragma unroll
        for (int u = 0; u < BW; ++u)
            if (u < b) Y[i * b + u] = (float)(-0.5 * ((double)acc[u] - t[u]));
    }
}

// ------------------------------------------------------------------ row order (create)
// S's rows are reordered at create when that makes 128-row blocks touch fewer landmarks
// (sbmds.cu reorder_rows; DESIGN.md §4 "Row order"). Key of a row: its two smallest column
// indices (c0 << 32 | c1): rows sharing their lowest landmarks are adjacent, and since FPS
// landmark indices are coarse-to-fine, the order is a hierarchy of landmark neighbourhoods.
__global__ void k_row_keys(int64_t n, int64_t l, const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                           uint64_t* __restrict__ keys, int32_t* __restrict__ iota) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t c0 = (uint32_t)l, c1 = (uint32_t)l;   // (an empty row sorts last)
        for (int32_t e = rp[i]; e < rp[i + 1]; ++e) {
            const uint32_t c = (uint32_t)col[e];
            if (c < c0) { c1 = c0; c0 = c; }
            else if (c < c1 && c != c0) c1 = c;
        }
        if (c1 == (uint32_t)l) c1 = c0;
        keys[i] = ((uint64_t)c0 << 32) | c1;
        iota[i] = (int32_t)i;
    }
}

// Distinct columns of sampled 128-row blocks (block s * stride) in the natural (perm = null) or
// a permuted order: a bitmap of l bits in shared memory per block.
__global__ void __launch_bounds__(256) k_block_distinct(int64_t n, int64_t l, int64_t stride, const int32_t* __restrict__ perm,
                                                        const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                        int32_t* __restrict__ counts) {
    extern __shared__ unsigned int bits[];
    const int64_t words = (l + 31) / 32;
    for (int64_t w = threadIdx.x; w < words; w += blockDim.x) bits[w] = 0u;
    __syncthreads();
    const int64_t r0 = blockIdx.x * stride * 128;
    for (int rr = threadIdx.x / 8; rr < 128; rr += blockDim.x / 8) {
        const int64_t r = r0 + rr;
        if (r >= n) break;
        const int64_t i = perm ? perm[r] : r;
        for (int32_t e = rp[i] + (threadIdx.x & 7); e < rp[i + 1]; e += 8) {
            const uint32_t c = (uint32_t)col[e];
            atomicOr(&bits[c >> 5], 1u << (c & 31));
        }
    }
    __syncthreads();
    int cnt = 0;
    for (int64_t w = threadIdx.x; w < words; w += blockDim.x) cnt += __popc(bits[w]);
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    __shared__ int red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int q = 0; q < 8; ++q) t += red[q];
        counts[blockIdx.x] = t;
    }
}

__global__ void k_perm_lengths(int64_t n, const int32_t* __restrict__ perm, const int32_t* __restrict__ rp,
                               int32_t* __restrict__ len) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        len[r] = rp[perm[r] + 1] - rp[perm[r]];
}

// new row r = old row perm[r] (one warp per row)
__global__ void __launch_bounds__(256) k_perm_rows(int64_t n, const int32_t* __restrict__ perm,
                                                   const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                   const float* __restrict__ val, const int32_t* __restrict__ nrp,
                                                   int32_t* __restrict__ ncol, float* __restrict__ nval) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < n;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int32_t i = perm[r], b0 = rp[i], len = rp[i + 1] - b0, d0 = nrp[r];
        for (int e = lane; e < len; e += 32) {
            ncol[d0 + e] = col[b0 + e];
            nval[d0 + e] = val[b0 + e];
        }
    }
}

// n x b blocks between the caller's row order and the handle's: out[r] = in[perm[r]] (gather)
// or out[perm[r]] = in[r] (scatter); one thread per element, rows of b contiguous floats.
template <bool SCATTER>
__global__ void k_permute_rows(int64_t n, int b, const int32_t* __restrict__ perm, const float* __restrict__ in,
                               float* __restrict__ out) {
    const int64_t total = n * b;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / b, c = e - r * b;
        const int64_t i = perm[r];
        if (SCATTER) out[i * b + c] = in[e];
        else out[e] = in[i * b + c];
    }
}

}  // namespace sbmds
