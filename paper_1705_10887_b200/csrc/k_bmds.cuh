// BMDS on the GPU (SURVEY.md §8(f) NEXT-3b): the paper's QR route for classical scaling on
// the BHA approximation, PAPER.md:217-218 (§3.3 "Classical Scaling with BHA"):
//   Q R = J P  (R in R^{l x l}),   -1/2 R W R^T = V~ Λ V~^T,   Z = Q V~_m Λ_m^{1/2}.
// Here Q is never stored: R comes from the Cholesky factor of the Gram (J P)^T (J P) (the
// "Cholesky-QR" form of QR = JP, the same R up to column signs), and Z = J P (R^{-1} V~_m)
// Λ_m^{1/2} is formed by the library's CSR SpMM with the rank-one centring. fp64 throughout
// the l x l algebra; the n x l matrix J P is formed densely (the O(nl) memory the paper notes
// for BMDS) only to take its Gram.
//   k_jp_dense     JP[i][a] = S_ia - w_a (row i of S scattered into -w)
//   k_dgemm        C = alpha op(A) op(B) + beta C, fp64, 64 x 64 tiles, fixed K order
//   k_potf2        Cholesky of one diagonal block (upper, in place), breakdown flag
//   k_trsm_rows    R[k0:k1, j] = R_kk^{-T} A[k0:k1, j] for the columns right of the block
//   k_zero_lower   zero the strict lower triangle (R as a plain matrix for the GEMMs)
//   k_backsolve    U = R^{-1} V (R upper), one warp per column
//   k_f2d_sym / k_dinit / k_bmds_to_y2   W in fp64, Gaussian start, U -> the SpMM's Y2 and t
//   k_symv_rows / k_vdot                  the sharded apply's t_g = (D w_g)^T Y1 (sbmds.cu)
#pragma once
#include "common.cuh"

namespace sbmds {

__global__ void __launch_bounds__(256) k_jp_dense(int64_t n, int64_t l, const int32_t* __restrict__ rp,
                                                  const int32_t* __restrict__ col, const float* __restrict__ val,
                                                  const double* __restrict__ w, double* __restrict__ JP) {
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        double* row = JP + i * l;
        for (int64_t a = threadIdx.x; a < l; a += blockDim.x) row[a] = -w[a];
        __syncthreads();
        if (threadIdx.x == 0)   // entries in stored order (duplicates summed in that order)
            for (int32_t e = rp[i]; e < rp[i + 1]; ++e) row[col[e]] += (double)val[e];
        __syncthreads();
    }
}

// C[M x N] (ldc) = alpha * op(A) op(B) + beta * C. op(A) is M x K: A[m lda + k] (TA = false) or
// A[k lda + m] (TA = true); op(B) is K x N: B[k ldb + n] (TB = false) or B[n ldb + k] (TB = true).
// beta == 0 does not read C. Each output's K sum runs in increasing k (deterministic).
template <bool TA, bool TB>
__global__ void __launch_bounds__(256) k_dgemm(int M, int N, int64_t K, double alpha, const double* __restrict__ A,
                                               int64_t lda, const double* __restrict__ B, int64_t ldb, double beta,
                                               double* __restrict__ C, int64_t ldc) {
    __shared__ double As[16][64 + 1];
    __shared__ double Bs[16][64 + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int64_t k0 = 0; k0 < K; k0 += 16) {
        for (int e = threadIdx.x; e < 1024; e += 256) {
            int mm, kk;
            if (TA) { mm = e & 63; kk = e >> 6; } else { kk = e & 15; mm = e >> 4; }
            const int64_t gm = m0 + mm, gk = k0 + kk;
            As[kk][mm] = (gm < M && gk < K) ? (TA ? A[gk * lda + gm] : A[gm * lda + gk]) : 0.0;
            int nn, kb;
            if (TB) { kb = e & 15; nn = e >> 4; } else { nn = e & 63; kb = e >> 6; }
            const int64_t gn = n0 + nn, gkb = k0 + kb;
            Bs[kb][nn] = (gn < N && gkb < K) ? (TB ? B[gn * ldb + gkb] : B[gkb * ldb + gn]) : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t gm = m0 + ty * 4 + i, gn = n0 + tx * 4 + j;
            if (gm < M && gn < N) {
                double* c = C + gm * ldc + gn;
                *c = beta == 0.0 ? alpha * acc[i][j] : fma(alpha, acc[i][j], beta * *c);
            }
        }
}

// max_i A_ii (one block): the scale of the semi-definite Cholesky's zero-pivot test
__global__ void __launch_bounds__(256) k_maxdiag(const double* __restrict__ A, int64_t lda, int64_t l,
                                                 double* __restrict__ out) {
    __shared__ double red[256];
    double m = 0.0;
    for (int64_t i = threadIdx.x; i < l; i += blockDim.x) m = fmax(m, A[i * lda + i]);
    red[threadIdx.x] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < 256; ++q) m = fmax(m, red[q]);
        *out = m;
    }
}

// The same product for large shapes (round 2): 128 x 128 tiles, 8 x 8 outputs per thread, the
// next K slice of A and B loaded into registers while the current one is multiplied out of
// shared memory. gridDim.z > 1 splits K into gridDim.z contiguous ranges: slice z writes its
// partial (alpha = 1, beta = 0) to W + z * M * N (row-major, ld N) and k_sum_splits adds the
// slices in z order into C (deterministic). At BMDS's Gram (1000 x 1000, K = 100,000) the 64 x 64
// kernel above ran at ~4.5 TFLOP/s.
template <bool TA, bool TB>
__global__ void __launch_bounds__(256, 1) k_dgemm128(int M, int N, int64_t K, double alpha, const double* __restrict__ A,
                                                     int64_t lda, const double* __restrict__ B, int64_t ldb, double beta,
                                                     double* __restrict__ C, int64_t ldc, double* __restrict__ Wsplit) {
    constexpr int BK = 8;
    __shared__ double As[2][BK][128 + 2];
    __shared__ double Bs[2][BK][128 + 2];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int m0 = blockIdx.y * 128, n0 = blockIdx.x * 128;
    const int64_t kchunk = (K + gridDim.z - 1) / gridDim.z;
    const int64_t kb = blockIdx.z * kchunk, ke = min(K, kb + kchunk);
    double acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
    // each thread loads 4 elements of A's and 4 of B's 128 x 8 slice
    double ra[4], rb[4];
    auto load = [&](int64_t k0) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = threadIdx.x + 256 * u;   // 0..1023
            int mm, kk;
            if (TA) { mm = e & 127; kk = e >> 7; } else { kk = e & 7; mm = e >> 3; }
            const int64_t gm = m0 + mm, gk = k0 + kk;
            ra[u] = (gm < M && gk < ke) ? (TA ? A[gk * lda + gm] : A[gm * lda + gk]) : 0.0;
            int nn, kb2;
            if (TB) { kb2 = e & 7; nn = e >> 3; } else { nn = e & 127; kb2 = e >> 7; }
            const int64_t gn = n0 + nn, gkb = k0 + kb2;
            rb[u] = (gn < N && gkb < ke) ? (TB ? B[gn * ldb + gkb] : B[gkb * ldb + gn]) : 0.0;
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = threadIdx.x + 256 * u;
            int mm, kk;
            if (TA) { mm = e & 127; kk = e >> 7; } else { kk = e & 7; mm = e >> 3; }
            As[buf][kk][mm] = ra[u];
            int nn, kb2;
            if (TB) { kb2 = e & 7; nn = e >> 3; } else { nn = e & 127; kb2 = e >> 7; }
            Bs[buf][kb2][nn] = rb[u];
        }
    };
    if (kb < ke) {
        load(kb);
        store(0);
    }
    __syncthreads();
    int buf = 0;
    for (int64_t k0 = kb; k0 < ke; k0 += BK) {
        const bool more = k0 + BK < ke;
        if (more) load(k0 + BK);
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            double a[8], b[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) {   // rows ty*4 .. +3 and 64 + ty*4 .. +3 (conflict-free halves)
                a[i] = As[buf][kk][ty * 4 + i];
                a[4 + i] = As[buf][kk][64 + ty * 4 + i];
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                b[j] = Bs[buf][kk][tx * 4 + j];
                b[4 + j] = Bs[buf][kk][64 + tx * 4 + j];
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        if (more) store(buf ^ 1);
        __syncthreads();
        buf ^= 1;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int64_t gm = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
            const int64_t gn = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
            if (gm < M && gn < N) {
                if (gridDim.z > 1) {
                    Wsplit[(int64_t)blockIdx.z * M * N + gm * N + gn] = acc[i][j];
                } else {
                    double* c = C + gm * ldc + gn;
                    *c = beta == 0.0 ? alpha * acc[i][j] : fma(alpha, acc[i][j], beta * *c);
                }
            }
        }
}

__global__ void k_sum_splits(int M, int N, int splits, double alpha, const double* __restrict__ Wsplit, double beta,
                             double* __restrict__ C, int64_t ldc) {
    const int64_t total = (int64_t)M * N;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        double v = 0.0;
        for (int z = 0; z < splits; ++z) v += Wsplit[(int64_t)z * total + e];
        double* c = C + (e / N) * ldc + e % N;
        *c = beta == 0.0 ? alpha * v : fma(alpha, v, beta * *c);
    }
}

// Upper Cholesky of the nb x nb diagonal block at (k0, k0) of A (lda), in place: A_kk = R^T R,
// semi-definite: J P is rank-deficient whenever some combination of S's columns is constant
// (for a partition of unity J P 1 = J 1 = 0), so a pivot <= 1e-13 max diag is a null direction
// (counted in *dropped): its row of R is zero (the exact-arithmetic value for a PSD matrix).
// status = 2 on a negative (< -1e-10 max diag) or non-finite pivot (G not PSD).
// (allow_drop = 0, the sBHA solve of the SPD M_uu: a non-positive pivot is a breakdown.)
__global__ void __launch_bounds__(256) k_potf2(double* __restrict__ A, int64_t lda, int k0, int nb,
                                               int* __restrict__ status, const double* __restrict__ dmax,
                                               int* __restrict__ dropped, int allow_drop) {
    __shared__ double T[64][65];
    __shared__ int fail;
    const int tid = threadIdx.x;
    for (int e = tid; e < nb * nb; e += blockDim.x) T[e / nb][e % nb] = A[(int64_t)(k0 + e / nb) * lda + k0 + e % nb];
    if (tid == 0) fail = 0;
    __syncthreads();
    const double tol0 = 1e-13 * *dmax;
    for (int k = 0; k < nb; ++k) {
        const double d = T[k][k];
        if (!isfinite(d) || d < -1e-10 * *dmax || (!allow_drop && !(d > 0.0))) {
            if (tid == 0) fail = 1;
            break;
        }
        if (allow_drop && d <= tol0) {   // null direction: R row k = 0, nothing to eliminate
            __syncthreads();
            for (int j = k + tid; j < nb; j += blockDim.x) T[k][j] = 0.0;
            if (tid == 0) atomicAdd(dropped, 1);
            __syncthreads();
            continue;
        }
        const double r = sqrt(d), ri = 1.0 / r;
        __syncthreads();
        for (int j = k + 1 + tid; j < nb; j += blockDim.x) T[k][j] *= ri;
        if (tid == 0) T[k][k] = r;
        __syncthreads();
        const int m = nb - k - 1;
        for (int e = tid; e < m * m; e += blockDim.x) {
            const int i = k + 1 + e / m, j = k + 1 + e % m;
            if (j >= i) T[i][j] = fma(-T[k][i], T[k][j], T[i][j]);
        }
        __syncthreads();
    }
    __syncthreads();
    if (fail) {
        if (tid == 0) *status = 2;
        return;
    }
    for (int e = tid; e < nb * nb; e += blockDim.x) {
        const int i = e / nb, j = e % nb;
        if (j >= i) A[(int64_t)(k0 + i) * lda + k0 + j] = T[i][j];
    }
}

// Rows k0..k0+nb of R right of the diagonal block: solve R_kk^T X = A[k0:k0+nb, j] (forward
// substitution, R_kk^T lower) for every column j in [k0 + nb, l); one thread per column.
__global__ void __launch_bounds__(256) k_trsm_rows(double* __restrict__ A, int64_t lda, int64_t l, int k0, int nb,
                                                   const int* __restrict__ status) {
    __shared__ double R[64][65];
    if (*status == 2) return;
    for (int e = threadIdx.x; e < nb * nb; e += blockDim.x)
        R[e / nb][e % nb] = A[(int64_t)(k0 + e / nb) * lda + k0 + e % nb];
    __syncthreads();
    const int64_t j = (int64_t)k0 + nb + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= l) return;
    double x[64];
#pragma unroll 1
    for (int i = 0; i < nb; ++i) {
        double acc = A[(int64_t)(k0 + i) * lda + j];
        for (int p = 0; p < i; ++p) acc = fma(-R[p][i], x[p], acc);
        x[i] = R[i][i] != 0.0 ? acc / R[i][i] : 0.0;   // (a dropped pivot's row of R stays 0)
        A[(int64_t)(k0 + i) * lda + j] = x[i];
    }
}

__global__ void k_zero_lower(double* __restrict__ A, int64_t lda, int64_t l) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < l * l; e += (int64_t)gridDim.x * blockDim.x)
        if (e / l > e % l) A[(e / l) * lda + e % l] = 0.0;
}

// U = R^{-1} V: R (l x l, upper, ldr), V and U l x m row-major (ldv), one warp per column, rows
// from the bottom; the sum over j > i in lane-strided order then a fixed shuffle tree.
__global__ void __launch_bounds__(256) k_backsolve(int64_t l, int m, const double* __restrict__ R, int64_t ldr,
                                                   const double* __restrict__ V, int64_t ldv, double* __restrict__ U) {
    const int lane = threadIdx.x & 31;
    const int c = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (c >= m) return;
    for (int64_t i = l - 1; i >= 0; --i) {
        double acc = 0.0;
        for (int64_t j = i + 1 + lane; j < l; j += 32) acc = fma(R[i * ldr + j], U[j * ldv + c], acc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        const double rii = R[i * ldr + i];   // (a dropped pivot: its equation is vacuous, U_i = 0)
        if (lane == 0) U[i * ldv + c] = rii != 0.0 ? (V[i * ldv + c] - acc) / rii : 0.0;
        __syncwarp();
    }
}

// D (fp32, ldD) -> W (fp64 l x l), mirroring the block upper triangle when only it is present
__global__ void k_f2d_sym(int64_t l, const float* __restrict__ D, int64_t ldD, double* __restrict__ W) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < l * l; e += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = e / l, j = e % l;
        if ((j >> 7) < (i >> 7)) { const int64_t t = i; i = j; j = t; }   // read the block upper triangle
        W[e] = (double)D[i * ldD + j];
    }
}

// X (l x b fp64) ~ N(0, 1): Box-Muller on a counter-based hash of (seed, index)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__global__ void k_dinit(int64_t count, uint64_t seed, double* __restrict__ X) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t h1 = mix64(seed * 0x9e3779b97f4a7c15ull + 2 * (uint64_t)e + 1);
        const uint64_t h2 = mix64(h1 + 0x632be59bd9b4e019ull);
        const double u1 = ((h1 >> 11) + 0.5) * 0x1.0p-53, u2 = (h2 >> 11) * 0x1.0p-53;
        X[e] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
    }
}

// Y2 (l x bp fp32, pitch bp) = -2 U (l x m fp64) and t = -2 w^T U, so that the CSR SpMM's
// -1/2 (S Y2 - 1 t^T) is J P U = S U - 1 (w^T U). One block; t in fixed row order.
__global__ void __launch_bounds__(256) k_bmds_to_y2(int64_t l, int m, int bp, const double* __restrict__ U,
                                                    const double* __restrict__ w, float* __restrict__ Y2,
                                                    double* __restrict__ t) {
    __shared__ double part[256];
    for (int64_t e = threadIdx.x; e < l * bp; e += blockDim.x) {
        const int c = (int)(e % bp);
        Y2[e] = c < m ? (float)(-2.0 * U[(e / bp) * m + c]) : 0.f;
    }
    const int c = threadIdx.x % 64, r0 = threadIdx.x / 64;
    double acc = 0.0;
    if (c < m)
        for (int64_t i = r0; i < l; i += 4) acc = fma(w[i], U[i * m + c], acc);
    part[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x < m) t[threadIdx.x] = -2.0 * (part[c] + part[64 + c] + part[128 + c] + part[192 + c]);
}

// Sharded apply (sbmds.cu shard_stage_dev): v_g = D w_g (D full, ldD; one warp per row, fixed
// lane-strided order) and t_g = v_g^T Y1 (Y1 l x bp, columns < b; one block, fixed order):
// t = w^T Y2 = w^T D Y1 = sum_g (D w_g)^T Y1 needs no second exchange.
__global__ void __launch_bounds__(256) k_symv_rows(int64_t l, const float* __restrict__ D, int64_t ldD,
                                                   const double* __restrict__ w, double* __restrict__ v) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = blockIdx.x * 8 + (threadIdx.x >> 5); i < l; i += (int64_t)gridDim.x * 8) {
        double acc = 0.0;
        for (int64_t j = lane; j < l; j += 32) acc = fma((double)D[i * ldD + j], w[j], acc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) v[i] = acc;
    }
}

// t = v^T Y1 (b values, fp64). Block B takes the contiguous row range B of gridDim.x and writes
// its partial to part[B][64]; k_vdot_sum adds the partials in block order (fixed order, bitwise
// reproducible for a given grid). A single CTA over all l rows took 3 ms at l = 50,000 (12,500
// dependent fp64 FMAs per thread): two thirds of a sharded eigs iteration.
constexpr int kVdotBlocks = 128;
__global__ void __launch_bounds__(256) k_vdot(int64_t l, int b, int bp, const double* __restrict__ v,
                                              const float* __restrict__ Y1, double* __restrict__ part) {
    __shared__ double red[256];
    const int c = threadIdx.x % 64, r0 = threadIdx.x / 64;
    const int64_t per = (l + gridDim.x - 1) / gridDim.x;
    const int64_t beg = blockIdx.x * per, end = min(l, beg + per);
    double acc = 0.0;
    if (c < b)
        for (int64_t i = beg + r0; i < end; i += 4) acc = fma(v[i], (double)Y1[i * bp + c], acc);
    red[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x < 64)
        part[blockIdx.x * 64 + threadIdx.x] = (red[c] + red[64 + c]) + (red[128 + c] + red[192 + c]);
}

__global__ void __launch_bounds__(64) k_vdot_sum(int nblocks, int b, const double* __restrict__ part,
                                                 double* __restrict__ t) {
    if ((int)threadIdx.x >= b) return;
    double acc = 0.0;
    for (int B = 0; B < nblocks; ++B) acc += part[B * 64 + threadIdx.x];
    t[threadIdx.x] = acc;
}

}  // namespace sbmds
