// Block Lanczos with full reorthogonalisation (the paper's sBMDS uses
// "the Lanczos method" on matrix-vector products; SPEC.md:49-53 asks for full
// reorthogonalisation). Small device pieces of the host-orchestrated iteration in
// sbmds.cu (eigs_lanczos): the n x b basis blocks Q_0..Q_{k-1} live block-major in one buffer.
//   k_combine      out = in0 + alpha * sum_{j < nq} Q_j M_j       (fp64 arithmetic per element)
//   k_tadd         T[i-block][j-block] += H  (b x b), and the transposed placement for R
//   k_chol_r       k_chol that also writes R (upper) for T's subdiagonal blocks
//   k_lanczos_prep T <- (T + T^T)/2, Gl = T T + E G_W E^T (so that k_rr's residual
//                  u^T Gl u - θ^2 = ||B_k E^T u||^2, the Lanczos residual), identity for R^-1
#pragma once
#include "common.cuh"
#include "k_small.cuh"

namespace sbmds {

constexpr int kLzMaxKB = kMaxB;   // the projected problem (k blocks of b) is solved by k_rr

// out[r][c] = (in0 ? in0[r][c] : 0) + alpha * sum_j sum_p Q_j[r][p] M[(j b + p) ldm + c], c < mo
template <int BT>
__global__ void __launch_bounds__(256) k_combine(int64_t n, int b, int nq, const float* __restrict__ Q, int mo, int ldm,
                                                 const double* __restrict__ M, const float* __restrict__ in0, double alpha,
                                                 float* __restrict__ out) {
    __shared__ double Ms[kLzMaxKB * kMaxB];
    for (int e = threadIdx.x; e < nq * b * mo; e += blockDim.x) Ms[e] = M[(e / mo) * ldm + (e % mo)];
    __syncthreads();
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        double acc[BT];
#pragma unroll
        for (int c = 0; c < BT; ++c) acc[c] = 0.0;
        for (int j = 0; j < nq; ++j) {
            const float* q = Q + ((int64_t)j * n + r) * b;
            for (int p = 0; p < b; ++p) {
                const double v = (double)q[p];
                const double* mr = Ms + (j * b + p) * mo;
#pragma unroll
                for (int c = 0; c < BT; ++c)
                    if (c < mo) acc[c] = fma(v, mr[c], acc[c]);
            }
        }
#pragma unroll
        for (int c = 0; c < BT; ++c)
            if (c < mo) out[r * mo + c] = (float)((in0 ? (double)in0[r * mo + c] : 0.0) + alpha * acc[c]);
    }
}

// T (kb x kb, row-major, ldt) block (bi, bj) += H (b x b, H[p b + q]); with `transposed` the
// block (bj, bi) receives H^T as well (for R: T[j+1][j] = R, T[j][j+1] = R^T)
__global__ void k_tadd(int b, int ldt, int bi, int bj, const double* __restrict__ H, double* __restrict__ T,
                       int also_transposed) {
    for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
        const int p = e / b, q = e % b;
        T[(bi * b + p) * ldt + bj * b + q] += H[e];
        if (also_transposed) T[(bj * b + q) * ldt + bi * b + p] += H[e];
    }
}

// k_chol plus R itself (upper triangle, zeros below) in Rout
__global__ void __launch_bounds__(256) k_chol_r(int b, const double* __restrict__ G, double* __restrict__ Rinv,
                                                int* __restrict__ status, double* __restrict__ Rout) {
    __shared__ double A[kMaxB][kMaxB + 1];
    __shared__ int fail;
    __shared__ double shift;
    chol_block(b, G, Rinv, status, A, &fail, &shift);
    __syncthreads();
    if (!fail)
        for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
            const int i = e / b, j = e % b;
            Rout[e] = j >= i ? A[i][j] : 0.0;
        }
}

// T <- (T + T^T) / 2; Gl = T T + E G_W E^T (E = the last b x b block); I = identity
__global__ void __launch_bounds__(256) k_lanczos_prep(int kb, int b, double* __restrict__ T, const double* __restrict__ GW,
                                                      double* __restrict__ Gl, double* __restrict__ I) {
    __shared__ double Ts[kLzMaxKB * kLzMaxKB];
    for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
        const int i = e / kb, j = e % kb;
        Ts[e] = 0.5 * (T[i * kb + j] + T[j * kb + i]);
    }
    __syncthreads();
    const int o = kb - b;
    for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
        const int i = e / kb, j = e % kb;
        double acc = 0.0;
        for (int p = 0; p < kb; ++p) acc = fma(Ts[i * kb + p], Ts[p * kb + j], acc);
        if (i >= o && j >= o) acc += GW[(i - o) * b + (j - o)];
        Gl[e] = acc;
        T[e] = Ts[e];
        I[e] = i == j ? 1.0 : 0.0;
    }
}

// Lanczos residuals without cancellation: B~ (Q u_i) - θ_i (Q u_i) = W_k R_k E^T u_i with W_k
// orthonormal, so r_i = ||R_k u_i[last block]|| (R_k from the Cholesky-QR of the final
// residual block); overwrites k_rr's residuals, max residual and convergence flag.
__global__ void k_lanczos_resid(int kb, int b, int m, double tol, const double* __restrict__ R, RrOut* __restrict__ rr) {
    __shared__ double res[kLzMaxKB];
    const int o = kb - b;
    for (int i = threadIdx.x; i < kb; i += blockDim.x) {
        double s2 = 0.0;
        for (int p = 0; p < b; ++p) {
            double acc = 0.0;
            for (int q = p; q < b; ++q) acc = fma(R[p * b + q], rr->U[(o + q) * kb + i], acc);
            s2 = fma(acc, acc, s2);
        }
        res[i] = sqrt(s2);
        rr->resid[i] = res[i];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double tmax = 0.0, rmax = 0.0;
        for (int i = 0; i < kb; ++i) tmax = fmax(tmax, fabs(rr->theta[i]));
        for (int i = 0; i < m; ++i) rmax = fmax(rmax, res[i]);
        rr->maxres = tmax > 0.0 ? rmax / tmax : rmax;
        rr->converged = (tol > 0.0 && rr->maxres <= tol) ? 1 : 0;
    }
}

}  // namespace sbmds
