// Cycle cost of chol_block (k_small.cuh) inside one CTA, b = 16: G random SPD, 20 repeats,
// clock64 per repeat (thread 0), both the warp-register path and the block smem path (b = 15).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1705_10887_b200/csrc/common.cuh"
#include "../paper_1705_10887_b200/csrc/k_small.cuh"
using namespace sbmds;
namespace sbmds {
__device__ void chol_timed(int b, const double* __restrict__ G, double* __restrict__ Rinv, int* __restrict__ status,
                           double (*A)[kMaxB + 1], int* fail_s, double* shift_s, long long* tm) {
    long long c0 = clock64();
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
            shift = attempt == 0 ? 0.0 : 1e-13 * tr + 1e-300;
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
    long long c1 = clock64();
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
    __syncthreads();
    long long c2 = clock64();
    if (tid == 0) { *status = (shift > 0.0) ? 1 : 0; tm[0] = c1 - c0; tm[1] = c2 - c1; }
}

}
__global__ void probe(int b, const double* G, double* Rinv, int* status, long long* cyc, int reps) {
    __shared__ double A[kMaxB][kMaxB + 1];
    __shared__ int fail;
    __shared__ double shift;
    for (int r = 0; r < reps; ++r) {
        __syncthreads();
        long long t0 = clock64();
        chol_block(b, G, Rinv, status, A, &fail, &shift);
        __syncthreads();
        long long t1 = clock64();
        if (threadIdx.x == 0) cyc[r] = t1 - t0;
    }
}
__global__ void probe_ops(double* out, long long* cyc) {
    double x = out[threadIdx.x] + 2.0;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 100; ++i) x = sqrt(x) + 1.0;
    long long t1 = clock64();
#pragma unroll 1
    for (int i = 0; i < 100; ++i) x = 1.0 / x + 1.0;
    long long t2 = clock64();
#pragma unroll 1
    for (int i = 0; i < 100; ++i) x = fma(x, 0.999, 0.5);
    long long t3 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / 100; cyc[1] = (t2 - t1) / 100; cyc[2] = (t3 - t2) / 100; }
}
__global__ void probe_t(int b, const double* G, double* Rinv, int* status, long long* tm) {
    __shared__ double A[kMaxB][kMaxB + 1];
    __shared__ int fail;
    __shared__ double shift;
    for (int r = 0; r < 3; ++r) { __syncthreads(); chol_timed(b, G, Rinv, status, A, &fail, &shift, tm + 2 * r); }
}
int main() {
    for (int b : {16, 15}) {
        std::vector<double> M(b * b), G(b * b, 0.0);
        srand(1);
        for (auto& v : M) v = rand() / (double)RAND_MAX - 0.5;
        for (int i = 0; i < b; ++i) for (int j = 0; j < b; ++j) { double s = 0; for (int k = 0; k < b; ++k) s += M[k * b + i] * M[k * b + j]; G[i * b + j] = s + (i == j); }
        double *dG, *dR; int* ds; long long* dc;
        cudaMalloc(&dG, b * b * 8); cudaMalloc(&dR, b * b * 8); cudaMalloc(&ds, 4); cudaMalloc(&dc, 20 * 8);
        cudaMemcpy(dG, G.data(), b * b * 8, cudaMemcpyHostToDevice);
        for (int threads : {256, 512}) {
            probe<<<1, threads>>>(b, dG, dR, ds, dc, 20);
            long long c[20]; cudaMemcpy(c, dc, sizeof c, cudaMemcpyDeviceToHost);
            int st; cudaMemcpy(&st, ds, 4, cudaMemcpyDeviceToHost);
            printf("b=%d threads=%d status=%d cycles: first %lld, then %lld %lld %lld\n", b, threads, st, c[0], c[5], c[10], c[19]);
            probe_t<<<1, threads>>>(b, dG, dR, ds, dc);
            cudaMemcpy(c, dc, 6 * 8, cudaMemcpyDeviceToHost);
            printf("   factor %lld / %lld / %lld, back-substitution %lld / %lld / %lld cycles\n", c[0], c[2], c[4], c[1], c[3], c[5]);
        }
    }
    double* o; long long* c; cudaMalloc(&o, 256 * 8); cudaMemset(o, 0, 256 * 8); cudaMalloc(&c, 24);
    probe_ops<<<1, 32>>>(o, c);
    long long h[3]; cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
    printf("fp64 dependent latency (cycles): sqrt+add %lld, rcp+add %lld, fma %lld\n", h[0], h[1], h[2]);
    return 0;
}
