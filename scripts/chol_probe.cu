// Cycle cost of chol_block (k_small.cuh) inside one CTA, b = 16: G random SPD, 20 repeats,
// clock64 per repeat (thread 0), both the warp-register path and the block smem path (b = 15).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1705_10887_b200/csrc/common.cuh"
#include "../paper_1705_10887_b200/csrc/k_small.cuh"
using namespace sbmds;
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
        }
    }
    double* o; long long* c; cudaMalloc(&o, 256 * 8); cudaMemset(o, 0, 256 * 8); cudaMalloc(&c, 24);
    probe_ops<<<1, 32>>>(o, c);
    long long h[3]; cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
    printf("fp64 dependent latency (cycles): sqrt+add %lld, rcp+add %lld, fma %lld\n", h[0], h[1], h[2]);
    return 0;
}
