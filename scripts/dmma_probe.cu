// FP64 tensor-core (mma.sync f64) cost on sm_100a: cycles per instruction per warp for the
// shapes m8n8k4 / m16n8k4 / m16n8k8 / m16n8k16, with 1..6 independent accumulator chains, one
// warp per SM sub-partition (and 2 warps on one), against plain DFMA. Prints cycles / instr.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void dmma1684(double (&d)[4], double (&a)[2], double b) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(b));
}
__device__ __forceinline__ void dmma1688(double (&d)[4], double (&a)[4], double (&b)[2]) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void dmma16816(double (&d)[4], double (&a)[8], double (&b)[4]) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
                 "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
                   "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int SHAPE, int CH>
__global__ void k(int iters, int active_warps_mask, double* out, long long* cyc) {
    const int warp = threadIdx.x >> 5;
    double a[8], b[4];
    for (int i = 0; i < 8; ++i) a[i] = 1.0 + 1e-9 * (threadIdx.x + i);
    for (int i = 0; i < 4; ++i) b[i] = 1.0 - 1e-9 * (threadIdx.x + i);
    double d[CH][4];
    for (int c = 0; c < CH; ++c) for (int i = 0; i < 4; ++i) d[c][i] = 0.0;
    __syncthreads();
    if (!((active_warps_mask >> warp) & 1)) return;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            if constexpr (SHAPE == 0) dmma884(*reinterpret_cast<double(*)[2]>(&d[c][0]), a[0], b[0]);
            if constexpr (SHAPE == 1) dmma1684(d[c], *reinterpret_cast<double(*)[2]>(&a[0]), b[0]);
            if constexpr (SHAPE == 2) dmma1688(d[c], *reinterpret_cast<double(*)[4]>(&a[0]), *reinterpret_cast<double(*)[2]>(&b[0]));
            if constexpr (SHAPE == 3) dmma16816(d[c], a, b);
            if constexpr (SHAPE == 4) {   // plain DFMA, 4 per "instruction" slot
                d[c][0] = fma(a[0], b[0], d[c][0]);
                d[c][1] = fma(a[1], b[1], d[c][1]);
                d[c][2] = fma(a[2], b[2], d[c][2]);
                d[c][3] = fma(a[3], b[3], d[c][3]);
            }
        }
    }
    long long t1 = clock64();
    double s = 0;
    for (int c = 0; c < CH; ++c) for (int i = 0; i < 4; ++i) s += d[c][i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if ((threadIdx.x & 31) == 0 && blockIdx.x == 0) cyc[warp] = t1 - t0;
}

template <int SHAPE, int CH>
void run(const char* name, int mask, int threads) {
    double* out; long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&cyc, 64 * 8);
    const int iters = 2000;
    k<SHAPE, CH><<<148, threads>>>(iters, mask, out, cyc);
    k<SHAPE, CH><<<148, threads>>>(iters, mask, out, cyc);
    cudaDeviceSynchronize();
    long long h[32];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    int w0 = 0; while (!((mask >> w0) & 1)) ++w0;
    printf("%-10s chains %d warps-mask 0x%x: %.1f cycles per instruction per warp (%.1f per chain step) err=%s\n", name, CH, mask,
           (double)h[w0] / (iters * CH), (double)h[w0] / iters, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out); cudaFree(cyc);
}

int main() {
    // one warp alone on the SM
    run<0, 1>("m8n8k4", 1, 128); run<0, 2>("m8n8k4", 1, 128); run<0, 3>("m8n8k4", 1, 128); run<0, 6>("m8n8k4", 1, 128);
    run<1, 1>("m16n8k4", 1, 128); run<1, 3>("m16n8k4", 1, 128); run<1, 6>("m16n8k4", 1, 128);
    run<2, 1>("m16n8k8", 1, 128); run<2, 3>("m16n8k8", 1, 128); run<2, 6>("m16n8k8", 1, 128);
    run<3, 1>("m16n8k16", 1, 128); run<3, 2>("m16n8k16", 1, 128); run<3, 4>("m16n8k16", 1, 128);
    run<4, 1>("4xDFMA", 1, 128); run<4, 4>("4xDFMA", 1, 128); run<4, 8>("4xDFMA", 1, 128);
    // four warps, one per sub-partition (SM-level throughput)
    run<0, 6>("m8n8k4", 0xF, 128); run<3, 4>("m16n8k16", 0xF, 128); run<2, 6>("m16n8k8", 0xF, 128); run<4, 8>("4xDFMA", 0xF, 128);
    // two warps on the same sub-partition (warps 0 and 4)
    run<0, 6>("m8n8k4", 0x11, 256); run<3, 4>("m16n8k16", 0x11, 256); run<4, 8>("4xDFMA", 0x11, 256);
    // 8 warps
    run<0, 6>("m8n8k4", 0xFF, 256); run<4, 8>("4xDFMA", 0xFF, 256);
    return 0;
}
