// A3/A4: Y2 = D_ll Y1 and t = w^T Y2 ("W is small compared to n").
//
// D (l x l fp32, 10 GB at config 4) is streamed from HBM exactly once per apply by TMA
// (cp.async.bulk.tensor 2-D boxes -> shared memory, mbarrier pipeline, evict-first L2
// policy); the matching Y1 rows ride along as a 1-D bulk copy. Because D is symmetric
// a TMA box of D rows [k0, k0+BK) x columns [r0, r0+TM) is the
// k-major tile of D^T, so a thread's RM output rows are contiguous in shared memory and
// each D element is read from shared memory exactly once (by the one lane that owns its
// output row); the BP columns of Y1[k] are broadcast.
//
// Work split: stream-K. The T = RT x KT (row tile, k tile) iterations are cut into
// `grid` contiguous equal ranges, one per CTA (grid <= #SMs: one persistent CTA per SM,
// perfect balance). A CTA flushes a row tile's partial sum (fp64) when its range leaves
// that tile; k_dreduce adds the <= few partials of each row tile in CTA order
// (deterministic) and forms t = w^T Y2 (A4).
//
// Accumulation: fp32 FFMA over one pipeline stage (BK terms), folded into an fp64
// accumulator after every stage, so the long sum over l (50,000 at config 4) is carried
// in fp64 and the fp32 error is that of a BK-term sum (SURVEY.md §7 hard part 2).
#pragma once
#include "common.cuh"

namespace sbmds {

template <int BP>
struct DsCfg {
    static constexpr int CN = BP < 8 ? BP : 8;        // output columns per thread
    static constexpr int LC = BP / CN;                // lanes along columns
    static constexpr int LR = 32 / LC;                // lanes along rows
    static constexpr int RM = 4;                      // output rows per thread
    static constexpr int WR = LR * RM;                // rows per warp
    static constexpr int NCW = 8;                     // consumer warps
    static constexpr int TM = NCW * WR;               // rows per CTA tile
    static constexpr int BOXW = TM < 256 ? TM : 256;  // TMA box inner extent (elements)
    static constexpr int NBOX = TM / BOXW;
    static constexpr int BK = (8192 / TM) > 32 ? 32 : (8192 / TM);  // k per stage (32 KB of D)
    static constexpr int D_BYTES = TM * BK * 4;
    static constexpr int Y_BYTES = BK * BP * 4 < 16 ? 16 : BK * BP * 4;
    static constexpr int STAGE_BYTES = D_BYTES + ((Y_BYTES + 127) / 128) * 128;
    static constexpr int NS = (215 * 1024) / STAGE_BYTES > 8 ? 8 : (215 * 1024) / STAGE_BYTES;
    static constexpr int THREADS = (NCW + 1) * 32;
    static constexpr int SMEM = NS * STAGE_BYTES + 2 * NS * 8 + 128;
    static_assert(TM % BOXW == 0, "tile");
    static_assert(WR <= BOXW && BOXW % WR == 0, "a warp's rows must sit inside one box");
};

struct StreamK {
    int64_t T, RT, KT;
    int grid;
    __host__ __device__ int64_t beg(int c) const { return (int64_t)c * T / grid; }
    // CTA whose range contains iteration x
    __host__ __device__ int cta_of(int64_t x) const {
        int c = (int)((x * grid) / T);
        while (c + 1 < grid && beg(c + 1) <= x) ++c;
        while (c > 0 && beg(c) > x) --c;
        return c;
    }
};

template <int BP>
__global__ void __launch_bounds__(DsCfg<BP>::THREADS, 1)
    k_dstream_ffma(const __grid_constant__ CUtensorMap dmap, int64_t l, const float* __restrict__ Y1,
                   StreamK sk, int maxseg, double* __restrict__ P) {
    using C = DsCfg<BP>;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(base + C::NS * C::STAGE_BYTES);
    uint64_t* empty = full + C::NS;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x;
    const int64_t it0 = sk.beg(c), it1 = sk.beg(c + 1);

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], C::NCW);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == C::NCW) {
        // ---------------- producer warp: one elected lane issues TMA
        if (lane == 0) {
            prefetch_tensormap(&dmap);
            const uint64_t pol = policy_evict_first();
            int s = 0;
            uint32_t ph = 0;
            int64_t rt = it0 / sk.KT, kt = it0 % sk.KT;
            for (int64_t it = it0; it < it1; ++it) {
                mbar_wait(&empty[s], ph ^ 1u);
                uint8_t* st = base + s * C::STAGE_BYTES;
                mbar_arrive_expect_tx(&full[s], C::D_BYTES + C::Y_BYTES);
#pragma unroll
                for (int q = 0; q < C::NBOX; ++q)
                    tma_load_2d(st + q * C::BOXW * C::BK * 4, &dmap, &full[s],
                                (int32_t)(rt * C::TM + q * C::BOXW), (int32_t)(kt * C::BK), pol);
                bulk_load(st + C::D_BYTES, Y1 + kt * C::BK * BP, C::Y_BYTES, &full[s]);
                if (++s == C::NS) { s = 0; ph ^= 1u; }
                if (++kt == sk.KT) { kt = 0; ++rt; }
            }
        }
        return;
    }

    // ---------------- consumer warps
    const int li_ = lane % C::LR;  // row group within the warp
    const int lj = lane / C::LR;   // column group
    const int row_in_tile = warp * C::WR + li_ * C::RM;
    const int box = (warp * C::WR) / C::BOXW;
    const int col_in_box = (warp * C::WR) % C::BOXW + li_ * C::RM;
    float acc[C::RM][C::CN];
    double acc2[C::RM][C::CN];
#pragma unroll
    for (int r = 0; r < C::RM; ++r)
#pragma unroll
        for (int q = 0; q < C::CN; ++q) acc2[r][q] = 0.0;

    int s = 0;
    uint32_t ph = 0;
    int64_t rt = it0 / sk.KT, kt = it0 % sk.KT;
    int seg = c - sk.cta_of(rt * sk.KT);
    for (int64_t it = it0; it < it1; ++it) {
        mbar_wait(&full[s], ph);
        const uint8_t* st = base + s * C::STAGE_BYTES;
        const float* Ds = reinterpret_cast<const float*>(st + box * C::BOXW * C::BK * 4) + col_in_box;
        const float* Ys = reinterpret_cast<const float*>(st + C::D_BYTES) + lj * C::CN;
#pragma unroll
        for (int r = 0; r < C::RM; ++r)
#pragma unroll
            for (int q = 0; q < C::CN; ++q) acc[r][q] = 0.f;
#pragma unroll
        for (int kk = 0; kk < C::BK; ++kk) {
            float a[C::RM], bv[C::CN];
            const float4* ap = reinterpret_cast<const float4*>(Ds + kk * C::BOXW);
#pragma unroll
            for (int r4 = 0; r4 < C::RM / 4; ++r4) {
                const float4 v = ap[r4];
                a[4 * r4 + 0] = v.x; a[4 * r4 + 1] = v.y; a[4 * r4 + 2] = v.z; a[4 * r4 + 3] = v.w;
            }
            if constexpr (C::CN >= 4) {
                const float4* bp4 = reinterpret_cast<const float4*>(Ys + kk * BP);
#pragma unroll
                for (int q4 = 0; q4 < C::CN / 4; ++q4) {
                    const float4 v = bp4[q4];
                    bv[4 * q4 + 0] = v.x; bv[4 * q4 + 1] = v.y; bv[4 * q4 + 2] = v.z; bv[4 * q4 + 3] = v.w;
                }
            } else {
#pragma unroll
                for (int q = 0; q < C::CN; ++q) bv[q] = Ys[kk * BP + q];
            }
#pragma unroll
            for (int r = 0; r < C::RM; ++r)
#pragma unroll
                for (int q = 0; q < C::CN; ++q) acc[r][q] = fmaf(a[r], bv[q], acc[r][q]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
#pragma unroll
        for (int r = 0; r < C::RM; ++r)
#pragma unroll
            for (int q = 0; q < C::CN; ++q) acc2[r][q] += (double)acc[r][q];

        const bool last_of_tile = (it + 1 == it1) || (kt + 1 == sk.KT);
        if (last_of_tile) {
            double* out = P + ((rt * maxseg + seg) * (int64_t)C::TM + row_in_tile) * BP + lj * C::CN;
#pragma unroll
            for (int r = 0; r < C::RM; ++r) {
#pragma unroll
                for (int q = 0; q < C::CN; ++q) {
                    out[r * BP + q] = acc2[r][q];
                    acc2[r][q] = 0.0;
                }
            }
        }
        if (++s == C::NS) { s = 0; ph ^= 1u; }
        if (++kt == sk.KT) { kt = 0; ++rt; seg = 0; }
    }
}

// Sum the stream-K partials of each row tile in CTA order -> Y2 (l x BP fp32), and
// t = w^T Y2 (fp64, first b columns) by block partials + last-block reduction.
__global__ void __launch_bounds__(256) k_dreduce(int64_t l, int bp, int b, int tm, StreamK sk, int maxseg,
                                                 const double* __restrict__ P, const double* __restrict__ w,
                                                 float* __restrict__ Y2, double* __restrict__ tpart,
                                                 double* __restrict__ t, unsigned int* __restrict__ counter) {
    __shared__ double red[256];
    const int rows_per_blk = 256 / bp;
    const int tid = threadIdx.x;
    const int cidx = tid % bp, rloc = tid / bp;
    double acc_t = 0.0;
    // grid-stride over row blocks
    for (int64_t r0 = (int64_t)blockIdx.x * rows_per_blk; r0 < l; r0 += (int64_t)gridDim.x * rows_per_blk) {
        const int64_t r = r0 + rloc;
        if (rloc < rows_per_blk && r < l) {
            const int64_t rt = r / tm;
            const int c0 = sk.cta_of(rt * sk.KT);
            const int c1 = sk.cta_of(rt * sk.KT + sk.KT - 1);
            double v = 0.0;
            for (int seg = 0; seg <= c1 - c0; ++seg)
                v += P[((rt * maxseg + seg) * (int64_t)tm + (r - rt * tm)) * bp + cidx];
            Y2[r * bp + cidx] = (float)v;
            if (cidx < b) acc_t += w[r] * v;
        }
    }
    red[tid] = (rloc < rows_per_blk) ? acc_t : 0.0;
    __syncthreads();
    if (tid < bp) {
        double v = 0.0;
        for (int q = 0; q < rows_per_blk; ++q) v += red[q * bp + tid];
        tpart[blockIdx.x * kMaxB + tid] = v;
    }
    if (last_block_done(counter)) {
        if (tid < bp) t[tid] = ordered_sum(tpart + tid, gridDim.x, kMaxB);
        if (tid == 0) *counter = 0;
    }
}

}  // namespace sbmds
