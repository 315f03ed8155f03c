// Shared device helpers for libsbmds (sm_100a). No method arithmetic lives here.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

namespace sbmds {

constexpr int kWarp = 32;
constexpr int kMaxB = 64;

extern std::atomic<int64_t> g_launches;  // every kernel launch / captured node replayed

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ---------------------------------------------------------------- mbarrier / TMA (PTX)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Watchdog for pipeline waits: a wait that has not completed after ~4 s records where it is
// stuck (tag, CTA, thread, parity) in host-mapped memory and traps, so a pipeline bug turns
// into an SBMDS_ECUDA error with a location instead of a hung process.
struct HangEntry {
    unsigned int tag, block, thread, parity, bar_lo, bar_hi;
};
struct HangRecord {
    unsigned int flag, count, pad0, pad1;
    HangEntry e[512];
};
__device__ HangRecord* g_hang = nullptr;   // single translation unit (sbmds.cu)

__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t"
        ".reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t"
        "}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// non-blocking test (test_wait never suspends the thread; try_wait may, for a time limit)
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t"
        ".reg .pred P1;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t"
        "}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __noinline__ void mbar_hang(uint64_t* bar, uint32_t parity, int tag) {
    HangRecord* r = g_hang;
    if (r) {
        const unsigned k = atomicAdd(&r->count, 1u);
        if (k < 512) {
            const uint64_t st = *reinterpret_cast<volatile uint64_t*>(bar);
            r->e[k] = HangEntry{(unsigned)tag, blockIdx.x, threadIdx.x, parity, (unsigned)st, (unsigned)(st >> 32)};
        }
        r->flag = 1u;
        __threadfence_system();
        // let the other stuck waits of this launch time out and record themselves too
        uint64_t t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while (t - t0 < 1500000000ull);
    }
    __trap();
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity, int tag = 0) {
    if (mbar_try(bar, parity)) return;
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (uint32_t k = 1;; ++k) {
        if (mbar_try(bar, parity)) return;
        if ((k & 1023u) == 0u) {
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > 4000000000ull) mbar_hang(bar, parity, tag);
        }
    }
}

// 2-D TMA tile load global -> shared, completion on mbarrier (complete_tx bytes).
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int32_t c0, int32_t c1, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::"
        "cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
        : "memory");
}

// 3-D TMA tile load (tile-packed D: {col, row, tile}).
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0, int32_t c1,
                                            int32_t c2, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::"
        "cache_hint [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
        : "memory");
}

// one lane of a converged warp (elect.sync): tcgen05 issue from warp-uniform code, so the
// operands stay in uniform registers (no per-instruction waterfall)
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .b32 rx;\n\t.reg .pred px;\n\telect.sync rx|px, 0xffffffff;\n\t@px mov.s32 %0, 1;\n\t}"
        : "+r"(pred));
    return pred != 0;
}

// ---------------------------------------------------------------- programmatic dependent launch
// Kernels of the eigs chain are launched with programmatic stream serialization: a kernel lets
// its successor start launching at once (trigger) and waits for its predecessor's completion
// and memory (wait) before touching anything an earlier kernel produced. Both are no-ops for a
// normal launch.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ---------------------------------------------------------------- thread-block clusters
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// all threads of all CTAs of the cluster
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
}
// shared::cluster address of `p` (own smem) in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster_u32(uint32_t cluster_addr, uint32_t v) {
    asm volatile("st.relaxed.cluster.shared::cluster.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.cluster.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}

// 1-D bulk copy global -> shared (bytes % 16 == 0, both 16-byte aligned).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ void prefetch_tensormap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// order-preserving unsigned keys of floats (atomicMax / atomicMin over signed values)
__host__ __device__ __forceinline__ unsigned int f32_order_key(float f) {
    unsigned int u;
    memcpy(&u, &f, 4);
    return (u >> 31) ? ~u : (u | 0x80000000u);
}
__host__ __device__ __forceinline__ float f32_from_order_key(unsigned int k) {
    const unsigned int u = (k >> 31) ? (k & 0x7FFFFFFFu) : ~k;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

// Fixed-order sum of p[0], p[stride], ..., p[(count-1)*stride] with 16 loads in flight:
// the additions happen in index order (bitwise reproducible) but the L2 latency of the
// partials is overlapped instead of serialised.
template <int U = 16>
__device__ __forceinline__ double ordered_sum(const double* __restrict__ p, int count, int64_t stride) {
    // U loads in flight per batch, the last batch predicated (no serial tail), added in index order
    double acc = 0.0;
    for (int q = 0; q < count; q += U) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = q + u < count ? p[(int64_t)(q + u) * stride] : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (q + u < count) acc += v[u];
    }
    return acc;
}

// ordered_sum for the four entries tid, tid + 256, tid + 512, tid + 768 (< nent) of a 256-thread
// last block at once: the loads of all four of a batch are in flight together (a b = 32 Gram's
// last block otherwise serialises ~80 L2 round trips per thread). Each entry is added in index
// order (absent entries and the batch tail add exact zeros), so the sums equal ordered_sum's.
template <int U = 8>
__device__ __forceinline__ void ordered_sum_x4(const double* __restrict__ p, int tid, int nent, int count,
                                               int64_t stride, double (&acc)[4]) {
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[e] = 0.0;
    for (int q = 0; q < count; q += U) {
        double v[4][U];
#pragma unroll
        for (int e = 0; e < 4; ++e)
#pragma unroll
            for (int u = 0; u < U; ++u)
                v[e][u] = (tid + 256 * e < nent && q + u < count) ? p[(int64_t)(q + u) * stride + tid + 256 * e] : 0.0;
#pragma unroll
        for (int e = 0; e < 4; ++e)
#pragma unroll
            for (int u = 0; u < U; ++u) acc[e] += v[e][u];
    }
}

// Block-wide fixed-order column sums for a last block: out[c] = sum over q < count of
// p[q * stride + c], 1 <= ncols <= 256. Thread (c, k), k < 256 / ncols, sums chunk k of the q
// range in order, then thread c adds the chunk results in order: a fixed order, so the result
// is bitwise reproducible, with up to 256 loads in flight instead of ncols.
__device__ __forceinline__ void ordered_colsum_block(const double* __restrict__ p, int count, int64_t stride, int ncols,
                                                     double* __restrict__ out) {
    __shared__ double chunk[256];
    const int tid = threadIdx.x, nk = 256 / ncols;
    const int c = tid % ncols, k = tid / ncols;
    if (k < nk) {
        const int per = (count + nk - 1) / nk, q0 = k * per, q1 = min(count, q0 + per);
        double a = 0.0;
        int q = q0;
        for (; q + 8 <= q1; q += 8) {   // eight loads in flight, added in index order (same result)
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = p[(int64_t)(q + u) * stride + c];
#pragma unroll
            for (int u = 0; u < 8; ++u) a += v[u];
        }
        for (; q < q1; ++q) a += p[(int64_t)q * stride + c];
        chunk[k * ncols + c] = a;
    }
    __syncthreads();
    if (tid < ncols) {
        double v = 0.0;
        for (int kk = 0; kk < nk; ++kk) v += chunk[kk * ncols + tid];
        out[tid] = v;
    }
}

// Last-block-done pattern for deterministic grid reductions: every block writes its
// partial, fences, and bumps a counter; the block that sees count == grid-1 does the
// final fixed-order reduction and resets the counter for the next launch.
// last_block_done among the first `nblocks` blocks only (they alone arrive on `counter`)
__device__ __forceinline__ bool last_block_of(unsigned int* counter, unsigned int nblocks) {
    __shared__ bool is_last_of;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last_of = atomicAdd(counter, 1u) == nblocks - 1;
    __syncthreads();
    if (is_last_of) __threadfence();
    return is_last_of;
}

__device__ __forceinline__ bool last_block_done(unsigned int* counter) {
    __shared__ bool is_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int prev = atomicAdd(counter, 1u);
        is_last = (prev == gridDim.x * gridDim.y * gridDim.z - 1);
    }
    __syncthreads();
    if (is_last) __threadfence();
    return is_last;
}

}  // namespace sbmds
