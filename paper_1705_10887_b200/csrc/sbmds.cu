// libsbmds — C-ABI implementation (include/sbmds.h). Host driver of the sBMDS hot path:
// create (C1, C2), apply (A1-A5), eigs (E1-E6); see DESIGN.md §4 for the step list.
#include <cub/cub.cuh>
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <nccl.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/sbmds.h"
#include "common.cuh"
#include "k_dstream.cuh"
#include "k_dstream_tc.cuh"
#include "k_dstream_pair.cuh"
#include "k_dstream_sym8.cuh"
#include "k_small.cuh"
#include "k_sparse.cuh"
#include "k_blocked.cuh"
#include "k_fused.cuh"
#include "k_sp8.cuh"
#include "k_lanczos.cuh"
#include "k_bmds.cuh"
#include "k_sbha.cuh"

namespace sbmds {
std::atomic<int64_t> g_launches{0};
}

using namespace sbmds;

// ============================================================================ errors
namespace {
thread_local std::string t_err;

sbmds_status fail(sbmds_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    t_err = buf;
    return st;
}

struct CudaError {
    cudaError_t e;
    const char* what;
};

#define CK(call)                                                  \
    do {                                                          \
        cudaError_t _e = (call);                                  \
        if (_e != cudaSuccess) throw CudaError{_e, #call};        \
    } while (0)

template <typename K, typename... Args>
void launch(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    kernel<<<grid, block, smem, st>>>(args...);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    CK(cudaGetLastError());
}

// Launch with programmatic stream serialization (the eigs chain kernels call pdl_trigger /
// pdl_wait, common.cuh): the launch overlaps the predecessor's tail.
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

// Cooperative launch (all blocks co-resident; the kernel may call grid.sync()).
template <typename... KArgs, typename... Args>
void launch_coop_x(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 2 : 1;
    CK(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

template <typename... KArgs, typename... Args>
void launch_coop(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    launch_coop_x(false, kernel, grid, block, smem, st, args...);
}
// cooperative + programmatic serialization (the kernel calls pdl_trigger / pdl_wait)
template <typename... KArgs, typename... Args>
void launch_coop_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    launch_coop_x(true, kernel, grid, block, smem, st, args...);
}

HangRecord* g_hang_host = nullptr;

// NVTX ranges (SURVEY §5 tracing): one per public call and per eigs / create stage, on the host
// timeline of nsys / ncu --nvtx; no cost without a tool attached.
struct Nvtx {
    explicit Nvtx(const char* what) { nvtxRangePushA(what); }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx&) = delete;
    Nvtx& operator=(const Nvtx&) = delete;
};

// Per-device one-time setup. CUDA keeps kernel attributes, the default memory pool and module
// symbols per device, so every "once" below is keyed by the current device and guarded by a
// mutex (distinct handles may live on different GPUs and be used from different threads).
std::mutex g_once_mu;

bool once_per_device(const void* what, int extra = 0) {
    static std::set<std::tuple<int, const void*, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(g_once_mu);
    return done.insert(std::make_tuple(dev, what, extra)).second;
}

// Opt `kernel` into `bytes` of dynamic shared memory on the current device (once per device
// and size; a later launch with the same size skips the driver call).
template <typename K>
void smem_attr(K* kernel, int bytes) {
    static std::mutex mu;
    static std::set<std::tuple<int, const void*, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);   // held across the call: no launch sees the key before the attribute
    const auto key = std::make_tuple(dev, (const void*)kernel, bytes);
    if (done.count(key)) return;
    CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done.insert(key);
}

// Host-mapped record the device watchdog writes before trapping (common.cuh mbar_wait); the
// symbol g_hang exists once per device, so each device gets the (shared) record's address.
void install_hang_record() {
    static HangRecord* hp = nullptr;
    static HangRecord* dp = nullptr;
    {
        std::lock_guard<std::mutex> g(g_once_mu);
        if (!hp) {
            if (cudaHostAlloc(reinterpret_cast<void**>(&hp), sizeof(HangRecord), cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
                cudaGetLastError();
                hp = nullptr;
                return;
            }
            memset(hp, 0, sizeof(HangRecord));
            if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&dp), hp, 0) != cudaSuccess) {
                cudaGetLastError();
                return;
            }
        }
    }
    if (!dp || !once_per_device((const void*)&install_hang_record)) return;
    if (cudaMemcpyToSymbol(g_hang, &dp, sizeof(dp)) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    g_hang_host = hp;
}

// Small device -> host readbacks during create go through a host-mapped buffer written by a
// kernel, not a copy: a D2H copy would queue behind the host D's multi-GB upload on the copy
// engines and stall the S-side builds that overlap it.
__global__ void k_peek(const unsigned char* __restrict__ src, unsigned char* __restrict__ dst, int bytes) {
    for (int i = threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
}

void peek_to_host(void* host_dst, const void* dev_src, size_t bytes, cudaStream_t st) {
    static std::mutex mu;   // one mapped buffer for all handles and threads
    std::lock_guard<std::mutex> g(mu);
    static unsigned char* hbuf = nullptr;
    static unsigned char* dbuf = nullptr;
    if (!hbuf) {
        CK(cudaHostAlloc(reinterpret_cast<void**>(&hbuf), 4096, cudaHostAllocMapped | cudaHostAllocPortable));
        CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dbuf), hbuf, 0));
    }
    if (bytes > 4096) throw CudaError{cudaErrorInvalidValue, "peek_to_host"};
    k_peek<<<1, 128, 0, st>>>(reinterpret_cast<const unsigned char*>(dev_src), dbuf, (int)bytes);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    memcpy(host_dst, hbuf, bytes);
}

// NCCL for the sharded apply, loaded on first use (dlopen "libnccl.so.2": the copy torch already
// loaded when there is one, so ids from either side match); the single-GPU library does not
// depend on it.
struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!so) {
            api.why = dlerror() ? dlerror() : "dlopen(libnccl.so.2) failed";
            return;
        }
        auto sym = [&](const char* name) { return dlsym(so, name); };
        api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(sym("ncclGetUniqueId"));
        api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(sym("ncclCommInitRank"));
        api.allReduce = reinterpret_cast<decltype(api.allReduce)>(sym("ncclAllReduce"));
        api.groupStart = reinterpret_cast<decltype(api.groupStart)>(sym("ncclGroupStart"));
        api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(sym("ncclGroupEnd"));
        api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(sym("ncclCommDestroy"));
        api.errorString = reinterpret_cast<decltype(api.errorString)>(sym("ncclGetErrorString"));
        api.ok = api.getUniqueId && api.commInitRank && api.allReduce && api.groupStart && api.groupEnd &&
                 api.commDestroy && api.errorString;
        if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
    });
    return api;
}

struct NcclError {
    ncclResult_t r;
    const char* what;
};
#define NK(call)                                             \
    do {                                                     \
        ncclResult_t _r = (call);                            \
        if (_r != ncclSuccess) throw NcclError{_r, #call};   \
    } while (0)

std::string hang_note() {
    if (!g_hang_host || !g_hang_host->flag) return "";
    std::string out = " [pipeline watchdog:";
    const unsigned n = std::min(512u, g_hang_host->count);
    std::vector<uint64_t> seen;
    for (unsigned k = 0; k < n; ++k) {
        const HangEntry& e = g_hang_host->e[k];
        const uint64_t key = ((uint64_t)e.tag << 32) | ((uint64_t)e.block << 8) | (e.thread / 32);
        if (std::find(seen.begin(), seen.end(), key) != seen.end()) continue;   // one line per (tag, block, warp)
        seen.push_back(key);
        char buf[128];
        snprintf(buf, sizeof buf, " tag %u.%u blk %u thr %u par %u;", e.tag >> 16, e.tag & 0xFFFF, e.block, e.thread,
                 e.parity);
        out += buf;
    }
    return out + "]";
}

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int next_pow2(int b) {
    int p = 1;
    while (p < b) p <<= 1;
    return p;
}

// Device buffers. Long-lived handle buffers (`pooled`) come from the device's default
// stream-ordered memory pool with an unbounded release threshold, so memory freed by
// sbmds_destroy stays mapped and the next sbmds_create reuses it (re-mapping ~12 GB per
// create/destroy cycle cost 0.1-0.3 s stalls). Frees of pooled buffers happen only when the
// device is idle for them (destroy syncs first; a growing ensure() syncs before freeing).
// Create-time temporaries use plain cudaMalloc/cudaFree.
void configure_pool_once() {
    if (!once_per_device((const void*)&configure_pool_once)) return;
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
}

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    bool pooled = false;
    DevBuf() = default;
    explicit DevBuf(bool pool) : pooled(pool) {}   // pool = true: stream-ordered pool allocation
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void ensure(size_t nb) {
        if (nb <= bytes) return;
        if (p && pooled) cudaDeviceSynchronize();   // the old buffer may still be in flight
        release();
        cudaError_t e;
        if (pooled) {
            e = cudaMallocAsync(&p, nb, 0);
            if (e == cudaSuccess) e = cudaStreamSynchronize(0);
        } else {
            e = cudaMalloc(&p, nb);
        }
        if (e != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            throw CudaError{e, pooled ? "cudaMallocAsync" : "cudaMalloc"};
        }
        bytes = nb;
    }
    void release() {
        if (p) {
            if (pooled) cudaFreeAsync(p, 0);
            else cudaFree(p);
        }
        p = nullptr;
        bytes = 0;
    }
    template <typename T>
    T* as() const { return reinterpret_cast<T*>(p); }
    void swap(DevBuf& o) {
        std::swap(p, o.p);
        std::swap(bytes, o.bytes);
        std::swap(pooled, o.pooled);
    }
};

// Row-blocked index of S (k_blocked.cuh) for blocks of rb rows: dictionaries, 16-bit local
// columns (CSR order), optional block-local CSC, and landmark -> dictionary-slot lists.
struct BlkIdx {
    DevBuf doff{true}, dict{true}, lcol{true}, lcp{true}, lrow{true}, lval{true}, jptr{true}, jlist{true};
    DevBuf brow0{true};   // (tensor-core step) first row of each block, nblk + 1 entries: blocks are <= rb rows
    int rb = 0;
    int64_t nblk = 0;
    int32_t total_u = 0;
    uint32_t umax = 0;
    void reset() {
        for (DevBuf* b : {&doff, &dict, &lcol, &lcp, &lrow, &lval, &jptr, &jlist, &brow0}) b->release();
        rb = 0;
        nblk = 0;
        total_u = 0;
        umax = 0;
    }
};

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda needed).
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !p) {
            cudaGetLastError();
            return nullptr;
        }
        fn = reinterpret_cast<EncodeFn>(p);
    }
    return fn;
}

// Per-kernel-family device timing with CUDA events recorded on the launching stream
// (sbmds_set_option "profile" = bitmask of families; read back with sbmds_get_stat
// "<family>_ns" / "<family>_launches"). Used by bench.py for the roofline line.
enum { PK_COLSUM = 0, PK_CSC, PK_DSTREAM, PK_DREDUCE, PK_CSR, PK_GRAM, PK_CHOL, PK_ROTATE, PK_RR, PK_SPLIT, PK_N };
const char* const kProfNames[PK_N] = {"colsum", "csc", "dstream", "dreduce", "csr", "gram", "chol", "rotate", "rr", "split"};

struct Profiler {
    uint32_t mask = 0;
    std::vector<cudaEvent_t> pool;
    struct Pend { int k; cudaEvent_t a, b; };
    std::vector<Pend> pend;
    double ns[PK_N] = {0};
    int64_t cnt[PK_N] = {0};
    cudaEvent_t get() {
        if (pool.empty()) {
            cudaEvent_t e;
            if (cudaEventCreate(&e) != cudaSuccess) throw CudaError{cudaErrorMemoryAllocation, "cudaEventCreate"};
            return e;
        }
        cudaEvent_t e = pool.back();
        pool.pop_back();
        return e;
    }
    void drain() {
        for (auto& p : pend) {
            float ms = 0.f;
            cudaEventSynchronize(p.b);
            cudaEventElapsedTime(&ms, p.a, p.b);
            ns[p.k] += 1e6 * (double)ms;
            cnt[p.k] += 1;
            pool.push_back(p.a);
            pool.push_back(p.b);
        }
        pend.clear();
    }
    ~Profiler() {
        for (auto& p : pend) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
        for (auto e : pool) cudaEventDestroy(e);
    }
};

template <typename F>
void profiled(Profiler& pr, int k, cudaStream_t st, F&& f) {
    if (!(pr.mask & (1u << k))) {
        f();
        return;
    }
    cudaEvent_t a = pr.get(), b = pr.get();
    CK(cudaEventRecord(a, st));
    f();
    CK(cudaEventRecord(b, st));
    pr.pend.push_back({k, a, b});
}

constexpr int kBmdsMaxL = 8192;  // BMDS: dense l x l fp64 factors (512 MB at the limit)
constexpr int kRedBlocks = 296;  // 2 x 148 SMs for the grid reductions
constexpr int kCounters = 8;
enum { CNT_COLSUM = 0, CNT_DRED = 1, CNT_GRAM = 2, CNT_ARGMAX = 3, CNT_ROTATE = 4, CNT_FOLD = 5 };

}  // namespace

// ============================================================================ handle
struct sbmds_ctx {
    int64_t n = 0, l = 0, nnz = 0;
    // sharded apply: this handle holds rows [row0, row0 + n) of an n_global-row S
    // and streams tile range `rank` of `world` of D's upper triangle; comm = NCCL communicator
    // attached by sbmds_shard_attach_nccl (NULL: the caller drives sbmds_shard_stage)
    int64_t n_global = 0, row0 = 0;
    int rank = 0, world = 1;
    bool shard = false;
    void* comm = nullptr;
    DevBuf Y1w, Y2w, tsave;    // b <= 4 / b > 32 on the int8 stream: Y1 / Y2 at pitch 8 / 32, t halves
    DevBuf vg;                 // shard: v_g = D w_g (t_g = v_g^T Y1, formed at the first stage 2)
    // row order (reorder_rows): the handle keeps S's rows permuted when 128-row blocks then touch
    // fewer landmarks; perm[r] = caller's row of handle row r. X / Y / V cross it at the ABI.
    bool permuted = false;
    DevBuf perm, xperm, yperm;
    int64_t order_distinct[2] = {0, 0};   // sampled blocks' distinct columns: natural, permuted
    bool vg_ok = false;
    int dev = 0, num_sms = 148;
    // S (CSR) and its device-built CSC copy
    DevBuf rp, col, val, cptr, ridx, cval, order, w;
    // row-blocked S (k_blocked.cuh): per 256-row block a landmark dictionary, 16-bit local
    // columns for S Y2, a block-local CSC (8-bit rows) for S^T X, and the landmark -> slot lists
    DevBuf bdoff, bdict, blcp, blcol, blrow, blval, bjptr, bjlist, P1;
    int64_t nblk = 0;
    int32_t total_u = 0;
    uint32_t umax = 0;
    bool blocked = false;
    int use_blocked = 1;   // bit 0: S Y2 through the blocked kernel, bit 1: S^T X too
    bool blocked_auto = true;   // (no "blocked" option set) standalone applies with b >= 32 use mask 2
    int gram_tc = 1;       // Gram on the FP64 tensor cores (b <= 32)
    int csr_nnz_per_lane = 4;   // narrow CSR SpMM: nonzeros per lane when choosing lanes per row
    int csr_sub_L = 0;          // (tuning) force lanes per row
    int csr_shfl = -1;          // (tuning) k_spmm_csr_vec4's shuffled pair loads: -1 auto, 0 off, 1 on
    int fuse = 3;          // eigs: 1 = A5 fused with the Gram, 2 = also the next A2's S^T partials (k_fused.cuh),
                           // 3 = the tensor-core sparse step where it applies (k_sp8.cuh), else 1
    // tensor-core sparse step (k_sp8.cuh): 128-row blocks, dense three-plane digit images of S_B
    BlkIdx s8;
    DevBuf s8img, s8ioff, s8esc, s8yd, s8trace, s8rs1, s8pos;
    int sp8_state = 0;     // 0 not built, 1 built, -1 not applicable (a dictionary > 128 entries)
    bool y1f_ready = false;   // the fused landmark reduce already formed Y1f (+ its column max) this apply
    bool y2d_want = false;    // the sparse step follows this apply's D stream: digitise Y2 in the reduce
    bool y2d_ready = false;   // k_dreduce_y2d formed Y2's digit planes (launch_sp8 skips k_y2_digits)
    bool gram_deferred = false;   // the last sparse step left G, s, R^-1 to the next fold (FoldGram)
    int gram_parts = 0;           // its CTA count
    DevBuf foldscr;               // lpad x 16 fp64 landmark sums of the deferred-Gram fold
    int solver = 0;        // eigs: 0 block subspace iteration, 1 restarted block Lanczos (k_lanczos.cuh)
    int lz_blocks = 0;     // Lanczos blocks per restart cycle (0: 64 / block)
    DevBuf lzQ, lzW, lzC, lzT, lzGl, lzI, lzR;
    int sp8_dbg = 0;       // diagnostics (timing only, results invalid): 1 = skip the T product,
                           // 2 = timeline of CTA 0, 4 = stream the images only, 8 = T product in the last iteration too,
                           // 16 = no H' (as between Rayleigh-Ritz steps), 256 = no Gram, 512 = no T drain arithmetic
    int sp8_poll = 0;      // k_sp8_step: the MMA warp's back-off (ns) between unready polls
    int sp8_pf = 0;        // k_sp8_step: L2 prefetch distance of the images, in blocks (0: off)
    int sp8_gram8 = 1;     // k_sp8_step: int8-tensor-core Gram on steps that feed no Rayleigh-Ritz step
    int sp8_apply = 1;     // standalone apply at b = 16: A5 through the tensor-core step's N products
    int64_t sp8_min_rows = 16 * 128 * 148;   // ... only from this many rows on (the kernels' fixed costs lose to the fp32
                                             // SpMMs on small problems: config 2 0.125 vs 0.087 ms per apply at b = 32)
    int64_t sp8_apply_launches = 0, sp8_apply_t_launches = 0, x_fallbacks = 0;
    int64_t sp8_splits = 0;   // 128-row blocks halved because their dictionary exceeded one image
    int64_t gram8_launches = 0;   // steps that took it (stat)
    int64_t s8_bytes = 0;
    // D_ll
    float* D = nullptr;
    int64_t ldD = 0;
    bool own_D = false;
    DevBuf Dbuf;
    CUtensorMap dmap[7];
    bool dmap_ok[7] = {false, false, false, false, false, false, false};
    CUtensorMap amap;            // D as the tcgen05 A operand: box 32 x 128, SWIZZLE_128B
    bool amap_ok = false;
    CUtensorMap bmap[7];         // Y1T = [Y_hi; Y_lo] as the B operand
    void* bmap_ptr[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    DevBuf Y1T;
    // symmetric-half stream (k_dstream_pair.cuh): D packed as upper-triangle 128 x 128 tiles,
    // and one schedule per tensor width bp in {8, 16, 32}
    DevBuf Dt, Y16T, Y1f, y16aux;
    bool dt_ok = false;
    // int8 symmetric-half stream (k_dstream_sym8.cuh): D as three digit planes per upper tile
    DevBuf Dt8, Y8T;
    bool dt8_ok = false;
    bool dmax8_ok = false;            // aux[2] = max |D| over the block upper triangle (formed in create, overlapping D's upload)
    cudaStream_t pack_st = nullptr;   // create's D pack (host D): runs past create's return
    cudaEvent_t pack_ev = nullptr;
    bool pack_pending = false;        // D-stream launches wait for pack_ev until it has completed
    // int8 stream precision check (dq_decide): binades between max |D| and the median |D| over
    // the block upper triangle; auto (dstream 0) keeps the int8 stream only when <= dq_max_range
    DevBuf dqhist;                    // 256 per-binade counters (k_absmax_upper)
    bool dq_hist_ok = false;
    int dq_state = 0;                 // 0 undecided, 1 int8 stream kept, -1 fell back to the fp32-grade stream
    int dq_range = -1;
    int dq_max_range = 6;
    // sparse-step precision check (ensure_sp8): binades between a 128-row block's max |S| and its
    // smallest nonzero row maximum; above sp8_max_range the fp32 sparse kernels are used
    int sp8_range = -1;
    int sp8_max_range = 7;
    int bmds_dropped = 0;             // last sbmds_bmds: null pivots of (JP)^T JP (rank deficiency of J P)
    int chol_retries = 0;
    // standalone apply: per-column check of Y1 before the int8 stream (its per-column quantum is
    // max |y_c| 2^-23): when max |y_c| > 2^dy_max_range rms(y_c) for some column, this apply
    // streams D on the fp32-grade kernel instead (y_fallback), counted in y_fallbacks
    int dy_max_range = 3;
    bool y_fallback = false;
    int64_t y_fallbacks = 0;
    DevBuf xstat;            // standalone apply: X's column max bits [0, 64) and sums of squares (64 doubles)
    DevBuf ychk;             // last eigs: Cholesky-QR factorisations that needed the shifted retry
    struct PairPlan {
        bool ok = false;
        int S = 0, NT = 0, P = 0, nslots = 0;
        int64_t ntiles = 0;
        DevBuf tiles, pbeg, sbase, xptr, xslot, smap;
        CUtensorMap bmap16;
        void* b16_enc = nullptr;
    } pplan[3], s8plan[3];
    bool d_lower_missing = false;   // create uploaded only the block upper triangle of D
    int64_t h2d_bytes = 0;          // host -> device bytes moved by create (D)
    int pair_dbg = 0;
    DevBuf pdbg;
    double pdbg_avg[2][16] = {};
    int last_dpath = 0;          // D-stream path of the last apply: 1 ffma, 2 tcgen05, 3 tcgen05 symmetric half
    int64_t last_dbytes = 0;     // its bytes per launch (bench roofline)
    // apply workspace
    DevBuf Y1, Y2, P, colpart, s, t, tpart, counters, vdpart;
    int64_t y1_rows = 0;
    // eigs workspace
    DevBuf X, Y, gpart, G, H, Rinv, Rinv2, status, rr, vtmp, ztmp, sign, apval, apidx, xhost, yhost, vsel;
    // options / stats
    int rr_period = 5;
    int center = 1;          // 0: sbmds_apply computes the uncentred S D S^T X
    bool raw_now = false;
    DevBuf w0, rawR;         // zeros(l); -2 I (b x b) folded into Y1 for the uncentred apply
    int use_graph = 0;   // CUDA-graph replay of eigs segments (measured: no gain)
    cudaStream_t gstream = nullptr;   // graph capture / replay stream (the caller's may be legacy 0)
    cudaEvent_t gev[2] = {nullptr, nullptr};
    int order_columns = 1;
    int dstream = 0;
    double rowsum_dev = 0.0;
    bool d_borrowed = false;
    Profiler prof;
};

namespace {

struct DevGuard {
    int prev = -1;
    explicit DevGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DevGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

int bp_index(int bp) {
    int i = 0;
    while ((1 << i) < bp) ++i;
    return i;  // 1->0, 2->1, ..., 64->6
}

template <int BP>
void encode_dmap(sbmds_ctx* h) {
    using C = DsCfg<BP>;
    const int i = bp_index(BP);
    if (h->dmap_ok[i]) return;
    EncodeFn enc = get_encode();
    if (!enc) throw CudaError{cudaErrorNotSupported, "cuTensorMapEncodeTiled entry point"};
    cuuint64_t dims[2] = {(cuuint64_t)h->l, (cuuint64_t)h->l};
    cuuint64_t strides[1] = {(cuuint64_t)(h->ldD * sizeof(float))};
    cuuint32_t box[2] = {(cuuint32_t)C::BOXW, (cuuint32_t)C::BK};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&h->dmap[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)h->D, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError{cudaErrorInvalidValue, "cuTensorMapEncodeTiled"};
    h->dmap_ok[i] = true;
}

// the w of the rank-one centring terms: zeros while an uncentred apply runs (center = 0)
const double* wvec(const sbmds_ctx* h) { return h->raw_now ? h->w0.as<double>() : h->w.as<double>(); }

constexpr size_t kBlkSmem = 96 * 1024;   // shared-memory budget of one staged dictionary

bool blocked_ok(const sbmds_ctx* h, int b, int bp, const void* X, const void* Y) {
    return h->blocked && b == bp && b >= 4 && (b % 4) == 0 &&
           (size_t)h->umax * bp * sizeof(float) <= kBlkSmem && ((reinterpret_cast<uintptr_t>(X) & 15) == 0) &&
           ((reinterpret_cast<uintptr_t>(Y) & 15) == 0);
}

// ---------------------------------------------------------------------------- A3 + A4
template <int BP>
void run_dstream(sbmds_ctx* h, int b, cudaStream_t st) {
    using C = DsCfg<BP>;
    encode_dmap<BP>(h);
    StreamK sk;
    sk.RT = (h->l + C::TM - 1) / C::TM;
    sk.KT = (h->l + C::BK - 1) / C::BK;
    sk.T = sk.RT * sk.KT;
    sk.grid = (int)std::min<int64_t>(h->num_sms, sk.T);
    const int maxseg = (int)((sk.grid + sk.RT - 1) / sk.RT) + 2;
    h->P.ensure((size_t)sk.RT * maxseg * C::TM * BP * sizeof(double));
    smem_attr(k_dstream_ffma<BP>, C::SMEM + 1024);
    profiled(h->prof, PK_DSTREAM, st, [&] {
        launch(k_dstream_ffma<BP>, dim3(sk.grid), dim3(C::THREADS), (size_t)C::SMEM + 1024, st,
               h->dmap[bp_index(BP)], h->l, (const float*)h->Y1.as<float>(), sk, maxseg, h->P.as<double>());
    });
    h->last_dpath = 1;
    h->last_dbytes = 4 * h->l * h->l + 12 * h->l * (int64_t)b;
    const int rows_per_blk = 256 / BP;
    const int grid = (int)std::min<int64_t>(kRedBlocks, (h->l + rows_per_blk - 1) / rows_per_blk);
    profiled(h->prof, PK_DREDUCE, st, [&] {
        launch(k_dreduce, dim3(grid), dim3(256), 0, st, h->l, BP, b, C::TM, sk, maxseg,
               (const double*)h->P.as<double>(), wvec(h), h->Y2.as<float>(),
               h->tpart.as<double>(), h->t.as<double>(), h->counters.as<unsigned int>() + CNT_DRED);
    });
}

void encode_tiled_dt(CUtensorMap* map, void* ptr, CUtensorMapDataType dt, uint64_t inner, uint64_t outer,
                     uint64_t pitch_bytes, uint32_t box0, uint32_t box1, CUtensorMapSwizzle sw) {
    EncodeFn enc = get_encode();
    if (!enc) throw CudaError{cudaErrorNotSupported, "cuTensorMapEncodeTiled entry point"};
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    cuuint64_t strides[1] = {(cuuint64_t)pitch_bytes};
    cuuint32_t box[2] = {box0, box1};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, dt, 2, ptr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError{cudaErrorInvalidValue, "cuTensorMapEncodeTiled"};
}
void encode_tiled(CUtensorMap* map, void* ptr, uint64_t inner, uint64_t outer, uint64_t pitch_bytes, uint32_t box0,
                  uint32_t box1, CUtensorMapSwizzle sw) {
    encode_tiled_dt(map, ptr, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, inner, outer, pitch_bytes, box0, box1, sw);
}

// A3 + A4 on the tensor cores (3xTF32, tcgen05): split Y1, stream D, reduce partials.
// Padded k length of Y1 / Y1T shared by the tensor paths (their cached B tensor maps
// encode it): a multiple of 384 = 3 swizzle atoms (k_dstream_tc) and of 128 (k_dstream_sym).
int64_t y1t_lpad(const sbmds_ctx* h) { return (h->l + 383) / 384 * 384; }

template <int BP>
void run_dstream_tc(sbmds_ctx* h, int b, cudaStream_t st, const double* Rinv) {
    using C = TcCfg<BP>;
    const int i = bp_index(BP);
    const int64_t lpad = y1t_lpad(h);
    if (!h->amap_ok) {
        encode_tiled(&h->amap, h->D, h->l, h->l, h->ldD * sizeof(float), 32, 128, CU_TENSOR_MAP_SWIZZLE_128B);
        h->amap_ok = true;
    }
    h->Y1T.ensure((size_t)2 * kMaxB * lpad * sizeof(float));
    if (h->bmap_ptr[i] != h->Y1T.p) {
        encode_tiled(&h->bmap[i], h->Y1T.p, lpad, C::NB, lpad * sizeof(float), 32, C::NB, CU_TENSOR_MAP_SWIZZLE_128B);
        h->bmap_ptr[i] = h->Y1T.p;
    }
    profiled(h->prof, PK_SPLIT, st, [&] {
        launch(k_split_y1, dim3((unsigned)std::min<int64_t>(8 * 148, (lpad + 255) / 256 * BP)), dim3(256), 0, st,
               lpad, b, BP, Rinv, (const float*)h->Y1.as<float>(), h->Y1T.as<float>());
    });
    StreamK sk;
    sk.RT = (h->l + C::TM - 1) / C::TM;
    sk.KT = (h->l + C::TK - 1) / C::TK;
    sk.T = sk.RT * sk.KT;
    sk.grid = (int)std::min<int64_t>(h->num_sms, sk.T);
    const int maxseg = (int)((sk.grid + sk.RT - 1) / sk.RT) + 2;
    h->P.ensure((size_t)sk.RT * maxseg * C::TM * BP * sizeof(double));
    smem_attr(k_dstream_tc<BP>, C::SMEM);
    profiled(h->prof, PK_DSTREAM, st, [&] {
        launch(k_dstream_tc<BP>, dim3(sk.grid), dim3(C::THREADS), (size_t)C::SMEM, st, h->amap, h->bmap[i], sk, maxseg,
               h->P.as<double>());
    });
    h->last_dpath = 2;
    h->last_dbytes = 4 * h->l * h->l + 12 * h->l * (int64_t)b;
    const int rows_per_blk = 256 / BP;
    const int grid = (int)std::min<int64_t>(kRedBlocks, (h->l + rows_per_blk - 1) / rows_per_blk);
    profiled(h->prof, PK_DREDUCE, st, [&] {
        launch(k_dreduce, dim3(grid), dim3(256), 0, st, h->l, BP, b, C::TM, sk, maxseg,
               (const double*)h->P.as<double>(), wvec(h), h->Y2.as<float>(),
               h->tpart.as<double>(), h->t.as<double>(), h->counters.as<unsigned int>() + CNT_DRED);
    });
}

// A3 + A4 streaming only the upper triangle of D (NEXT-1, k_dstream_pair.cuh).

// Host schedule of the pair kernel: the walk (blocks of S x S tiles, block rows bi, block
// columns bj >= bi, row-major inside a block), balanced contiguous ranges per CTA pair, the
// partial slots each role writes (simulating exactly the kernel's flush rule: a segment ends
// when the walk enters another block; its touched accumulators flush in index order), and
// per row tile X the list of its slots in slot order (the fixed reduction order).
// gN > 1 (k_dstream_sym8): the row ("N") accumulators live across gN consecutive blocks of a
// block row (their segments end when (bi, bj / gN) changes), the column ("T") ones per block.
// contiguous: physical slot = rank of (X, logical slot), so each row tile's partials are
// contiguous for k_dreduce_pair; the kernel maps logical -> physical through pl.smap.
struct PlanHost {
    int S = 0, SC = 0, NT = 0, P = 0;   // blocks of S x SC tiles
    int64_t T = 0;
    std::vector<uint32_t> tiles;
    std::vector<int64_t> pbeg;
    std::vector<int> sbase, slot_x, xptr, xslot, smap;
};

// The upper tiles in walk order (blocks of S x S tiles, block rows, row-major inside a block);
// a shard (rank of world) keeps the contiguous range [T r / W, T (r + 1) / W).
// (SC = 0: square blocks of S x S tiles; else S rows x SC columns, the int8 stream's 9 x 1)
PlanHost plan_host(int64_t l, int max_pairs, int S, int gN, bool contiguous, int rank = 0, int world = 1, int SC = 0) {
    PlanHost ph;
    if (SC <= 0) SC = S;
    const int NT = (int)((l + 127) / 128);
    if (NT > 65535) throw std::runtime_error("l too large for the symmetric-half stream");
    const int NBr = (NT + S - 1) / S, NBc = (NT + SC - 1) / SC;
    auto& tiles = ph.tiles;
    tiles.reserve((size_t)NT * (NT + 1) / 2);
    for (int bi = 0; bi < NBr; ++bi)
        for (int bj = (bi * S) / SC; bj < NBc; ++bj)   // block columns that reach the diagonal or lie right of it
            for (int r = 0; r < S; ++r)
                for (int c = 0; c < SC; ++c) {
                    const int I = bi * S + r, J = bj * SC + c;
                    if (I < NT && J < NT && J >= I) tiles.push_back(((uint32_t)I << 16) | (uint32_t)J);
                }
    if (world > 1) {
        const int64_t Tall = (int64_t)tiles.size();
        const int64_t t0 = Tall * rank / world, t1 = Tall * (rank + 1) / world;
        tiles.erase(tiles.begin() + t1, tiles.end());
        tiles.erase(tiles.begin(), tiles.begin() + t0);
    }
    const int64_t T = (int64_t)tiles.size();
    const int P = (int)std::max<int64_t>(1, std::min<int64_t>(max_pairs, T / 8));
    auto& pbeg = ph.pbeg;
    pbeg.resize(P + 1);
    for (int p = 0; p <= P; ++p) pbeg[p] = (int64_t)p * T / P;
    auto& sbase = ph.sbase;
    auto& slot_x = ph.slot_x;
    sbase.resize(2 * P);
    for (int p = 0; p < P; ++p)
        for (int role = 0; role < 2; ++role) {
            sbase[2 * p + role] = (int)slot_x.size();
            uint32_t mask = 0;
            int cbi = -1, cbj = -1, ckey = -1;
            auto emit = [&]() {
                for (int a = 0; a < (role ? SC : S); ++a)
                    if (mask & (1u << a)) slot_x.push_back(role ? cbj * SC + a : cbi * S + a);
                mask = 0;
            };
            for (int64_t t = pbeg[p]; t < pbeg[p + 1]; ++t) {
                const int I = (int)(tiles[t] >> 16), J = (int)(tiles[t] & 0xFFFFu);
                const int bi = I / S, bj = J / SC;
                const int key = role ? bj : bj / gN;
                if ((bi != cbi || key != ckey) && mask) emit();
                cbi = bi;
                cbj = bj;
                ckey = key;
                if (role == 1 && I == J) continue;
                mask |= 1u << (role ? J - bj * SC : I - bi * S);
            }
            emit();
        }
    const int nslots = (int)slot_x.size();
    auto& xptr = ph.xptr;
    auto& xslot = ph.xslot;
    xptr.assign(NT + 1, 0);
    xslot.resize(nslots);
    for (int q = 0; q < nslots; ++q) ++xptr[slot_x[q] + 1];
    for (int X = 0; X < NT; ++X) xptr[X + 1] += xptr[X];
    {
        std::vector<int> fill(xptr.begin(), xptr.end() - 1);
        for (int q = 0; q < nslots; ++q) xslot[fill[slot_x[q]]++] = q;   // ascending slot ids per X
    }
    if (contiguous) {   // smap[logical] = physical (X-major, then logical order); xslot = identity
        ph.smap.assign(std::max(1, nslots), 0);
        for (int pq = 0; pq < nslots; ++pq) ph.smap[xslot[pq]] = pq;
        for (int pq = 0; pq < nslots; ++pq) xslot[pq] = pq;
    }
    ph.S = S;
    ph.SC = SC;
    ph.NT = NT;
    ph.P = P;
    ph.T = T;
    return ph;
}

void build_pair_plan(sbmds_ctx* h, sbmds_ctx::PairPlan& pl, int max_pairs, int S, int gN = 1, bool contiguous = false,
                     const PlanHost* pre = nullptr, int SC = 0) {
    const PlanHost ph = pre ? *pre : plan_host(h->l, max_pairs, S, gN, contiguous, h->rank, h->world, SC);
    const int nslots = (int)ph.slot_x.size();
    if (contiguous) {
        pl.smap.ensure(ph.smap.size() * sizeof(int));
        CK(cudaMemcpy(pl.smap.p, ph.smap.data(), ph.smap.size() * sizeof(int), cudaMemcpyHostToDevice));
    }
    pl.tiles.ensure(ph.tiles.size() * sizeof(uint32_t));
    pl.pbeg.ensure(ph.pbeg.size() * sizeof(int64_t));
    pl.sbase.ensure(ph.sbase.size() * sizeof(int));
    pl.xptr.ensure(ph.xptr.size() * sizeof(int));
    pl.xslot.ensure(std::max<size_t>(1, ph.xslot.size()) * sizeof(int));
    CK(cudaMemcpy(pl.tiles.p, ph.tiles.data(), ph.tiles.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(pl.pbeg.p, ph.pbeg.data(), ph.pbeg.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(pl.sbase.p, ph.sbase.data(), ph.sbase.size() * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(pl.xptr.p, ph.xptr.data(), ph.xptr.size() * sizeof(int), cudaMemcpyHostToDevice));
    if (nslots) CK(cudaMemcpy(pl.xslot.p, ph.xslot.data(), ph.xslot.size() * sizeof(int), cudaMemcpyHostToDevice));
    pl.S = S;
    pl.NT = ph.NT;
    pl.P = ph.P;
    pl.ntiles = ph.T;
    pl.nslots = nslots;
    pl.ok = true;
}

}  // namespace

// Self-check of the symmetric-half schedule on the host (no GPU): replays the kernels'
// accumulate / flush rules tile by tile (end-of-segment lookahead as in k_dstream_sym8, gN > 1,
// and k_dstream_pair, gN = 1) against the plan plan_host emitted, and counts violations: every
// upper tile exactly once; every (tile, N) contribution in exactly one slot of row tile I and
// every (tile, T), I < J, in exactly one slot of row tile J; slot -> row tile as recorded; the
// reduction lists (or the contiguous slot map) consistent.
namespace {
int64_t plan_selfcheck(int64_t l, int32_t S, int32_t gN, int32_t max_ctas, int32_t contiguous, int rank, int world,
                       int32_t SC = 0) {
    if (l < 1 || S < 1 || S > 16 || SC < 0 || SC > 16 || gN < 1 || max_ctas < 1 || world < 1 || rank < 0 || rank >= world)
        return -1;
    if (SC == 0) SC = S;
    int64_t err = 0;
    PlanHost ph;
    try {
        ph = plan_host(l, max_ctas, S, gN, contiguous != 0, rank, world, SC);
    } catch (...) {
        return -2;
    }
    const int NT = ph.NT;
    const int64_t T = ph.T;
    const int64_t Tall = (int64_t)NT * (NT + 1) / 2;
    if (T != Tall * (rank + 1) / world - Tall * rank / world) ++err;
    std::vector<uint8_t> seen((size_t)NT * NT, 0);
    for (int64_t t = 0; t < T; ++t) {
        const int I = (int)(ph.tiles[t] >> 16), J = (int)(ph.tiles[t] & 0xFFFFu);
        if (I > J || J >= NT || seen[(size_t)I * NT + J]++) ++err;
    }
    if (ph.pbeg.front() != 0 || ph.pbeg.back() != T) ++err;
    for (size_t p = 0; p + 1 < ph.pbeg.size(); ++p)
        if (ph.pbeg[p] > ph.pbeg[p + 1]) ++err;
    const int nslots = (int)ph.slot_x.size();
    std::vector<int> used_n(T, 0), used_t(T, 0);
    std::vector<int> slot_seen(nslots, 0);
    for (int p = 0; p < ph.P; ++p) {
        std::vector<std::vector<int64_t>> accN(S), accT(SC);
        uint32_t maskN = 0, maskT = 0;
        int slotN = ph.sbase[2 * p], slotT = ph.sbase[2 * p + 1];
        auto flush = [&](uint32_t mask, std::vector<std::vector<int64_t>>& acc, int& slot, int role, int bi, int bj) {
            for (int a = 0; a < (role ? SC : S); ++a) {
                if (!(mask & (1u << a))) continue;
                const int X = role ? bj * SC + a : bi * S + a;
                if (slot < 0 || slot >= nslots || ph.slot_x[slot] != X) ++err;
                if (slot >= 0 && slot < nslots) ++slot_seen[slot];
                for (const int64_t t : acc[a]) {
                    const int I = (int)(ph.tiles[t] >> 16), J = (int)(ph.tiles[t] & 0xFFFFu);
                    if ((role ? J : I) != X) ++err;
                    ++(role ? used_t : used_n)[t];
                }
                acc[a].clear();
                ++slot;
            }
        };
        for (int64_t t = ph.pbeg[p]; t < ph.pbeg[p + 1]; ++t) {
            const int I = (int)(ph.tiles[t] >> 16), J = (int)(ph.tiles[t] & 0xFFFFu);
            const int bi = I / S, bj = J / SC;
            bool end_seg = (t + 1 == ph.pbeg[p + 1]), end_n = end_seg;
            if (!end_seg) {
                const int I2 = (int)(ph.tiles[t + 1] >> 16), J2 = (int)(ph.tiles[t + 1] & 0xFFFFu);
                end_seg = (I2 / S != bi) || (J2 / SC != bj);
                end_n = (I2 / S != bi) || ((J2 / SC) / gN != bj / gN);
            }
            const int aN = I - bi * S, aT = J - bj * SC;
            accN[aN].push_back(t);
            maskN |= 1u << aN;
            if (I != J) {
                accT[aT].push_back(t);
                maskT |= 1u << aT;
            }
            if (end_seg) {
                if (end_n) {
                    flush(maskN, accN, slotN, 0, bi, bj);
                    maskN = 0;
                }
                flush(maskT, accT, slotT, 1, bi, bj);
                maskT = 0;
            }
        }
        if (p + 1 < ph.P && (slotN != ph.sbase[2 * p + 1] || slotT != ph.sbase[2 * p + 2])) ++err;
    }
    for (int64_t t = 0; t < T; ++t) {
        const int I = (int)(ph.tiles[t] >> 16), J = (int)(ph.tiles[t] & 0xFFFFu);
        if (used_n[t] != 1) ++err;
        if (used_t[t] != (I < J ? 1 : 0)) ++err;
    }
    for (int q = 0; q < nslots; ++q)
        if (slot_seen[q] != 1) ++err;
    // reduction lists: row tile X owns exactly its slots
    for (int X = 0; X < NT; ++X)
        for (int q = ph.xptr[X]; q < ph.xptr[X + 1]; ++q) {
            const int logical = contiguous ? -1 : ph.xslot[q];
            if (!contiguous && ph.slot_x[logical] != X) ++err;
        }
    if (contiguous) {
        std::vector<int> inv(nslots, -1);
        for (int q = 0; q < nslots; ++q) {
            const int phys = ph.smap[q];
            if (phys < 0 || phys >= nslots || inv[phys] >= 0) { ++err; continue; }
            inv[phys] = q;
            const int X = ph.slot_x[q];
            if (phys < ph.xptr[X] || phys >= ph.xptr[X + 1]) ++err;
        }
    }
    return err;
}
}  // namespace

extern "C" int64_t sbmds_plan_selfcheck(int64_t l, int32_t S, int32_t gN, int32_t max_ctas, int32_t contiguous) {
    return plan_selfcheck(l, S, gN, max_ctas, contiguous, 0, 1);
}

extern "C" int64_t sbmds_plan_selfcheck_rect(int64_t l, int32_t SR, int32_t SC, int32_t gN, int32_t max_ctas,
                                             int32_t contiguous, int32_t rank, int32_t world) {
    if (SC < 1) return -1;
    return plan_selfcheck(l, SR, gN, max_ctas, contiguous, rank, world, SC);
}

extern "C" int64_t sbmds_shard_plan_selfcheck(int64_t l, int32_t S, int32_t gN, int32_t max_ctas, int32_t contiguous,
                                              int32_t rank, int32_t world) {
    return plan_selfcheck(l, S, gN, max_ctas, contiguous, rank, world);
}

extern "C" int64_t sbmds_shard_tiles(int64_t l, int32_t S, int32_t rank, int32_t world, uint32_t* tiles_out,
                                     int64_t capacity) {
    if (l < 1 || S < 1 || S > 16 || world < 1 || rank < 0 || rank >= world) return -1;
    PlanHost ph;
    try {
        ph = plan_host(l, 1, S, 1, false, rank, world);
    } catch (...) {
        return -2;
    }
    if (tiles_out)
        for (int64_t t = 0; t < std::min<int64_t>(capacity, ph.T); ++t) tiles_out[t] = ph.tiles[t];
    return ph.T;
}

namespace {

template <int BP>
void run_dstream_pair(sbmds_ctx* h, int b, cudaStream_t st, const double* Rinv) {
    using C = PairCfg<BP>;
    const int pi = BP == 8 ? 0 : (BP == 16 ? 1 : 2);
    auto& pl = h->pplan[pi];
    static int max_clusters[3] = {0, 0, 0};   // (occupancy: the same on every device of one arch)
    smem_attr(k_dstream_pair<BP>, C::SMEM);
    if (!max_clusters[pi]) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2 * (h->num_sms / 2));
        cfg.blockDim = dim3(C::THREADS);
        cfg.dynamicSmemBytes = C::SMEM;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nc = 0;
        CK(cudaOccupancyMaxActiveClusters(&nc, k_dstream_pair<BP>, &cfg));
        max_clusters[pi] = std::max(1, std::min(nc, h->num_sms / 2));
    }
    const int64_t lpad = y1t_lpad(h);
    if (!pl.ok) build_pair_plan(h, pl, max_clusters[pi], C::S);
    // aux: [0] max |D| bits, [1] D exponent, [64..128) per-column max |Y1| bits, [128..192)
    // column exponents; [2] max |D| of the int8 packing, [3] its exponent
    h->y16aux.ensure(352 * sizeof(unsigned int));   // + [192, 320): Y2 column max / min keys, [320, 336) exponents
    unsigned int* dmax = h->y16aux.as<unsigned int>();
    int* dexp = reinterpret_cast<int*>(dmax + 1);
    unsigned int* ymax = dmax + 64;
    int* yexp = reinterpret_cast<int*>(dmax + 128);
    if (!h->dt_ok) {
        h->Dt.ensure((size_t)pl.ntiles * 128 * 128 * 2 * sizeof(__half));
        CK(cudaMemsetAsync(dmax, 0, sizeof(unsigned int), st));
        launch(k_absmax_upper, dim3((unsigned)std::min<int64_t>(8 * (int64_t)h->num_sms, h->l)), dim3(256),
               0, st, (const float*)h->D, h->l, h->ldD, dmax, (int64_t)0, (int64_t)-1, (unsigned int*)nullptr);
        launch(k_pack_upper, dim3((unsigned)std::min<int64_t>(pl.ntiles, 16 * (int64_t)h->num_sms)), dim3(256), 0, st,
               (const float*)h->D, h->ldD, h->l, (const uint32_t*)pl.tiles.p, (int64_t)pl.NT, pl.ntiles,
               (const unsigned int*)dmax, dexp, h->Dt.as<__half>());
        h->dt_ok = true;
    }
    h->Y16T.ensure((size_t)2 * kMaxB * lpad * sizeof(__half));
    h->Y1f.ensure((size_t)lpad * kMaxB * sizeof(float));
    if (pl.b16_enc != h->Y16T.p) {
        encode_tiled_dt(&pl.bmap16, h->Y16T.p, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, lpad, C::NB, lpad * sizeof(__half), 64,
                        C::NB, CU_TENSOR_MAP_SWIZZLE_128B);
        pl.b16_enc = h->Y16T.p;
    }
    profiled(h->prof, PK_SPLIT, st, [&] {
        CK(cudaMemsetAsync(ymax, 0, 64 * sizeof(unsigned int), st));
        launch(k_y16_prep, dim3((unsigned)std::min<int64_t>(4 * 148, (lpad * BP + 255) / 256)), dim3(256), 0, st,
               lpad, b, BP, Rinv, (const float*)h->Y1.as<float>(), h->Y1f.as<float>(), ymax, dmax + 192);
        launch(k_y16_split, dim3((unsigned)std::min<int64_t>(4 * 148, (lpad * BP + 255) / 256)), dim3(256), 0, st,
               lpad, BP, (const float*)h->Y1f.as<float>(), (const unsigned int*)ymax, h->Y16T.as<__half>(), yexp);
    });
    h->P.ensure((size_t)std::max(1, pl.nslots) * 128 * BP * sizeof(float));
    if (h->pair_dbg) {
        h->pdbg.ensure((size_t)2 * pl.P * 16 * sizeof(unsigned long long));
        CK(cudaMemsetAsync(h->pdbg.p, 0, (size_t)2 * pl.P * 16 * sizeof(unsigned long long), st));
    }
    profiled(h->prof, PK_DSTREAM, st, [&] {
        launch(k_dstream_pair<BP>, dim3(2 * pl.P), dim3(C::THREADS), (size_t)C::SMEM, st, (const __half*)h->Dt.p,
               pl.bmap16, (const uint32_t*)pl.tiles.p, (const int64_t*)pl.pbeg.p, (const int*)pl.sbase.p,
               (int)pl.NT, h->P.as<float>(), h->pair_dbg ? h->pdbg.as<unsigned long long>() : nullptr,
               h->pair_dbg >> 1);
    });
    if (h->pair_dbg) {   // per-role average wait cycles (sites: see k_dstream_pair)
        std::vector<unsigned long long> d((size_t)2 * pl.P * 16);
        CK(cudaStreamSynchronize(st));
        CK(cudaMemcpy(d.data(), h->pdbg.p, d.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 16; ++k) {
                double acc = 0;
                for (int p = 0; p < pl.P; ++p) acc += (double)d[(size_t)(2 * p + r) * 16 + k];
                h->pdbg_avg[r][k] = acc / pl.P;
            }
    }
    const int rows_per_blk = 256 / BP;
    const int grid = (int)std::min<int64_t>(4 * kRedBlocks, (h->l + rows_per_blk - 1) / rows_per_blk);
    h->tpart.ensure((size_t)4 * kRedBlocks * kMaxB * sizeof(double));
    profiled(h->prof, PK_DREDUCE, st, [&] {
        launch(k_dreduce_pair, dim3(grid), dim3(256), 0, st, h->l, BP, b, (const int*)pl.xptr.p,
               (const int*)pl.xslot.p, (const float*)h->P.as<float>(), (const int*)dexp,
               (const int*)yexp, wvec(h), h->Y2.as<float>(), h->tpart.as<double>(),
               h->t.as<double>(), h->counters.as<unsigned int>() + CNT_DRED, dmax + 192);
    });
    h->last_dpath = 4;
    h->last_dbytes = pl.ntiles * (int64_t)128 * 128 * 4 + 12 * h->l * (int64_t)b;
}

// A3 + A4 on the int8 tensor cores over the symmetric half of D (k_dstream_sym8.cuh).
template <int BP>
void run_dstream_sym8(sbmds_ctx* h, int b, cudaStream_t st, const double* Rinv) {
    using C = Sym8Cfg<BP>;
    const int pi = BP == 8 ? 0 : (BP == 16 ? 1 : 2);
    auto& pl = h->s8plan[pi];
    smem_attr(k_dstream_sym8<BP>, C::SMEM);
    const int64_t lpad = y1t_lpad(h);
    if (h->pack_pending) {   // create's D pack, possibly still running on its own stream
        CK(cudaStreamWaitEvent(st, h->pack_ev, 0));
        const cudaError_t q = cudaEventQuery(h->pack_ev);   // only a completed pack ends the waits
        if (q == cudaSuccess) h->pack_pending = false;
        else if (q != cudaErrorNotReady) throw CudaError{q, "D pack (issued by sbmds_create)"};
    }
    static const bool trace = getenv("SBMDS_TRACE_EIGS") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    auto dphase = [&](const char* what) {
        if (!trace) return;
        cudaStreamSynchronize(st);
        fprintf(stderr, "[sbmds_dstream]  %8.2f ms  %s\n",
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(), what);
    };
    if (!pl.ok) { build_pair_plan(h, pl, h->num_sms, C::SR, C::GN, true, nullptr, C::SC); dphase("pair plan"); }   // one CTA per SM, both roles
    h->y16aux.ensure(352 * sizeof(unsigned int));   // + [192, 320): Y2 column max / min keys, [320, 336) exponents
    unsigned int* aux = h->y16aux.as<unsigned int>();
    unsigned int* dmax8 = aux + 2;
    int* dexp8 = reinterpret_cast<int*>(aux + 3);
    unsigned int* ymax = aux + 64;
    int* yexp = reinterpret_cast<int*>(aux + 128);
    if (!h->dt8_ok) {
        h->Dt8.ensure((size_t)((int64_t)pl.NT * (pl.NT + 1) / 2) * C::A_BYTES);   // (normally allocated in create; indexed by upper_tile_index, also on a shard)
        dphase("Dt8 allocated");
        if (!h->dmax8_ok) {
            CK(cudaMemsetAsync(dmax8, 0, sizeof(unsigned int), st));
            launch(k_absmax_upper, dim3((unsigned)std::min<int64_t>(8 * (int64_t)h->num_sms, h->l)), dim3(256), 0, st,
                   (const float*)h->D, h->l, h->ldD, dmax8, (int64_t)0, (int64_t)-1, (unsigned int*)nullptr);
            h->dmax8_ok = true;
        }
        dphase("absmax");
        launch(k_pack_sym8, dim3((unsigned)std::min<int64_t>(pl.ntiles, 16 * (int64_t)h->num_sms)), dim3(256), 0, st,
               (const float*)h->D, h->ldD, h->l, (const uint32_t*)pl.tiles.p, (int64_t)pl.NT, pl.ntiles,
               (const unsigned int*)dmax8, dexp8, h->Dt8.as<int8_t>());
        h->dt8_ok = true;
        dphase("pack");
    }
    h->Y8T.ensure((size_t)3 * kMaxB * lpad);
    h->Y1f.ensure((size_t)lpad * kMaxB * sizeof(float));
    if (pl.b16_enc != h->Y8T.p) {
        encode_tiled_dt(&pl.bmap16, h->Y8T.p, CU_TENSOR_MAP_DATA_TYPE_UINT8, lpad, C::NB, lpad, 128, C::NB,
                        CU_TENSOR_MAP_SWIZZLE_128B);
        pl.b16_enc = h->Y8T.p;
    }
    profiled(h->prof, PK_SPLIT, st, [&] {
        if (!h->y1f_ready) {   // (else k_blk_reduce_fold formed Y1f, its column max and the digits)
            CK(cudaMemsetAsync(ymax, 0, 64 * sizeof(unsigned int), st));
            launch(k_y16_prep, dim3((unsigned)std::min<int64_t>(4 * 148, (lpad * BP + 255) / 256)), dim3(256), 0, st,
                   lpad, b, BP, Rinv, (const float*)h->Y1.as<float>(), h->Y1f.as<float>(), ymax, aux + 192);
            launch_pdl(k_y8_split, dim3((unsigned)std::min<int64_t>(4 * 148, (lpad * BP + 255) / 256)), dim3(256), 0, st,
                       lpad, BP, (const float*)h->Y1f.as<float>(), (const unsigned int*)ymax, h->Y8T.as<int8_t>(), yexp);
        }
        h->y1f_ready = false;
    });
    h->P.ensure((size_t)std::max(1, pl.nslots) * 128 * BP * sizeof(float));
    profiled(h->prof, PK_DSTREAM, st, [&] {
        launch_pdl(k_dstream_sym8<BP>, dim3(pl.P), dim3(C::THREADS), (size_t)C::SMEM, st, (const int8_t*)h->Dt8.p,
               pl.bmap16, (const uint32_t*)pl.tiles.p, (const int64_t*)pl.pbeg.p, (const int*)pl.sbase.p,
               (const int*)pl.smap.p, (int)pl.NT, h->P.as<float>(), h->pair_dbg >> 1);
    });
    const int rows_per_blk = 256 / BP;
    const int grid = (int)std::min<int64_t>(4 * kRedBlocks, (h->l + rows_per_blk - 1) / rows_per_blk);
    h->tpart.ensure((size_t)4 * kRedBlocks * kMaxB * sizeof(double));
    profiled(h->prof, PK_DREDUCE, st, [&] {
        if (BP == 16 && h->y2d_want) {
            // one cooperative launch: reduce, grid sync on t and the Y2 keys, Y2's digit planes
            static int per_sm = 0;
            if (!per_sm) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dreduce_y2d<16>, 256, 0));
            const int cg = (int)std::min<int64_t>(grid, std::max(1, per_sm) * (int64_t)h->num_sms);
            h->s8yd.ensure((size_t)3 * h->l * 16);
            launch_coop_pdl(k_dreduce_y2d<16>, dim3(cg), dim3(256), 0, st, h->l, b, (const int*)pl.xptr.p,
                        (const float*)h->P.as<float>(), (const int*)dexp8, (const int*)yexp, wvec(h),
                        h->Y2.as<float>(), h->tpart.as<double>(), h->t.as<double>(),
                        h->counters.as<unsigned int>() + CNT_DRED, aux + 192, reinterpret_cast<int*>(aux + 320),
                        h->s8yd.as<uint8_t>(), aux + 64);
            h->y2d_ready = true;
        } else {
            launch_pdl(k_dreduce_pair, dim3(grid), dim3(256), 0, st, h->l, BP, b, (const int*)pl.xptr.p,
                       (const int*)nullptr, (const float*)h->P.as<float>(), (const int*)dexp8, (const int*)yexp,
                       wvec(h), h->Y2.as<float>(), h->tpart.as<double>(), h->t.as<double>(),
                       h->counters.as<unsigned int>() + CNT_DRED, aux + 192);
        }
    });
    h->last_dpath = 3;
    h->last_dbytes = pl.ntiles * (int64_t)C::A_BYTES + 12 * h->l * (int64_t)b;
}

bool uses_tc(const sbmds_ctx* h, int bp) { return bp >= 8 && (h->dstream == 2 || h->dstream == 0 || h->dstream == 3); }
// symmetric-half stream: forced by dstream = 3, chosen by auto (0) once D has >= 8 tiles per
// CTA pair (below that D is L2-resident and the full stream on all SMs wins)
bool sym_size_ok(const sbmds_ctx* h) {
    const int64_t nt = (h->l + 127) / 128;
    return nt * (nt + 1) / 2 >= 8 * (int64_t)(h->num_sms / 2);
}
bool uses_sym(const sbmds_ctx* h, int bp) {
    if (!(bp == 8 || bp == 16 || bp == 32)) return false;
    if (h->dstream == 3 || h->dstream == 4) return true;
    return h->dstream == 0 && sym_size_ok(h) && h->dq_state >= 0 && !h->y_fallback;   // (auto: the precision checks)
}

// Precision check of the int8 stream's fixed point (DESIGN.md §4 "precision contract"). The
// stream stores D as integers on one global quantum q = 2^-sD, max|D| 2^-22 < q <= max|D| 2^-21,
// so an entry |D_ij| keeps a relative precision of q / (2|D_ij|). The check takes the median
// |D| over the block upper triangle from the per-binade histogram (k_absmax_upper) and keeps
// the int8 stream only while the median entry lies within dq_max_range binades (default 6) of
// max |D|: the median entry then keeps >= 15 significant bits (relative rounding <= 2^-16 of
// it, mean zero). Squared geodesics sit 1-3 binades below their max (configs 1-4: 2), uniform
// config-5 D 1. A D with a few far outliers or clusters far apart (max / median >= 2^7) would
// leave most entries with few bits; auto then streams the full D on the fp32-grade 3xTF32
// kernel instead. Reads the histogram and max back (stream sync).
void dq_decide(sbmds_ctx* h, cudaStream_t st) {
    unsigned int hist[256], mbits = 0;
    peek_to_host(hist, h->dqhist.p, sizeof hist, st);
    peek_to_host(&mbits, h->y16aux.as<unsigned int>() + 2, sizeof mbits, st);
    uint64_t total = 0;
    for (int e = 0; e < 256; ++e) total += hist[e];
    int range = 0;
    if (total > 0 && mbits != 0) {
        uint64_t acc = 0;
        int emed = 0;
        for (int e = 0; e < 256; ++e) {
            acc += hist[e];
            if (2 * acc >= total) { emed = e; break; }
        }
        range = (int)(mbits >> 23) - emed;   // (a zero / subnormal median: emed = 0, a huge range)
    }
    h->dq_range = range;
    h->dq_state = range <= h->dq_max_range ? 1 : -1;
}

// Decide the precision check before the first apply / eigs of an auto handle that would take
// the int8 stream (create already did it for a host D large enough for that stream).
void ensure_dq(sbmds_ctx* h, cudaStream_t st) {
    if (h->dq_state != 0 || h->dstream != 0 || !sym_size_ok(h)) return;
    h->y16aux.ensure(352 * sizeof(unsigned int));
    if (!h->dq_hist_ok) {
        h->dqhist.ensure(256 * sizeof(unsigned int));
        unsigned int* aux = h->y16aux.as<unsigned int>();
        // max |D| into aux[2] unless create (or a pack) already formed it; else a scratch word
        unsigned int* mx = h->dmax8_ok ? aux + 4 : aux + 2;
        CK(cudaMemsetAsync(mx, 0, sizeof(unsigned int), st));
        CK(cudaMemsetAsync(h->dqhist.p, 0, 256 * sizeof(unsigned int), st));
        launch(k_absmax_upper, dim3((unsigned)std::min<int64_t>(8 * (int64_t)h->num_sms, h->l)), dim3(256), 0, st,
               (const float*)h->D, h->l, h->ldD, mx, (int64_t)0, (int64_t)-1, h->dqhist.as<unsigned int>());
        h->dmax8_ok = true;
        h->dq_hist_ok = true;
    }
    dq_decide(h, st);
    if (h->dq_state < 0 && h->dt8_ok) {   // (cannot happen after create's check; kept for safety)
        if (h->pack_st) CK(cudaStreamSynchronize(h->pack_st));
        h->pack_pending = false;
        h->Dt8.release();
        h->dt8_ok = false;
    }
}

// Mirror the lower triangle of D on the device before the first full-D kernel (see create).
void ensure_full_d(sbmds_ctx* h, cudaStream_t st) {
    if (!h->d_lower_missing) return;
    const unsigned t = (unsigned)((h->l + 31) / 32);
    launch(k_mirror_lower, dim3(t, t), dim3(256), 0, st, h->D, h->l, h->ldD);
    h->d_lower_missing = false;
}

// whether dstream() takes a symmetric-half stream (tile-partitioned on a shard) at width bp
// (b = 64 only without an R^-1 fold: the fold couples the two column halves)
bool takes_sym(const sbmds_ctx* h, int bp, bool fold) {
    if (bp < 8) return h->dstream == 0 && uses_sym(h, 8);
    if (bp == 64) return !fold && h->dstream == 0 && uses_sym(h, 32);
    return uses_sym(h, bp);
}

void dstream(sbmds_ctx* h, int b, int bp, cudaStream_t st, const double* Rinv) {
    if (bp < 8 && h->dstream == 0 && uses_sym(h, 8)) {
        // b <= 4 (round 2): the symmetric int8 stream at width 8 reads 3 l^2 / 2 bytes where the
        // FFMA stream reads 4 l^2 (config 5, l = 20k: 0.61 vs 1.6 GB). Y1 is widened to pitch 8
        // (zero columns) around it and Y2 narrowed back to pitch bp for the CSR SpMM.
        const int64_t lpad = y1t_lpad(h);
        h->Y1w.ensure((size_t)lpad * kMaxB * sizeof(float));
        h->Y2w.ensure((size_t)h->l * kMaxB * sizeof(float));
        CK(cudaMemsetAsync(h->Y1w.p, 0, (size_t)lpad * 8 * sizeof(float), st));
        CK(cudaMemcpy2DAsync(h->Y1w.p, 8 * sizeof(float), h->Y1.p, bp * sizeof(float), b * sizeof(float), h->l,
                             cudaMemcpyDeviceToDevice, st));
        h->Y1.swap(h->Y1w);
        h->Y2.swap(h->Y2w);
        struct Back {
            sbmds_ctx* h;
            ~Back() { h->Y1.swap(h->Y1w); h->Y2.swap(h->Y2w); }
        } back{h};
        run_dstream_sym8<8>(h, b, st, Rinv);
        CK(cudaMemcpy2DAsync(h->Y2w.p, bp * sizeof(float), h->Y2.p, 8 * sizeof(float), b * sizeof(float), h->l,
                             cudaMemcpyDeviceToDevice, st));   // (Y2w is the caller's Y2 until the swap back)
        return;
    }
    if (bp == 64 && !Rinv && h->dstream == 0 && uses_sym(h, 32)) {
        // b in 33..64 without a fold (round 2): two passes of the width-32 int8 stream over the
        // column halves, 2 x 3 l^2 / 2 bytes instead of the 3xTF32 stream's 4 l^2 (config 5:
        // 1.2 vs 1.6 GB); Y1's halves at pitch 32, Y2's halves and t merged back
        const int64_t lpad = y1t_lpad(h);
        h->Y1w.ensure((size_t)lpad * kMaxB * sizeof(float));
        h->Y2w.ensure((size_t)h->l * kMaxB * sizeof(float));
        h->tsave.ensure(kMaxB * sizeof(double));
        int64_t bytes2 = 0;
        for (int half = 0; half < 2; ++half) {
            const int c0 = 32 * half, bh = std::min(32, b - c0);
            CK(cudaMemsetAsync(h->Y1w.p, 0, (size_t)lpad * 32 * sizeof(float), st));
            CK(cudaMemcpy2DAsync(h->Y1w.p, 32 * sizeof(float), h->Y1.as<float>() + c0, 64 * sizeof(float),
                                 bh * sizeof(float), h->l, cudaMemcpyDeviceToDevice, st));
            h->Y1.swap(h->Y1w);
            h->Y2.swap(h->Y2w);
            struct Back {
                sbmds_ctx* h;
                ~Back() { h->Y1.swap(h->Y1w); h->Y2.swap(h->Y2w); }
            } back{h};
            run_dstream_sym8<32>(h, bh, st, nullptr);
            bytes2 += h->last_dbytes;
            CK(cudaMemcpy2DAsync(h->Y2w.as<float>() + c0, 64 * sizeof(float), h->Y2.p, 32 * sizeof(float),
                                 bh * sizeof(float), h->l, cudaMemcpyDeviceToDevice, st));
            CK(cudaMemcpyAsync(h->tsave.as<double>() + c0, h->t.p, bh * sizeof(double), cudaMemcpyDeviceToDevice, st));
        }
        CK(cudaMemcpyAsync(h->t.p, h->tsave.p, b * sizeof(double), cudaMemcpyDeviceToDevice, st));
        h->last_dbytes = bytes2 / 2;   // (per launch, as the profile counts launches)
        return;
    }
    if (uses_sym(h, bp)) {
        if (h->dstream == 4) {   // 2xFP16 on CTA pairs (k_dstream_pair), kept for comparison
            if (bp == 8) run_dstream_pair<8>(h, b, st, Rinv);
            else if (bp == 16) run_dstream_pair<16>(h, b, st, Rinv);
            else run_dstream_pair<32>(h, b, st, Rinv);
        } else {
            if (bp == 8) run_dstream_sym8<8>(h, b, st, Rinv);
            else if (bp == 16) run_dstream_sym8<16>(h, b, st, Rinv);
            else run_dstream_sym8<32>(h, b, st, Rinv);
        }
        return;
    }
    ensure_full_d(h, st);
    if (uses_tc(h, bp)) {
        switch (bp) {
            case 8: run_dstream_tc<8>(h, b, st, Rinv); return;
            case 16: run_dstream_tc<16>(h, b, st, Rinv); return;
            case 32: run_dstream_tc<32>(h, b, st, Rinv); return;
            default: run_dstream_tc<64>(h, b, st, Rinv); return;
        }
    }
    // widths < 8 (or dstream=1): FFMA stream; the R^-1 fold runs as its own small kernel
    if (Rinv)
        profiled(h->prof, PK_ROTATE, st, [&] {
            launch(k_y1_rot, dim3((unsigned)std::min<int64_t>(8 * 148, (h->l * bp + 255) / 256)), dim3(256), 0, st,
                   h->l, b, bp, Rinv, h->Y1.as<float>());
        });
    switch (bp) {
        case 1: run_dstream<1>(h, b, st); break;
        case 2: run_dstream<2>(h, b, st); break;
        case 4: run_dstream<4>(h, b, st); break;
        case 8: run_dstream<8>(h, b, st); break;
        case 16: run_dstream<16>(h, b, st); break;
        case 32: run_dstream<32>(h, b, st); break;
        default: run_dstream<64>(h, b, st); break;
    }
}

// ---------------------------------------------------------------------------- A2 / A5 dispatch
void spmm_csc(sbmds_ctx* h, int b, int bp, const float* X, cudaStream_t st) {
    const int grid = (int)((h->l + 7) / 8);
    const int32_t* ord = h->order_columns ? h->order.as<int32_t>() : nullptr;
    const bool vec = (b == bp) && (b % 4 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
    auto args = std::make_tuple(h->l, b, bp, (const int32_t*)h->cptr.as<int32_t>(),
                                (const int32_t*)h->ridx.as<int32_t>(), (const float*)h->cval.as<float>(), ord, X,
                                wvec(h), (const double*)h->s.as<double>(),
                                h->Y1.as<float>());
    auto go = [&](auto kern) {
        std::apply([&](auto... a) { launch(kern, dim3(grid), dim3(256), 0, st, a...); }, args);
    };
    if (vec) {
        switch (b / 4) {
            case 1: go(k_spmm_csc_vec4<1>); break;
            case 2: go(k_spmm_csc_vec4<2>); break;
            case 4: go(k_spmm_csc_vec4<4>); break;
            case 8: go(k_spmm_csc_vec4<8>); break;
            default: go(k_spmm_csc_vec4<16>); break;
        }
    } else {
        switch (bp) {
            case 1: go(k_spmm_csc_gen<1, 1>); break;
            case 2: go(k_spmm_csc_gen<2, 1>); break;
            case 4: go(k_spmm_csc_gen<4, 1>); break;
            case 8: go(k_spmm_csc_gen<8, 1>); break;
            case 16: go(k_spmm_csc_gen<16, 1>); break;
            case 32: go(k_spmm_csc_gen<32, 1>); break;
            default: go(k_spmm_csc_gen<32, 2>); break;
        }
    }
}

void spmm_csr(sbmds_ctx* h, int b, int bp, float* Y, cudaStream_t st) {
    if (bp <= 4) {   // narrow: L lanes per row over its nonzeros (k_spmm_csr_sub)
        const double avg = (double)h->nnz / (double)std::max<int64_t>(1, h->n);
        int L = 1;   // ~4 nonzeros per lane, at most 8 lanes per row (measured on the config-5 sweep)
        while (L < 8 && L * h->csr_nnz_per_lane < avg) L *= 2;
        if (h->csr_sub_L) L = h->csr_sub_L;
        const int64_t warps = (h->n + (32 / L) - 1) / (32 / L);
        const int grid = (int)((warps + 7) / 8);
        auto go = [&](auto kern) {
            launch(kern, dim3(grid), dim3(256), 0, st, h->n, b, bp, (const int32_t*)h->rp.as<int32_t>(),
                   (const int32_t*)h->col.as<int32_t>(), (const float*)h->val.as<float>(),
                   (const float*)h->Y2.as<float>(), (const double*)h->t.as<double>(), Y);
        };
        auto by_bw = [&](auto l4, auto l2, auto l1) { bp == 4 ? go(l4) : (bp == 2 ? go(l2) : go(l1)); };
        switch (L) {
            case 32: by_bw(k_spmm_csr_sub<32, 4>, k_spmm_csr_sub<32, 2>, k_spmm_csr_sub<32, 1>); break;
            case 16: by_bw(k_spmm_csr_sub<16, 4>, k_spmm_csr_sub<16, 2>, k_spmm_csr_sub<16, 1>); break;
            case 8: by_bw(k_spmm_csr_sub<8, 4>, k_spmm_csr_sub<8, 2>, k_spmm_csr_sub<8, 1>); break;
            case 4: by_bw(k_spmm_csr_sub<4, 4>, k_spmm_csr_sub<4, 2>, k_spmm_csr_sub<4, 1>); break;
            case 2: by_bw(k_spmm_csr_sub<2, 4>, k_spmm_csr_sub<2, 2>, k_spmm_csr_sub<2, 1>); break;
            default: by_bw(k_spmm_csr_sub<1, 4>, k_spmm_csr_sub<1, 2>, k_spmm_csr_sub<1, 1>); break;
        }
        return;
    }
    const bool vec = (b == bp) && (b % 4 == 0) && ((reinterpret_cast<uintptr_t>(Y) & 15) == 0);
    const int lpr = vec ? b / 4 : std::min(bp, 32);
    const int G = 32 / lpr;
    const int64_t warps = (h->n + G - 1) / G;
    const int grid = (int)((warps + 7) / 8);
    auto args = std::make_tuple(h->n, b, bp, (const int32_t*)h->rp.as<int32_t>(), (const int32_t*)h->col.as<int32_t>(),
                                (const float*)h->val.as<float>(), (const float*)h->Y2.as<float>(),
                                (const double*)h->t.as<double>(), Y);
    auto go = [&](auto kern) {
        std::apply([&](auto... a) { launch(kern, dim3(grid), dim3(256), 0, st, a...); }, args);
    };
    if (vec) {
        // pairs loaded once per group and broadcast by shuffles (option csr_shfl: -1 auto, 0, 1). Auto:
        // b <= 16, or rows long enough to fill a group's four chunks (>= 4 * lanes per row entries on
        // average): measured on the config-5 sweep (scripts/csr_shfl_sweep.py) 1.1-1.7x faster there,
        // 1.1-1.5x slower for short rows at b >= 32 (most of a chunk's shuffles are padding).
        const double avg = (double)h->nnz / (double)std::max<int64_t>(1, h->n);
        const bool shf = h->csr_shfl < 0 ? (lpr <= 4 || avg >= 4.0 * lpr) : h->csr_shfl != 0;
        switch (b / 4) {
            case 1: shf ? go(k_spmm_csr_vec4<1, true>) : go(k_spmm_csr_vec4<1, false>); break;
            case 2: shf ? go(k_spmm_csr_vec4<2, true>) : go(k_spmm_csr_vec4<2, false>); break;
            case 4: shf ? go(k_spmm_csr_vec4<4, true>) : go(k_spmm_csr_vec4<4, false>); break;
            case 8: shf ? go(k_spmm_csr_vec4<8, true>) : go(k_spmm_csr_vec4<8, false>); break;
            default: shf ? go(k_spmm_csr_vec4<16, true>) : go(k_spmm_csr_vec4<16, false>); break;
        }
    } else {
        switch (bp) {
            case 1: go(k_spmm_csr_gen<1, 1>); break;
            case 2: go(k_spmm_csr_gen<2, 1>); break;
            case 4: go(k_spmm_csr_gen<4, 1>); break;
            case 8: go(k_spmm_csr_gen<8, 1>); break;
            case 16: go(k_spmm_csr_gen<16, 1>); break;
            case 32: go(k_spmm_csr_gen<32, 1>); break;
            default: go(k_spmm_csr_gen<32, 2>); break;
        }
    }
}

void ensure_apply_ws(sbmds_ctx* h, int bp) {
    const int64_t rows = (h->l + 383) / 384 * 384;   // >= every D-stream path's padded k range
    if (h->Y1.bytes < (size_t)rows * bp * sizeof(float)) {
        h->Y1.ensure((size_t)rows * kMaxB * sizeof(float));
        CK(cudaMemset(h->Y1.p, 0, h->Y1.bytes));  // pad rows/cols stay 0 (TMA tail reads them)
    }
    h->Y2.ensure((size_t)h->l * kMaxB * sizeof(float));
}

// Y1's per-column dynamic range against the int8 stream's per-column fixed point: the quantum
// of column c is ~max |y_c| 2^-23 and the dropped digit products add ~2^-22 max|D| max|y_c| per
// product, so a column whose max sits far above its rms (an X with a dominant row) keeps its
// bulk with few bits. Measured: max/rms = 17 gave 2.5e-5 relative error on the apply (bar 1e-5);
// Gaussian blocks sit at ~4. Above 2^dy_max_range this apply uses the fp32-grade stream.
// x_ok (optional): the standalone apply's X statistics (h->xstat, formed by colsum_xstat before
// its tensor-core A2) ride in the same readback; *x_ok = false when a column of X fails the same
// bound (dominant row). want_y = false reads only them.
void ycheck(sbmds_ctx* h, int b, int bp, cudaStream_t st, bool want_y = true, bool* x_ok = nullptr) {
    constexpr size_t kStat = 64 * sizeof(unsigned int) + 64 * sizeof(double);
    h->ychk.ensure(2 * kStat);   // [0, kStat): Y1's statistics; [kStat, 2 kStat): a copy of X's
    unsigned char buf[2 * kStat];
    if (want_y) {
        CK(cudaMemsetAsync(h->ychk.p, 0, kStat, st));
        launch(k_ycheck, dim3((unsigned)std::min<int64_t>(2 * (int64_t)h->num_sms, (h->l * bp + 255) / 256)), dim3(256), 0,
               st, h->l, b, bp, (const float*)h->Y1.as<float>(), h->ychk.as<unsigned int>());
    }
    if (x_ok) CK(cudaMemcpyAsync(h->ychk.as<unsigned char>() + kStat, h->xstat.p, kStat, cudaMemcpyDeviceToDevice, st));
    peek_to_host(buf, h->ychk.p, x_ok ? 2 * kStat : kStat, st);
    const double lim = std::ldexp(1.0, h->dy_max_range);
    auto bad = [&](const unsigned char* q, double count) {
        const unsigned int* mx = reinterpret_cast<const unsigned int*>(q);
        const double* ss = reinterpret_cast<const double*>(q + 256);
        for (int c = 0; c < b; ++c) {
            float m;
            memcpy(&m, &mx[c], 4);
            const double rms = std::sqrt(ss[c] / count);
            // (a NaN / Inf anywhere in the column shows in its sum of squares: the fp32-grade kernels
            // propagate it, the fixed point would turn it into garbage digits)
            if (!(m < 3.0e38f) || !std::isfinite(rms) || (m > 0.f && (double)m > lim * rms)) return true;
        }
        return false;
    };
    if (x_ok) *x_ok = !bad(buf + kStat, (double)h->n);
    if (want_y && bad(buf, (double)h->l)) {
        h->y_fallback = true;
        ++h->y_fallbacks;
    }
}

// A1: s = 1^T X (fp64, fixed order): float4 loads where b % 4 == 0 and X is 16-byte aligned
void colsum(sbmds_ctx* h, int b, const float* X, cudaStream_t st) {
    const unsigned grid = (unsigned)std::min<int64_t>(4 * kRedBlocks, (h->n + 255) / 256);
    if (b % 4 == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0)
        launch(k_colsum4<false>, dim3(grid), dim3(256), 0, st, h->n, b, X, h->colpart.as<double>(), h->s.as<double>(),
               h->counters.as<unsigned int>() + CNT_COLSUM, (unsigned int*)nullptr);
    else
        launch(k_colsum, dim3(grid), dim3(256), 0, st, h->n, b, X, h->colpart.as<double>(), h->s.as<double>(),
               h->counters.as<unsigned int>() + CNT_COLSUM);
}

// A1 with the per-column max |x| and sum of squares of X (b = 16 / 32, X 16-byte aligned) into
// h->xstat: the scales of the standalone apply's tensor-core A2 (X's 24-bit digits take one scale
// per column) and its check, read back together with Y1's after A2 (ycheck): a column whose max
// is > 2^dy_max_range times its rms (a dominant row) redoes A2 on the fp32 CSC SpMM (stat
// x_fallbacks).
void colsum_xstat(sbmds_ctx* h, int b, const float* X, cudaStream_t st) {
    h->xstat.ensure(64 * sizeof(unsigned int) + 64 * sizeof(double));
    CK(cudaMemsetAsync(h->xstat.p, 0, h->xstat.bytes, st));
    const unsigned grid = (unsigned)std::min<int64_t>(4 * kRedBlocks, (h->n + 255) / 256);
    launch(k_colsum4<true>, dim3(grid), dim3(256), 0, st, h->n, b, X, h->colpart.as<double>(), h->s.as<double>(),
           h->counters.as<unsigned int>() + CNT_COLSUM, h->xstat.as<unsigned int>());
}

// The standalone apply's A2 on the tensor cores: the T products of the sparse step on X's rows
// (k_sp8_step TONLY), partials per 128-row block slot; k_blk_reduce then sums them per landmark.
void launch_sp8_t(sbmds_ctx* h, int b, const float* X, cudaStream_t st) {
    using C = Sp8Cfg<16>;
    auto kern = k_sp8_step<16, false, false, true>;
    smem_attr(kern, C::SMEM);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(h->s8.nblk, h->num_sms));
    h->gpart.ensure((size_t)std::max(grid, kRedBlocks) * kGramPart * sizeof(double));
    h->P1.ensure((size_t)std::max<int32_t>(std::max(1, h->s8.total_u), h->total_u) * kMaxB * sizeof(float));
    h->s8yd.ensure((size_t)3 * h->l * 16);
    h->y16aux.ensure(352 * sizeof(unsigned int));
    for (int c0 = 0; c0 < b; c0 += 16)   // (b = 32: one pass per 16-column half of X)
        launch_pdl(kern, dim3(grid), dim3(C::THREADS), (size_t)C::SMEM, st, h->n, h->l, h->s8.nblk,
                   (const int8_t*)h->s8img.as<int8_t>(), (const int64_t*)h->s8ioff.as<int64_t>(),
                   (const int32_t*)h->s8.doff.as<int32_t>(), (const int32_t*)h->s8.dict.as<int32_t>(),
                   (const int*)h->s8esc.as<int>(), (const uint8_t*)h->s8yd.as<uint8_t>(),
                   (const int*)(h->y16aux.as<unsigned int>() + 320), (const double*)h->t.as<double>(),
                   (const float*)h->s8rs1.as<float>(), (const float*)h->xstat.as<float>() + c0,
                   (const int32_t*)h->s8pos.as<int32_t>(), (float*)nullptr, h->P1.as<float>() + c0, X + c0,
                   h->gpart.as<double>(), h->G.as<double>(), h->H.as<double>(), h->s.as<double>(),
                   h->counters.as<unsigned int>() + CNT_GRAM, (unsigned long long*)nullptr, 0, (double*)nullptr,
                   h->status.as<int>(), 1, b, b, (const int32_t*)h->s8.brow0.as<int32_t>());
}

// The whole operator apply on device buffers (stream-ordered; the standalone apply on the int8
// stream reads Y1's column check back once, see ycheck).
// Fused-step flags (eigs only, row-blocked S, b in {4, 8, 16, 32}):
//   kApplyY1Ready: A2 comes from the S^T partials P1 the previous fused step wrote (k_blk_reduce)
//   kApplyFused:   A5 runs as k_blk_spmm_fused, which also writes the next P1 (unless
//                  kApplyNoP1) and G = Y^T Y, s = 1^T Y (and H' = Yprev^T Y when Yprev != NULL)
//   kApplySp8:     (with kApplyFused) the tensor-core sparse step k_sp8_step instead, and the
//                  partials of kApplyY1Ready are its 128-row-block slots
//   kApplyChol:    (with kApplySp8) the step's last CTA also factors G = R^T R into h->Rinv2
//   kApplyGram8:   (with kApplySp8) G and 1^T Y from Y's 24-bit digits on the int8 tensor cores
//                  (steps whose Gram feeds only the next Cholesky-QR, not a Rayleigh-Ritz step)
//   kApplySp8Halves: (with kApplySp8, b = 32) the step as two 16-column passes over the images, then the
//                  Gram kernel on Y (the halves share no Gram)
constexpr int kApplyY1Ready = 1, kApplyFused = 2, kApplyNoP1 = 4, kApplySp8 = 8, kApplyChol = 16, kApplyGram8 = 32,
              kApplySp8Halves = 64;

bool ensure_sp8(sbmds_ctx* h, cudaStream_t st);
void gram(sbmds_ctx* h, int b, const float* Y, const float* X, cudaStream_t st, bool want_s);
// index of the two norms behind the padded row-sum deviations in h->s8rs1
int64_t sp8_rs_pad(const sbmds_ctx* h) { return ((h->n + 3) & ~(int64_t)3) + kSp8RB; }

bool sp8_ok(sbmds_ctx* h, int b, cudaStream_t st) {
    if (h->sp8_state == 0) {   // (the build reads sizes back: never inside a stream capture)
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return false;
    }
    return h->fuse == 3 && b == 16 && h->blocked && (h->use_blocked & 1) && ensure_sp8(h, st);
}

// no_gram: the standalone apply's A5 (N products only: no T partials, no Gram).
// b = 32: two passes over the images, one per 16-column half of the block (the kernel's widths
// are 16: a 32-wide step would need TMEM and shared memory it does not have); the halves share
// nothing but the images, so no Gram is formed here (the caller runs the Gram kernel on Y).
void launch_sp8(sbmds_ctx* h, int b, float* Y, const float* Yprev, bool want_p1, cudaStream_t st, bool with_chol,
                bool gram8, bool no_gram = false) {
    using C = Sp8Cfg<16>;
    smem_attr(k_sp8_step<16, false, false>, C::SMEM);
    smem_attr(k_sp8_step<16, true, false>, C::SMEM);
    smem_attr(k_sp8_step<16, false, true>, Sp8Cfg<16, true>::SMEM);
    const int nh = b / 16;   // 16-column halves
    gram8 = gram8 && !Yprev && want_p1 && nh == 1;   // (the int8 Gram reads the digits the T product stages)
    if (gram8) ++h->gram8_launches;
    if (no_gram) {   // (the GRAM8 variant without T products forms nothing but Y)
        gram8 = true;
        want_p1 = false;
        Yprev = nullptr;
    }
    if (nh == 2) {   // (no Gram in the kernel: GRAM8 layout, mode bit 8)
        gram8 = true;
        Yprev = nullptr;
    }
    h->y16aux.ensure(352 * sizeof(unsigned int));
    unsigned int* y2mm = h->y16aux.as<unsigned int>() + 192;   // Y2 column max [0, 64) / min [64, 128) keys
    int* ey2 = reinterpret_cast<int*>(h->y16aux.as<unsigned int>() + 320);
    if (h->last_dpath != 3 && h->last_dpath != 4) {   // the full-D reductions do not form the keys
        CK(cudaMemsetAsync(y2mm, 0, 64 * sizeof(unsigned int), st));
        CK(cudaMemsetAsync(y2mm + 64, 0xFF, 64 * sizeof(unsigned int), st));
        launch(k_colminmax, dim3((unsigned)std::min<int64_t>(2 * 148, (h->l + 15) / 16)), dim3(256), 0, st, h->l, b,
               (const float*)h->Y2.as<float>(), y2mm);
    }
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(h->s8.nblk, h->num_sms));
    h->gpart.ensure((size_t)std::max(grid, kRedBlocks) * kGramPart * sizeof(double));
    h->P1.ensure((size_t)std::max<int32_t>(std::max(1, h->s8.total_u), h->total_u) * kMaxB * sizeof(float));
    // Y2's digit planes (one pass over l x 16 per half), then the step
    h->s8yd.ensure((size_t)3 * h->l * 16 * nh);
    if (h->sp8_dbg & 2) h->s8trace.ensure((2048 + 8 * 64) * sizeof(unsigned long long));
    auto kern = Yprev ? k_sp8_step<16, true, false> : (gram8 ? k_sp8_step<16, false, true> : k_sp8_step<16, false, false>);
    // non-Rayleigh-Ritz eigs steps whose next apply folds through k_blk_reduce_fold (sym8 D
    // stream) leave E2/E3 to that fold (off this kernel's tail)
    const bool defer = no_gram || nh == 2 ||
                       (with_chol && !Yprev && grid >= 1 && uses_sym(h, 16) && h->dstream != 4 && !(h->sp8_dbg & 128));
    for (int hf = 0; hf < nh; ++hf) {
        const int c0 = 16 * hf;
        uint8_t* yd = h->s8yd.as<uint8_t>() + (size_t)hf * 3 * h->l * 16;
        if (!h->y2d_ready)
            launch_pdl(k_y2_digits<16>, dim3((unsigned)std::min<int64_t>(4 * 148, (h->l + 255) / 256)), dim3(256), 0, st, h->l,
                       (const float*)h->Y2.as<float>() + c0, (const double*)h->t.as<double>() + c0,
                       (const unsigned int*)y2mm + c0, ey2 + c0, yd,
                       hf == 0 ? h->y16aux.as<unsigned int>() + 64 : (unsigned int*)nullptr, b);
        launch_pdl(kern, dim3(grid), dim3(C::THREADS), (size_t)(gram8 ? Sp8Cfg<16, true>::SMEM : C::SMEM), st, h->n, h->l,
               h->s8.nblk, (const int8_t*)h->s8img.as<int8_t>(),
               (const int64_t*)h->s8ioff.as<int64_t>(), (const int32_t*)h->s8.doff.as<int32_t>(),
               (const int32_t*)h->s8.dict.as<int32_t>(), (const int*)h->s8esc.as<int>(), (const uint8_t*)yd,
               (const int*)ey2 + c0, (const double*)h->t.as<double>() + c0, (const float*)h->s8rs1.as<float>(),
               (const float*)h->s8rs1.as<float>() + sp8_rs_pad(h), (const int32_t*)h->s8pos.as<int32_t>(), Y + c0,
               want_p1 ? h->P1.as<float>() + c0 : nullptr,
               Yprev, h->gpart.as<double>(), h->G.as<double>(), h->H.as<double>(), h->s.as<double>(),
               h->counters.as<unsigned int>() + CNT_GRAM, (h->sp8_dbg & 2) ? h->s8trace.as<unsigned long long>() : nullptr,
               ((h->sp8_dbg & 4) ? 1 : 0) | ((h->sp8_dbg >> 7) & 6) | (nh == 2 ? 8 : 0) | ((h->sp8_pf & 15) << 4) |
                   (h->sp8_poll << 8),
               with_chol && nh == 1 ? h->Rinv2.as<double>() : nullptr, h->status.as<int>(), defer ? 1 : 0, b, b,
               (const int32_t*)h->s8.brow0.as<int32_t>());
    }
    h->gram_deferred = defer && !no_gram && nh == 1;
    h->gram_parts = grid;
}

// G = Y^T Y and s = 1^T Y of an n x 32 block from Y's digits on the int8 tensor cores (k_gram8_32;
// the scales are the sparse step's: its ey2 exponents, t and norms of this apply)
void gram8_32(sbmds_ctx* h, const float* Y, cudaStream_t st) {
    smem_attr(k_gram8_32, Gram8Cfg::SMEM);
    const int64_t nblk = (h->n + kSp8RB - 1) / kSp8RB;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(nblk, 2 * (int64_t)h->num_sms));
    h->gpart.ensure((size_t)std::max(grid, kRedBlocks) * kGramPart * sizeof(double));
    profiled(h->prof, PK_GRAM, st, [&] {
        launch(k_gram8_32, dim3(grid), dim3(Gram8Cfg::THREADS), (size_t)Gram8Cfg::SMEM, st, h->n, Y,
               (const int*)(h->y16aux.as<unsigned int>() + 320), (const double*)h->t.as<double>(),
               (const float*)h->s8rs1.as<float>() + sp8_rs_pad(h), h->gpart.as<double>(), h->G.as<double>(),
               h->s.as<double>(), (unsigned int*)nullptr);
        launch(k_gram_sum, dim3((unsigned)((4 * (32 * 32 + 32) + 255) / 256)), dim3(256), 0, st, 32, grid,
               (const double*)h->gpart.as<double>(), h->G.as<double>(), (double*)nullptr, h->s.as<double>());
    });
    ++h->gram8_launches;
}

bool fused_ok(const sbmds_ctx* h, int b) {
    return h->fuse && h->blocked && (h->use_blocked & 1) && (b == 4 || b == 8 || b == 16 || b == 32) &&
           (size_t)h->umax * b * sizeof(float) <= kBlkSmem;
}

template <int LPR>
void launch_fused(sbmds_ctx* h, int b, float* Y, const float* Yprev, bool want_p1, cudaStream_t st) {
    const bool with_h = Yprev != nullptr;
    const size_t smem = fused_smem_bytes(h->umax, b, with_h);
    // attribute and occupancy per (variant, smem), queried once: never inside a graph capture
    static int occ[2][5] = {};
    static size_t occ_smem[2][5] = {};
    const int li = LPR == 1 ? 0 : (LPR == 2 ? 1 : (LPR == 4 ? 2 : 3));
    auto kern = with_h ? k_blk_spmm_fused<LPR, true> : k_blk_spmm_fused<LPR, false>;
    if (smem > 48 * 1024) smem_attr(kern, (int)smem);   // (per device)
    if (occ_smem[with_h][li] != smem) {
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[with_h][li], kern, 256, smem));
        occ_smem[with_h][li] = smem;
    }
    const int per_sm = occ[with_h][li];
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(h->nblk, (int64_t)std::max(1, per_sm) * h->num_sms));
    h->gpart.ensure((size_t)std::max(grid, kRedBlocks) * kGramPart * sizeof(double));
    h->P1.ensure((size_t)std::max<int32_t>(1, h->total_u) * kMaxB * sizeof(float));
    launch(kern, dim3(grid), dim3(256), smem, st, h->n, h->nblk, b, (const int32_t*)h->rp.as<int32_t>(),
           (const uint16_t*)h->blcol.as<uint16_t>(), (const float*)h->val.as<float>(),
           (const int32_t*)h->bdict.as<int32_t>(), (const int32_t*)h->bdoff.as<int32_t>(), (uint32_t)h->umax,
           (const float*)h->Y2.as<float>(), (const double*)h->t.as<double>(), Y,
           (const int32_t*)h->blcp.as<int32_t>(), (const uint8_t*)h->blrow.as<uint8_t>(),
           (const float*)h->blval.as<float>(), want_p1 ? h->P1.as<float>() : nullptr, Yprev,
           h->gpart.as<double>(), h->G.as<double>(), h->H.as<double>(), h->s.as<double>(),
           h->counters.as<unsigned int>() + CNT_GRAM);
}

void apply_device(sbmds_ctx* h, int b, const float* X, float* Y, cudaStream_t st, bool s_ready = false,
                  const double* Rinv = nullptr, int flags = 0, const float* Yprev = nullptr) {
    const int bp = next_pow2(b);
    ensure_apply_ws(h, bp);
    const bool blk = blocked_ok(h, b, bp, X, Y);
    // standalone apply at b = 16 with S local (k_sp8.cuh's images): A2 as the T products, A5 as the
    // N products of the tensor-core sparse step
    const bool sp8_a = flags == 0 && (b == 16 || b == 32) && blk && h->sp8_apply && h->n >= h->sp8_min_rows &&
                       (reinterpret_cast<uintptr_t>(X) & 15) == 0 && sp8_ok(h, 16, st);
    bool sp8_a2 = false;
    // A1: s = 1^T X (inside eigs it was produced by the previous rotate)
    if (!s_ready) profiled(h->prof, PK_COLSUM, st, [&] {
        if (sp8_a && h->dy_max_range < 64) {
            colsum_xstat(h, b, X, st);
            sp8_a2 = true;   // (optimistic: X's check is read with Y1's, after A2)
        } else {
            colsum(h, b, X, st);
        }
    });
    // blocked mask: the option, or (auto, standalone apply) S^T X blocked and S Y2 plain for
    // b >= 32: measured on config 3 (b = 32) 0.63 ms vs 0.83 ms with the b = 16 default
    // (blocked S Y2, CSC S^T X), DESIGN.md §4
    const int bmask = (h->blocked_auto && flags == 0 && b >= 32) ? 2 : h->use_blocked;
    if (blk) {
        // opt the blocked kernels into > 48 KB of dynamic smem (once per device)
        for (auto k : {k_blk_spmmt<1>, k_blk_spmmt<2>, k_blk_spmmt<4>, k_blk_spmmt<8>, k_blk_spmmt<16>})
            smem_attr(k, kRB * kMaxB * 4);
        for (auto k : {k_blk_spmm<1>, k_blk_spmm<2>, k_blk_spmm<4>, k_blk_spmm<8>, k_blk_spmm<16>})
            smem_attr(k, (int)kBlkSmem);
    }
    // A2: Y1 = S^T X - w s^T   (CSC SpMM by default; row-blocked partials + landmark
    // reduction when enabled: both are bound by the 64-B-per-nonzero gather traffic; inside
    // eigs the partials come from the previous fused step, leaving only the reduction)
    if ((flags & kApplyY1Ready) && (flags & kApplySp8) && b == 16 && Rinv && uses_sym(h, 16) && h->dstream != 4) {
        // landmark reduce of the step's T partials fused with the R^-1 fold of the int8 D stream
        const int64_t lpad = y1t_lpad(h);
        h->Y1f.ensure((size_t)lpad * kMaxB * sizeof(float));
        h->y16aux.ensure(352 * sizeof(unsigned int));
        unsigned int* aux = h->y16aux.as<unsigned int>();
        profiled(h->prof, PK_CSC, st, [&] {
            // (aux[64, 128), the column maxima, were zeroed by the last k_y2_digits); one cooperative
            // launch also splits Y1f into the D stream's digits (k_y8_split's work)
            static int per_sm = 0;
            if (!per_sm) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_blk_reduce_fold, 256, 0));
            h->Y8T.ensure((size_t)3 * kMaxB * lpad);
            // (4 blocks per SM under __launch_bounds__(256, 4): 0.050 vs 0.053 ms with 3 at config 4)
            const int64_t grid = std::min<int64_t>(std::min(4, std::max(1, per_sm)) * (int64_t)h->num_sms, (lpad + 7) / 8);
            FoldGram fg;
            if (h->gram_deferred) {   // E2/E3 of the previous step (R^-1 into the buffer this apply folds with)
                h->foldscr.ensure((size_t)lpad * 16 * sizeof(double));
                fg.part = h->gpart.as<double>();
                fg.nparts = h->gram_parts;
                fg.G = h->G.as<double>();
                fg.s_out = h->s.as<double>();
                fg.Rinv_out = const_cast<double*>(Rinv);
                fg.status = h->status.as<int>();
                fg.scratch = h->foldscr.as<double>();
                fg.counter = h->counters.as<unsigned int>() + CNT_FOLD;
                h->gram_deferred = false;
            }
            launch_coop_pdl(k_blk_reduce_fold, dim3((unsigned)std::max<int64_t>(kFoldGramBlocks + 1, grid)), dim3(256), 0, st, h->l, lpad,
                        (const int32_t*)h->s8.jptr.as<int32_t>(), (const float*)h->P1.as<float>(), wvec(h),
                        (const double*)h->s.as<double>(), Rinv, h->Y1f.as<float>(), aux + 64, aux + 192,
                        h->Y8T.as<int8_t>(), reinterpret_cast<int*>(aux + 128), fg);
        });
        h->y1f_ready = true;
    } else if (flags & kApplyY1Ready) {
        const bool s8 = (flags & kApplySp8) != 0;
        auto go_r = [&](auto kern) {
            launch(kern, dim3((unsigned)((h->l + 7) / 8)), dim3(256), 0, st, h->l, b, bp,
                   (const int32_t*)(s8 ? h->s8.jptr : h->bjptr).as<int32_t>(),
                   s8 ? (const int32_t*)nullptr : (const int32_t*)h->bjlist.as<int32_t>(),   // sp8: landmark-major
                   (const float*)h->P1.as<float>(), wvec(h), (const double*)h->s.as<double>(),
                   h->Y1.as<float>());
        };
        profiled(h->prof, PK_CSC, st, [&] {
            switch (b / 4) {
                case 1: go_r(k_blk_reduce<1>); break;
                case 2: go_r(k_blk_reduce<2>); break;
                case 4: go_r(k_blk_reduce<4>); break;
                default: go_r(k_blk_reduce<8>); break;
            }
        });
    } else if (sp8_a2) {
        profiled(h->prof, PK_CSC, st, [&] {
            launch_sp8_t(h, b, X, st);
            auto go_r = [&](auto kern) {
                launch(kern, dim3((unsigned)((h->l + 7) / 8)), dim3(256), 0, st, h->l, b, bp,
                       (const int32_t*)h->s8.jptr.as<int32_t>(), (const int32_t*)nullptr,   // landmark-major partials
                       (const float*)h->P1.as<float>(), wvec(h), (const double*)h->s.as<double>(), h->Y1.as<float>());
            };
            if (b == 16) go_r(k_blk_reduce<4>);
            else go_r(k_blk_reduce<8>);
        });
        ++h->sp8_apply_t_launches;
    } else if (blk && (bmask & 2)) {
        h->P1.ensure((size_t)std::max<int32_t>(1, h->total_u) * kMaxB * sizeof(float));
        const size_t smem_t = (size_t)kRB * bp * sizeof(float);
        auto go_t = [&](auto kern) {
            launch(kern, dim3((unsigned)h->nblk), dim3(256), smem_t, st, h->n, b, bp, X,
                   (const int32_t*)h->bdoff.as<int32_t>(), (const int32_t*)h->blcp.as<int32_t>(),
                   (const uint8_t*)h->blrow.as<uint8_t>(), (const float*)h->blval.as<float>(), h->P1.as<float>());
        };
        auto go_r = [&](auto kern) {
            launch(kern, dim3((unsigned)((h->l + 7) / 8)), dim3(256), 0, st, h->l, b, bp,
                   (const int32_t*)h->bjptr.as<int32_t>(), (const int32_t*)h->bjlist.as<int32_t>(),
                   (const float*)h->P1.as<float>(), wvec(h), (const double*)h->s.as<double>(),
                   h->Y1.as<float>());
        };
        profiled(h->prof, PK_CSC, st, [&] {
            switch (b / 4) {
                case 1: go_t(k_blk_spmmt<1>); go_r(k_blk_reduce<1>); break;
                case 2: go_t(k_blk_spmmt<2>); go_r(k_blk_reduce<2>); break;
                case 4: go_t(k_blk_spmmt<4>); go_r(k_blk_reduce<4>); break;
                case 8: go_t(k_blk_spmmt<8>); go_r(k_blk_reduce<8>); break;
                default: go_t(k_blk_spmmt<16>); go_r(k_blk_reduce<16>); break;
            }
        });
    } else {
        profiled(h->prof, PK_CSC, st, [&] { spmm_csc(h, b, bp, X, st); });
    }
    // standalone apply on the int8 stream (auto): check Y1's columns first (one small readback)
    const bool want_y = flags == 0 && (!Rinv || h->raw_now) && h->dstream == 0 && h->dy_max_range < 64 &&
                        takes_sym(h, bp, Rinv != nullptr);
    if (want_y || sp8_a2) {
        bool x_ok = true;
        ycheck(h, b, bp, st, want_y, sp8_a2 ? &x_ok : nullptr);   // one readback for both
        if (!x_ok) {   // a dominant row in X: A2 again on the fp32 CSC kernel, and Y1's check on that Y1
            ++h->x_fallbacks;
            --h->sp8_apply_t_launches;
            if (h->y_fallback) {
                h->y_fallback = false;
                --h->y_fallbacks;
            }
            profiled(h->prof, PK_CSC, st, [&] { spmm_csc(h, b, bp, X, st); });
            if (want_y) ycheck(h, b, bp, st);
        }
    }
    // A3, A4: Y2 = D Y1, t = w^T Y2   (eigs: Y1 <- Y1 R^-1 first, the R^-1 fold)
    // standalone apply at b = 16: A5 through the N products of the tensor-core sparse step
    const bool sp8_a5 = sp8_a;
    h->y2d_want = (((flags & kApplyFused) && (flags & kApplySp8)) || sp8_a5) && b == 16 && !(h->sp8_dbg & 64);   // (sp8_dbg & 64: separate k_y2_digits, diagnostics)
    h->y2d_ready = false;
    dstream(h, b, bp, st, Rinv);
    h->y2d_want = false;
    h->y_fallback = false;
    // A5: Y = -1/2 (S Y2 - 1 t^T)
    if ((flags & kApplyFused) && (flags & kApplySp8)) {
        profiled(h->prof, PK_CSR, st, [&] {
            launch_sp8(h, b, Y, Yprev, !(flags & kApplyNoP1) && !(h->sp8_dbg & 1), st, (flags & kApplyChol) != 0,
                       (flags & kApplyGram8) != 0);
        });
        // G = Y^T Y, s = 1^T Y (and H' = Yprev^T Y) of the two halves together
        if (flags & kApplySp8Halves) {
            if ((flags & kApplyGram8) && !Yprev) gram8_32(h, Y, st);   // (reading R18: no Rayleigh-Ritz step reads it)
            else gram(h, b, Y, Yprev, st, true);
        }
    } else if (flags & kApplyFused) {
        const bool want_p1 = !(flags & kApplyNoP1);
        profiled(h->prof, PK_CSR, st, [&] {
            switch (b / 4) {
                case 1: launch_fused<1>(h, b, Y, Yprev, want_p1, st); break;
                case 2: launch_fused<2>(h, b, Y, Yprev, want_p1, st); break;
                case 4: launch_fused<4>(h, b, Y, Yprev, want_p1, st); break;
                default: launch_fused<8>(h, b, Y, Yprev, want_p1, st); break;
            }
        });
    } else if (sp8_a5) {
        // standalone apply: the N products of the tensor-core sparse step (S_B as dense digit
        // images, Y2 - 1 t^T as 24-bit digits; k_sp8.cuh) instead of the row-blocked fp32 SpMM
        profiled(h->prof, PK_CSR, st, [&] { launch_sp8(h, b, Y, nullptr, false, st, false, false, true); });
        ++h->sp8_apply_launches;
    } else if (blk && (bmask & 1)) {
        const size_t smem = (size_t)h->umax * bp * sizeof(float);
        auto go = [&](auto kern) {
            launch(kern, dim3((unsigned)h->nblk), dim3(256), smem, st, h->n, b, bp, (const int32_t*)h->rp.as<int32_t>(),
                   (const uint16_t*)h->blcol.as<uint16_t>(), (const float*)h->val.as<float>(),
                   (const int32_t*)h->bdict.as<int32_t>(), (const int32_t*)h->bdoff.as<int32_t>(),
                   (const float*)h->Y2.as<float>(), (const double*)h->t.as<double>(), Y);
        };
        profiled(h->prof, PK_CSR, st, [&] {
            switch (b / 4) {
                case 1: go(k_blk_spmm<1>); break;
                case 2: go(k_blk_spmm<2>); break;
                case 4: go(k_blk_spmm<4>); break;
                case 8: go(k_blk_spmm<8>); break;
                default: go(k_blk_spmm<16>); break;
            }
        });
    } else {
        profiled(h->prof, PK_CSR, st, [&] { spmm_csr(h, b, bp, Y, st); });
    }
}

// Row-blocked S (k_blocked.cuh): segmented stable sort of each rb-row block's entries by
// column, unique -> per-block dictionary, 16-bit local columns (CSR order), optionally the
// block-local CSC (sorted order), and for each landmark its dictionary slots in block order.
// (brow0 / blkof / nblk_var: blocks of <= rb rows with explicit row ranges instead of rb rows each)
void build_blk_index(sbmds_ctx* h, const int32_t* rowof, int rb, bool want_csc, BlkIdx& o, cudaStream_t st,
                     const int32_t* brow0 = nullptr, const int32_t* blkof = nullptr, int64_t nblk_var = 0) {
    const int64_t n = h->n, l = h->l, nnz = h->nnz;
    o.rb = rb;
    o.nblk = brow0 ? nblk_var : (n + rb - 1) / rb;
    const int64_t nb = o.nblk;
    // temporaries from the stream-ordered pool (every use completes before the stream syncs below)
    DevBuf off{true}, scol{true}, iota_perm{true}, flag{true}, incl{true}, tmp{true}, keys2{true};
    off.ensure((nb + 1) * sizeof(int32_t));
    scol.ensure(nnz * sizeof(int32_t));
    iota_perm.ensure(2 * nnz * sizeof(int32_t));
    flag.ensure(nnz * sizeof(int32_t));
    incl.ensure(nnz * sizeof(int32_t));
    int32_t* iota = iota_perm.as<int32_t>();
    int32_t* perm = iota + nnz;
    launch(k_blk_offsets, dim3((unsigned)std::min<int64_t>(1024, (nb + 256) / 256)), dim3(256), 0, st, n, nb, rb,
           (const int32_t*)h->rp.as<int32_t>(), off.as<int32_t>(), brow0);
    launch(k_iota, dim3(1024), dim3(256), 0, st, (int32_t)nnz, iota);
    size_t tb = 0;
    CK(cub::DeviceSegmentedSort::StableSortPairs(nullptr, tb, h->col.as<int32_t>(), scol.as<int32_t>(), iota, perm,
                                                 (int)nnz, (int)nb, off.as<int32_t>(), off.as<int32_t>() + 1, st));
    tmp.ensure(tb + 16);
    CK(cub::DeviceSegmentedSort::StableSortPairs(tmp.p, tb, h->col.as<int32_t>(), scol.as<int32_t>(), iota, perm,
                                                 (int)nnz, (int)nb, off.as<int32_t>(), off.as<int32_t>() + 1, st));
    g_launches.fetch_add(1);
    launch(k_blk_flags, dim3(1024), dim3(256), 0, st, (int32_t)nnz, rb, (const int32_t*)scol.as<int32_t>(),
           (const int32_t*)perm, rowof, (const int32_t*)off.as<int32_t>(), flag.as<int32_t>(), blkof);
    tb = 0;
    CK(cub::DeviceScan::InclusiveSum(nullptr, tb, flag.as<int32_t>(), incl.as<int32_t>(), (int)nnz, st));
    DevBuf tmp2{true};
    tmp2.ensure(tb + 16);
    CK(cub::DeviceScan::InclusiveSum(tmp2.p, tb, flag.as<int32_t>(), incl.as<int32_t>(), (int)nnz, st));
    g_launches.fetch_add(1);
    int32_t total_u = 0;
    peek_to_host(&total_u, incl.as<int32_t>() + nnz - 1, sizeof(int32_t), st);
    o.total_u = total_u;
    o.doff.ensure((nb + 1) * sizeof(int32_t));
    o.dict.ensure(std::max<int64_t>(1, total_u) * sizeof(int32_t));
    o.lcol.ensure(nnz * sizeof(uint16_t));
    if (want_csc) {
        o.lcp.ensure((total_u + 1) * sizeof(int32_t));
        o.lrow.ensure(nnz * sizeof(uint8_t));
        o.lval.ensure(nnz * sizeof(float));
    }
    o.jptr.ensure((l + 1) * sizeof(int32_t));
    o.jlist.ensure(std::max<int64_t>(1, total_u) * sizeof(int32_t));
    launch(k_blk_dictoff, dim3((unsigned)std::min<int64_t>(1024, (nb + 256) / 256)), dim3(256), 0, st, nb,
           (int32_t)nnz, (const int32_t*)off.as<int32_t>(), (const int32_t*)flag.as<int32_t>(),
           (const int32_t*)incl.as<int32_t>(), total_u, o.doff.as<int32_t>());
    launch(k_blk_scatter, dim3(1024), dim3(256), 0, st, (int32_t)nnz, rb, (const int32_t*)scol.as<int32_t>(),
           (const int32_t*)perm, rowof, (const float*)h->val.as<float>(), (const int32_t*)flag.as<int32_t>(),
           (const int32_t*)incl.as<int32_t>(), (const int32_t*)o.doff.as<int32_t>(), o.dict.as<int32_t>(),
           want_csc ? o.lcp.as<int32_t>() : nullptr, o.lcol.as<uint16_t>(), want_csc ? o.lrow.as<uint8_t>() : nullptr,
           want_csc ? o.lval.as<float>() : nullptr, blkof, brow0);
    const int32_t nnz32 = (int32_t)nnz;
    if (want_csc)
        CK(cudaMemcpyAsync(o.lcp.as<int32_t>() + total_u, &nnz32, sizeof(int32_t), cudaMemcpyHostToDevice, st));
    // largest dictionary (decides which block widths fit in shared memory)
    DevBuf um{true};
    um.ensure(sizeof(unsigned int));
    CK(cudaMemsetAsync(um.p, 0, sizeof(unsigned int), st));
    launch(k_blk_umax, dim3(256), dim3(256), 0, st, nb, (const int32_t*)o.doff.as<int32_t>(), um.as<unsigned int>());
    // landmark -> dictionary slots, ascending slot (= block) order: stable sort of (dict, slot)
    keys2.ensure(std::max<int64_t>(1, total_u) * sizeof(int32_t));
    DevBuf slot{true};
    slot.ensure(std::max<int64_t>(1, total_u) * sizeof(int32_t));
    launch(k_iota, dim3(256), dim3(256), 0, st, total_u, slot.as<int32_t>());
    int end_bit = 1;
    while ((int64_t(1) << end_bit) <= l) ++end_bit;
    tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, o.dict.as<int32_t>(), keys2.as<int32_t>(), slot.as<int32_t>(),
                                       o.jlist.as<int32_t>(), total_u, 0, end_bit, st));
    DevBuf tmp3{true};
    tmp3.ensure(tb + 16);
    CK(cub::DeviceRadixSort::SortPairs(tmp3.p, tb, o.dict.as<int32_t>(), keys2.as<int32_t>(), slot.as<int32_t>(),
                                       o.jlist.as<int32_t>(), total_u, 0, end_bit, st));
    g_launches.fetch_add(1);
    launch(k_col_ptr, dim3((unsigned)((l + 256) / 256)), dim3(256), 0, st, l, total_u,
           (const int32_t*)keys2.as<int32_t>(), o.jptr.as<int32_t>());
    unsigned int umax = 0;
    peek_to_host(&umax, um.p, sizeof umax, st);
    o.umax = umax;
}

void build_blocked(sbmds_ctx* h, const int32_t* rowof, cudaStream_t st) {
    BlkIdx o;
    build_blk_index(h, rowof, kRB, true, o, st);
    h->nblk = o.nblk;
    h->total_u = o.total_u;
    h->umax = o.umax;
    h->bdoff.swap(o.doff);
    h->bdict.swap(o.dict);
    h->blcp.swap(o.lcp);
    h->blcol.swap(o.lcol);
    h->blrow.swap(o.lrow);
    h->blval.swap(o.lval);
    h->bjptr.swap(o.jptr);
    h->bjlist.swap(o.jlist);
    // staging pays only when a staged landmark row is reused: mean uses per dictionary entry
    // >= 4 (config 4: ~40; random rows over wide column windows: ~1)
    h->blocked = (double)h->nnz >= 4.0 * (double)std::max<int32_t>(1, h->total_u);
}

// Tensor-core sparse step (k_sp8.cuh): 128-row blocks whose dictionaries all fit 128 entries,
// S_B stored once as a dense three-plane digit image. Built at the first eigs that can use it
// (the row index of every entry is re-expanded from the row pointers).
// One round of the tensor-core sparse kernels' block splitting: every block [r0[B], r0[B + 1]) whose
// dictionary (doff[B + 1] - doff[B] landmarks) exceeds `limit` is halved at a multiple of 4 rows
// from its start (the step stages 16-byte groups of per-row data from a block's first row). Returns
// the number of blocks halved, or -1 when such a block has fewer than 8 rows (it cannot be halved
// into pieces of >= 4 rows); out = the new boundaries.
int64_t sp8_split_rows(int64_t n, const std::vector<int32_t>& r0, const std::vector<int32_t>& doff, int limit,
                       std::vector<int32_t>& out) {
    const int64_t nblk = (int64_t)r0.size() - 1;
    out.clear();
    out.reserve(r0.size() + 64);
    int64_t nsplit = 0;
    for (int64_t B = 0; B < nblk; ++B) {
        out.push_back(r0[B]);
        const int32_t rows = r0[B + 1] - r0[B];
        if (doff[B + 1] - doff[B] > limit) {
            if (rows < 8) return -1;
            out.push_back(r0[B] + ((rows / 2 + 3) & ~3));
            ++nsplit;
        }
    }
    out.push_back((int32_t)n);
    return nsplit;
}

bool ensure_sp8(sbmds_ctx* h, cudaStream_t st) {
    if (h->sp8_state != 0) return h->sp8_state > 0;
    h->sp8_state = -1;
    if (!h->blocked || h->nnz == 0) return false;
    DevBuf rowof{true}, bad{true};
    rowof.ensure(h->nnz * sizeof(int32_t));
    bad.ensure(sizeof(int));
    CK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    launch(k_expand_rows, dim3(1024), dim3(256), 0, st, h->n, (const int32_t*)h->rp.as<int32_t>(),
           (const int32_t*)h->col.as<int32_t>(), (const float*)h->val.as<float>(), h->l, rowof.as<int32_t>(),
           bad.as<int>());
    BlkIdx& o = h->s8;
    build_blk_index(h, rowof.as<int32_t>(), kSp8RB, false, o, st);
    // block row ranges: 128 rows each; a block whose dictionary exceeds one image (an ordering
    // jump inside it: a Morton-numbered mesh has a few) is halved, at multiples of 4 rows, until
    // its pieces fit (the image keeps 128 row slots, the unused ones zero)
    std::vector<int32_t> r0((size_t)o.nblk + 1);
    for (int64_t B = 0; B <= o.nblk; ++B) r0[B] = (int32_t)std::min<int64_t>(B * kSp8RB, h->n);
    h->sp8_splits = 0;
    for (int round = 0; o.umax > (uint32_t)kSp8DK && round < 6; ++round) {
        if ((double)o.umax > 4.0 * kSp8DK && round == 0) break;   // (not local at all: random structure)
        std::vector<int32_t> doff((size_t)o.nblk + 1);
        CK(cudaMemcpyAsync(doff.data(), o.doff.p, doff.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        std::vector<int32_t> nr;
        const int64_t ns = sp8_split_rows(h->n, r0, doff, kSp8DK, nr);
        if (ns < 0 || nr.size() > (size_t)2 * ((h->n + kSp8RB - 1) / kSp8RB) + 2) break;   // (stuck, or would double the images)
        h->sp8_splits += ns;
        r0.swap(nr);
        const int64_t nb2 = (int64_t)r0.size() - 1;
        o.reset();
        o.brow0.ensure(r0.size() * sizeof(int32_t));
        CK(cudaMemcpyAsync(o.brow0.p, r0.data(), r0.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
        DevBuf blkof{true};
        blkof.ensure(h->n * sizeof(int32_t));
        launch(k_blk_fill_blkof, dim3((unsigned)std::min<int64_t>(1024, (nb2 + 255) / 256)), dim3(256), 0, st, nb2,
               (const int32_t*)o.brow0.as<int32_t>(), blkof.as<int32_t>());
        DevBuf keep{true};
        keep.swap(o.brow0);   // (build_blk_index leaves brow0 alone, reset() above must not free it mid-build)
        build_blk_index(h, rowof.as<int32_t>(), kSp8RB, false, o, st, (const int32_t*)keep.as<int32_t>(),
                        (const int32_t*)blkof.as<int32_t>(), nb2);
        o.brow0.swap(keep);
        CK(cudaStreamSynchronize(st));   // (r0 / the pool temporaries of this round)
    }
    if (o.umax > (uint32_t)kSp8DK ||   // a block touches more landmarks than one image holds, or
        (o.nblk + h->num_sms - 1) / h->num_sms > Sp8Cfg<16>::MAXNB) {   // a CTA's metadata table overflows
        o.reset();
        return false;
    }
    if (!o.brow0.p) {   // the plain ranges
        o.brow0.ensure(r0.size() * sizeof(int32_t));
        CK(cudaMemcpyAsync(o.brow0.p, r0.data(), r0.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
    }
    h->s8ioff.ensure((o.nblk + 1) * sizeof(int64_t));
    DevBuf sizes{true}, tmp{true};
    sizes.ensure((o.nblk + 1) * sizeof(int64_t));
    launch(k_sp8_sizes, dim3((unsigned)std::min<int64_t>(1024, (o.nblk + 255) / 256)), dim3(256), 0, st, o.nblk,
           (const int32_t*)o.doff.as<int32_t>(), sizes.as<int64_t>());
    CK(cudaMemsetAsync(sizes.as<int64_t>() + o.nblk, 0, sizeof(int64_t), st));
    size_t tb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, sizes.as<int64_t>(), h->s8ioff.as<int64_t>(), (int)(o.nblk + 1), st));
    tmp.ensure(tb + 16);
    CK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, sizes.as<int64_t>(), h->s8ioff.as<int64_t>(), (int)(o.nblk + 1), st));
    g_launches.fetch_add(1);
    int64_t total = 0;
    peek_to_host(&total, h->s8ioff.as<int64_t>() + o.nblk, sizeof(int64_t), st);
    h->s8img.ensure((size_t)total + 64 * 1024);   // + slack: the T product's M = 128 rows read past a short image
    CK(cudaMemsetAsync(h->s8img.p, 0, h->s8img.bytes, st));
    h->s8esc.ensure(o.nblk * sizeof(int));
    bad.ensure(sizeof(unsigned int));
    CK(cudaMemsetAsync(bad.p, 0, sizeof(unsigned int), st));
    launch(k_sp8_build, dim3((unsigned)std::min<int64_t>(o.nblk, 32 * (int64_t)h->num_sms)), dim3(128), 0, st, h->n,
           o.nblk, (const int32_t*)h->rp.as<int32_t>(), (const float*)h->val.as<float>(),
           (const uint16_t*)o.lcol.as<uint16_t>(), (const int32_t*)o.doff.as<int32_t>(),
           (const int64_t*)h->s8ioff.as<int64_t>(), h->s8img.as<int8_t>(), h->s8esc.as<int>(), bad.as<unsigned int>(),
           (const int32_t*)o.brow0.as<int32_t>());
    unsigned int rrange = 0;
    peek_to_host(&rrange, bad.p, sizeof rrange, st);
    h->sp8_range = (int)rrange;
    if (h->sp8_range > h->sp8_max_range) {
        // precision check failed (a row's weights sit > sp8_max_range binades below its block's
        // max): the eigs step keeps the fp32 sparse kernels (DESIGN.md §4 precision contract)
        o.reset();
        h->s8img.release();
        h->s8ioff.release();
        h->s8esc.release();
        h->sp8_state = -2;
        return false;
    }
    o.lcol.release();   // only the images are read from now on
    h->s8pos.ensure(std::max<int32_t>(1, o.total_u) * sizeof(int32_t));
    launch(k_inverse_perm, dim3(1024), dim3(256), 0, st, o.total_u, (const int32_t*)o.jlist.as<int32_t>(),
           h->s8pos.as<int32_t>());
    // rs1 padded with 128 zeros (the step stages 512 B from each block's first row), then the
    // two norms of the step's a-priori bound on |Y| (k_rowsum_m1)
    const int64_t rs_pad = sp8_rs_pad(h);
    h->s8rs1.ensure((rs_pad + 4) * sizeof(float));
    CK(cudaMemsetAsync(h->s8rs1.as<float>() + h->n, 0, (rs_pad + 4 - h->n) * sizeof(float), st));
    launch(k_rowsum_m1, dim3((unsigned)std::min<int64_t>(4 * 148, (h->n + 255) / 256)), dim3(256), 0, st, h->n,
           (const int32_t*)h->rp.as<int32_t>(), (const float*)h->val.as<float>(), h->s8rs1.as<float>(),
           reinterpret_cast<unsigned int*>(h->s8rs1.as<float>() + rs_pad));
    h->s8_bytes = total;
    h->sp8_state = 1;
    return true;
}

template <typename F>
void for_each_buf(sbmds_ctx* h, F&& f) {
    DevBuf* bufs[] = {&h->rp, &h->col, &h->val, &h->cptr, &h->ridx, &h->cval, &h->order, &h->w, &h->Dbuf,
                      &h->bdoff, &h->bdict, &h->blcp, &h->blcol, &h->blrow, &h->blval, &h->bjptr, &h->bjlist,
                      &h->P1, &h->Y1, &h->Y2, &h->P, &h->colpart, &h->s, &h->t, &h->tpart, &h->counters, &h->X, &h->Y,
                      &h->gpart, &h->G, &h->H, &h->Rinv, &h->Rinv2, &h->status, &h->rr, &h->vtmp, &h->ztmp, &h->sign,
                      &h->s8.doff, &h->s8.dict, &h->s8.lcol, &h->s8.jptr, &h->s8.jlist, &h->s8.brow0, &h->s8img, &h->s8ioff, &h->s8esc, &h->s8yd, &h->s8rs1, &h->s8pos,
                      &h->lzQ, &h->lzW, &h->lzC, &h->lzT, &h->lzGl, &h->lzI, &h->lzR,
                      &h->apval, &h->apidx, &h->xhost, &h->yhost, &h->vsel, &h->Y1T, &h->w0, &h->rawR, &h->Dt, &h->pdbg, &h->Y16T, &h->Y1f, &h->y16aux, &h->Dt8, &h->Y8T, &h->dqhist, &h->ychk, &h->xstat, &h->Y1w, &h->Y2w, &h->tsave, &h->vg, &h->perm, &h->xperm, &h->yperm, &h->foldscr, &h->s8trace,
                      &h->s8plan[0].tiles, &h->s8plan[0].pbeg, &h->s8plan[0].sbase, &h->s8plan[0].xptr, &h->s8plan[0].xslot, &h->s8plan[0].smap,
                      &h->s8plan[1].tiles, &h->s8plan[1].pbeg, &h->s8plan[1].sbase, &h->s8plan[1].xptr, &h->s8plan[1].xslot, &h->s8plan[1].smap,
                      &h->s8plan[2].tiles, &h->s8plan[2].pbeg, &h->s8plan[2].sbase, &h->s8plan[2].xptr, &h->s8plan[2].xslot, &h->s8plan[2].smap,
                      &h->pplan[0].tiles, &h->pplan[0].pbeg, &h->pplan[0].sbase, &h->pplan[0].xptr, &h->pplan[0].xslot,
                      &h->pplan[1].tiles, &h->pplan[1].pbeg, &h->pplan[1].sbase, &h->pplan[1].xptr, &h->pplan[1].xslot,
                      &h->pplan[2].tiles, &h->pplan[2].pbeg, &h->pplan[2].sbase, &h->pplan[2].xptr, &h->pplan[2].xslot};
    for (DevBuf* b : bufs) f(b);
}

void destroy_ctx(sbmds_ctx* h) {
    if (!h) return;
    if (h->comm) {
        cudaDeviceSynchronize();
        nccl_api().commDestroy(reinterpret_cast<ncclComm_t>(h->comm));
        h->comm = nullptr;
    }
    if (h->pack_st) {
        cudaStreamSynchronize(h->pack_st);
        cudaStreamDestroy(h->pack_st);
        h->pack_st = nullptr;
    }
    if (h->pack_ev) {
        cudaEventDestroy(h->pack_ev);
        h->pack_ev = nullptr;
    }
    if (h->gstream) {
        cudaStreamSynchronize(h->gstream);
        cudaStreamDestroy(h->gstream);
        h->gstream = nullptr;
    }
    for (auto& e : h->gev)
        if (e) {
            cudaEventDestroy(e);
            e = nullptr;
        }
    for_each_buf(h, [](DevBuf* b) { b->release(); });
    cudaStreamSynchronize(0);
    delete h;
}

}  // namespace

// One round of the block splitting of the tensor-core sparse kernels on the host (no GPU; CPU tests):
// r0[nblk + 1] block boundaries, dsize[nblk] dictionary sizes, limit = 128 in the library. Writes
// the new boundaries to r0_out (capacity entries) and returns their count - 1 = the new block
// count, or -1 (a block over the limit has fewer than 8 rows) / -2 (bad arguments, capacity).
extern "C" int64_t sbmds_sparse_split_rows(int64_t n, int64_t nblk, const int32_t* r0, const int32_t* dsize, int32_t limit,
                                        int32_t* r0_out, int64_t capacity) {
    if (n < 1 || nblk < 1 || !r0 || !dsize || limit < 1 || !r0_out) return -2;
    std::vector<int32_t> rv(r0, r0 + nblk + 1), doff((size_t)nblk + 1, 0), out;
    for (int64_t B = 0; B < nblk; ++B) doff[B + 1] = doff[B] + dsize[B];
    if (sp8_split_rows(n, rv, doff, limit, out) < 0) return -1;
    if ((int64_t)out.size() > capacity) return -2;
    std::copy(out.begin(), out.end(), r0_out);
    return (int64_t)out.size() - 1;
}

// ============================================================================ create
namespace {
// Row order (DESIGN.md §4 "Row order"): sort S's rows by their two smallest column indices and
// keep the permuted order when sampled 128-row blocks then touch < 3/4 of the distinct landmarks
// they touch in the caller's order (torus grids keep theirs; the icosphere and the random-window
// rows of config 5 do not). The CSR is rewritten in place; h->perm maps back.
void reorder_rows(sbmds_ctx* h, cudaStream_t st) {
    const int64_t n = h->n, l = h->l, nnz = h->nnz;
    const int64_t nblk = (n + 127) / 128;
    if (nblk < 4 || nnz == 0) return;
    DevBuf keys{true}, keys2{true}, iota{true}, perm{true}, tot{true};
    keys.ensure(n * sizeof(uint64_t));
    keys2.ensure(n * sizeof(uint64_t));
    iota.ensure(n * sizeof(int32_t));
    perm.ensure(n * sizeof(int32_t));
    launch(k_row_keys, dim3((unsigned)std::min<int64_t>(8 * (int64_t)h->num_sms, (n + 255) / 256)), dim3(256), 0, st,
           n, l, (const int32_t*)h->rp.as<int32_t>(), (const int32_t*)h->col.as<int32_t>(), keys.as<uint64_t>(),
           iota.as<int32_t>());
    int lbits = 1;
    while ((int64_t(1) << lbits) <= l) ++lbits;
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.as<uint64_t>(), keys2.as<uint64_t>(), iota.as<int32_t>(),
                                       perm.as<int32_t>(), (int)n, 0, 32 + lbits, st));
    DevBuf tmp{true};
    tmp.ensure(tb + 16);
    CK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.as<uint64_t>(), keys2.as<uint64_t>(), iota.as<int32_t>(),
                                       perm.as<int32_t>(), (int)n, 0, 32 + lbits, st));
    g_launches.fetch_add(1);
    const int64_t stride = std::max<int64_t>(1, nblk / 1024);
    const int64_t ns = (nblk + stride - 1) / stride;
    tot.ensure(2 * ns * sizeof(int32_t));
    const size_t smem = (size_t)((l + 31) / 32) * sizeof(unsigned int);
    if (smem > 48 * 1024) smem_attr(k_block_distinct, (int)smem);
    launch(k_block_distinct, dim3((unsigned)ns), dim3(256), smem, st, n, l, stride, (const int32_t*)nullptr,
           (const int32_t*)h->rp.as<int32_t>(), (const int32_t*)h->col.as<int32_t>(), tot.as<int32_t>());
    launch(k_block_distinct, dim3((unsigned)ns), dim3(256), smem, st, n, l, stride, (const int32_t*)perm.as<int32_t>(),
           (const int32_t*)h->rp.as<int32_t>(), (const int32_t*)h->col.as<int32_t>(), tot.as<int32_t>() + ns);
    std::vector<int32_t> hc(2 * ns);
    for (int64_t o = 0; o < 2 * ns; o += 1024)   // (small readbacks through the mapped buffer)
        peek_to_host(hc.data() + o, tot.as<int32_t>() + o, (size_t)std::min<int64_t>(1024, 2 * ns - o) * 4, st);
    int64_t nat = 0, prm = 0;
    for (int64_t q = 0; q < ns; ++q) { nat += hc[q]; prm += hc[ns + q]; }
    h->order_distinct[0] = nat;
    h->order_distinct[1] = prm;
    if (4 * prm >= 3 * nat) return;
    // rewrite the CSR in the new row order
    DevBuf len{true}, nrp{true}, ncol{true}, nval{true};
    len.ensure((n + 1) * sizeof(int32_t));
    CK(cudaMemsetAsync(len.as<int32_t>() + n, 0, sizeof(int32_t), st));
    launch(k_perm_lengths, dim3((unsigned)std::min<int64_t>(8 * (int64_t)h->num_sms, (n + 255) / 256)), dim3(256), 0, st,
           n, (const int32_t*)perm.as<int32_t>(), (const int32_t*)h->rp.as<int32_t>(), len.as<int32_t>());
    nrp.ensure((n + 1) * sizeof(int32_t));
    ncol.ensure(nnz * sizeof(int32_t));
    nval.ensure(nnz * sizeof(float));
    tb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, len.as<int32_t>(), nrp.as<int32_t>(), (int)(n + 1), st));
    tmp.ensure(tb + 16);
    CK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, len.as<int32_t>(), nrp.as<int32_t>(), (int)(n + 1), st));
    g_launches.fetch_add(1);
    launch(k_perm_rows, dim3((unsigned)std::min<int64_t>(16 * (int64_t)h->num_sms, (n + 7) / 8)), dim3(256), 0, st, n,
           (const int32_t*)perm.as<int32_t>(), (const int32_t*)h->rp.as<int32_t>(), (const int32_t*)h->col.as<int32_t>(),
           (const float*)h->val.as<float>(), (const int32_t*)nrp.as<int32_t>(), ncol.as<int32_t>(), nval.as<float>());
    CK(cudaStreamSynchronize(st));
    h->rp.swap(nrp);
    h->col.swap(ncol);
    h->val.swap(nval);
    h->perm.swap(perm);
    h->permuted = true;
}

// n x b block between the caller's row order and the handle's (no-op copies avoided by callers)
void permute_block(sbmds_ctx* h, int b, const float* in, float* out, bool scatter, cudaStream_t st) {
    const int64_t total = h->n * b;
    const dim3 g((unsigned)std::min<int64_t>(16 * (int64_t)h->num_sms, (total + 255) / 256));
    if (scatter) launch(k_permute_rows<true>, g, dim3(256), 0, st, h->n, b, (const int32_t*)h->perm.as<int32_t>(), in, out);
    else launch(k_permute_rows<false>, g, dim3(256), 0, st, h->n, b, (const int32_t*)h->perm.as<int32_t>(), in, out);
}

// V (n x m, handle order, in place) -> the caller's order, before the sign rule (ties: lowest
// caller index) and Z
void unpermute_v(sbmds_ctx* h, int m, float* V, cudaStream_t st) {
    if (!h->permuted) return;
    h->yperm.ensure((size_t)h->n * m * sizeof(float));
    permute_block(h, m, V, h->yperm.as<float>(), true, st);
    CK(cudaMemcpyAsync(V, h->yperm.p, (size_t)h->n * m * sizeof(float), cudaMemcpyDeviceToDevice, st));
}

sbmds_status create_impl(int64_t n, int64_t n_global, int64_t row0, int rank, int world, int64_t l, int64_t nnz,
                         const int64_t* row_ptr, const int32_t* col_idx, const float* val, const float* D_ll,
                         uint32_t flags, void* cuda_stream, sbmds_t* out, bool create_as_shard = false) {
    // (diagnostics) SBMDS_TRACE_CREATE=1: host-clock phase times of this create on stderr
    static const bool trace_create = getenv("SBMDS_TRACE_CREATE") != nullptr;
    const auto t_create0 = std::chrono::steady_clock::now();
    auto tphase = [&](const char* what) {
        nvtxMarkA(what);   // stage boundary on the NVTX timeline
        if (!trace_create) return;
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_create0).count();
        fprintf(stderr, "[sbmds_create] %8.2f ms  %s\n", ms, what);
    };

    Nvtx nv_create("sbmds_create");
    if (!out) return fail(SBMDS_EINVAL, "out is NULL");
    *out = nullptr;
    if (n < 1 || l < 1 || l > n_global)
        return fail(SBMDS_EINVAL, "need 1 <= l <= n (n=%lld, l=%lld)", (long long)n_global, (long long)l);
    if (nnz < 0 || nnz >= (int64_t(1) << 31)) return fail(SBMDS_EINVAL, "need 0 <= nnz < 2^31");
    if (n >= (int64_t(1) << 31) || l > 46340 * 4) return fail(SBMDS_EINVAL, "n or l too large");
    if (!row_ptr || !D_ll || (nnz > 0 && (!col_idx || !val))) return fail(SBMDS_EINVAL, "NULL input pointer");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
    sbmds_ctx* h = new sbmds_ctx();
    h->n = n;
    h->l = l;
    h->nnz = nnz;
    h->n_global = n_global;
    h->row0 = row0;
    h->rank = rank;
    h->world = world;
    h->shard = world > 1 || n_global != n || create_as_shard;
    cudaStream_t dside = nullptr;      // host-D upload stream (see below)
    cudaStream_t dabs = nullptr;       // max |D| of the landed strips, behind the upload
    std::vector<cudaEvent_t> dstrips;  // strip groups landed
    cudaEvent_t dside_done = nullptr;
    auto join_dside = [&]() {          // wait for and release it (idempotent; also on errors)
        if (dside) {
            cudaStreamSynchronize(dside);
            cudaStreamDestroy(dside);
            dside = nullptr;
        }
        if (dabs) {
            cudaStreamSynchronize(dabs);
            cudaStreamDestroy(dabs);
            dabs = nullptr;
        }
        for (auto e : dstrips) cudaEventDestroy(e);
        dstrips.clear();
        if (dside_done) {
            cudaEventDestroy(dside_done);
            dside_done = nullptr;
        }
    };
    try {
        CK(cudaGetDevice(&h->dev));
        CK(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->dev));
        install_hang_record();
        configure_pool_once();
        for_each_buf(h, [](DevBuf* b) { b->pooled = true; });
        const int64_t nz = std::max<int64_t>(nnz, 1);
        h->rp.ensure((n + 1) * sizeof(int32_t));
        h->col.ensure(nz * sizeof(int32_t));
        h->val.ensure(nz * sizeof(float));
        h->cptr.ensure((l + 1) * sizeof(int32_t));
        h->ridx.ensure(nz * sizeof(int32_t));
        h->cval.ensure(nz * sizeof(float));
        h->order.ensure(l * sizeof(int32_t));
        h->w.ensure(l * sizeof(double));
        h->colpart.ensure(4 * kRedBlocks * kMaxB * sizeof(double));
        h->tpart.ensure(kRedBlocks * kMaxB * sizeof(double));
        h->s.ensure(kMaxB * sizeof(double));
        h->t.ensure(kMaxB * sizeof(double));
        h->counters.ensure(kCounters * sizeof(unsigned int));
        CK(cudaMemsetAsync(h->counters.p, 0, h->counters.bytes, st));

        // S crosses the host link first (0.5 GB at config 4), then a host D (the bulk of create's
        // input) on an internal stream, so D's transfer overlaps C1/C2's kernels on `st` (which
        // need only S); `st` joins it below.
        // (temporaries from the stream-ordered pool: a cudaFree would synchronise the device and
        // wait for the D upload)
        DevBuf rp64{true}, tmpA{true}, tmpB{true}, tmpC{true}, flags_d{true};
        rp64.ensure((n + 1) * sizeof(int64_t));
        CK(cudaMemcpyAsync(rp64.p, row_ptr, (n + 1) * sizeof(int64_t), cudaMemcpyDefault, st));
        if (nnz > 0) {
            CK(cudaMemcpyAsync(h->col.p, col_idx, nnz * sizeof(int32_t), cudaMemcpyDefault, st));
            CK(cudaMemcpyAsync(h->val.p, val, nnz * sizeof(float), cudaMemcpyDefault, st));
        }
        const bool d_dev = is_device_ptr(D_ll);
        h->ldD = (l + 3) / 4 * 4;
        if (!d_dev) {
            h->Dbuf.ensure((size_t)l * h->ldD * sizeof(float));
            CK(cudaStreamCreateWithFlags(&dside, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&dside_done, cudaEventDisableTiming));
            CK(cudaEventRecord(dside_done, st));   // the device buffers above are ready and S has crossed
            CK(cudaStreamWaitEvent(dside, dside_done, 0));
            if (!(flags & SBMDS_VALIDATE)) {
                // only the block upper triangle crosses the host link (D is symmetric, R12; the
                // default D stream reads only these tiles): row strip I from column 128 I on;
                // the lower part is mirrored on the device if a full-D path is ever used.
                // Where the int8 symmetric-half stream will pack D (large l), max |D| over the
                // landed strips is taken on a third stream group by group, hidden behind the
                // transfer, and the packed copy is allocated here (both were first-eigs work).
                const bool pre8 = uses_sym(h, 16);
                unsigned int* dmax8 = nullptr;
                if (pre8) {
                    const int64_t NT = (l + 127) / 128;
                    h->Dt8.ensure((size_t)(NT * (NT + 1) / 2) * Sym8Cfg<16>::A_BYTES);
                    h->y16aux.ensure(352 * sizeof(unsigned int));
                    dmax8 = h->y16aux.as<unsigned int>() + 2;
                    CK(cudaMemsetAsync(dmax8, 0, sizeof(unsigned int), st));
                    h->dqhist.ensure(256 * sizeof(unsigned int));
                    CK(cudaMemsetAsync(h->dqhist.p, 0, 256 * sizeof(unsigned int), st));
                    CK(cudaStreamCreateWithFlags(&dabs, cudaStreamNonBlocking));
                    CK(cudaEventRecord(dside_done, st));
                    CK(cudaStreamWaitEvent(dabs, dside_done, 0));
                }
                constexpr int64_t kGroupRows = 16 * 128;
                for (int64_t r0 = 0; r0 < l; r0 += 128) {
                    const int64_t rows = std::min<int64_t>(128, l - r0);
                    CK(cudaMemcpy2DAsync(h->Dbuf.as<float>() + r0 * h->ldD + r0, h->ldD * sizeof(float),
                                         D_ll + r0 * l + r0, l * sizeof(float), (size_t)(l - r0) * sizeof(float),
                                         (size_t)rows, cudaMemcpyHostToDevice, dside));
                    h->h2d_bytes += rows * (l - r0) * (int64_t)sizeof(float);
                    if (pre8 && (r0 + 128 >= l || (r0 + 128) % kGroupRows == 0)) {
                        const int64_t g0 = r0 / kGroupRows * kGroupRows, g1 = std::min<int64_t>(l, r0 + 128);
                        cudaEvent_t ev;
                        CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                        dstrips.push_back(ev);
                        CK(cudaEventRecord(ev, dside));
                        CK(cudaStreamWaitEvent(dabs, ev, 0));
                        launch(k_absmax_upper, dim3((unsigned)std::min<int64_t>(4 * (int64_t)h->num_sms, g1 - g0)),
                               dim3(256), 0, dabs, (const float*)h->Dbuf.as<float>(), l, h->ldD, dmax8, g0, g1,
                               h->dqhist.as<unsigned int>());
                    }
                }
                if (pre8) {
                    cudaEvent_t ev;
                    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                    dstrips.push_back(ev);
                    CK(cudaEventRecord(ev, dabs));
                    CK(cudaStreamWaitEvent(dside, ev, 0));   // dside_done below covers the maxima too
                    h->dmax8_ok = true;
                    h->dq_hist_ok = true;
                }
                h->d_lower_missing = true;
            } else {
                CK(cudaMemcpy2DAsync(h->Dbuf.p, h->ldD * sizeof(float), D_ll, l * sizeof(float), l * sizeof(float), l,
                                     cudaMemcpyHostToDevice, dside));
                h->h2d_bytes += l * l * (int64_t)sizeof(float);
            }
            CK(cudaEventRecord(dside_done, dside));
            h->D = h->Dbuf.as<float>();
            h->own_D = true;
        }

        tphase("allocated, D upload issued");
        // ---- C1: check S's structure (uploaded above)
        flags_d.ensure(64);
        CK(cudaMemsetAsync(flags_d.p, 0, 64, st));
        int* bad = flags_d.as<int>();
        launch(k_rowptr_to_i32, dim3(256), dim3(256), 0, st, n, (const int64_t*)rp64.as<int64_t>(),
               h->rp.as<int32_t>(), nnz, bad);
        int hbad = 0;
        peek_to_host(&hbad, bad, sizeof(int), st);
        rp64.release();
        if (hbad) {
            join_dside(); destroy_ctx(h);
            return fail(SBMDS_EINVAL, "row_ptr must start at 0, be nondecreasing and end at nnz");
        }

        tphase("S uploaded and checked");
        // ---- C2: CSC (stable radix sort of (col, entry) pairs keeps rows ascending)
        if (nnz > 0) {
            tmpA.ensure(nnz * sizeof(int32_t));  // rowof
            launch(k_expand_rows, dim3(1024), dim3(256), 0, st, n, (const int32_t*)h->rp.as<int32_t>(),
                   (const int32_t*)h->col.as<int32_t>(), (const float*)h->val.as<float>(), l, tmpA.as<int32_t>(), bad);
            peek_to_host(&hbad, bad, sizeof(int), st);
            if (hbad) {
                join_dside(); destroy_ctx(h);
                return fail(SBMDS_EINVAL, "col_idx out of [0, l) or non-finite val");
            }
            if (!create_as_shard && (flags & SBMDS_REORDER_ROWS)) {
                reorder_rows(h, st);
                if (h->permuted)   // (the row of every entry, in the new order)
                    launch(k_expand_rows, dim3(1024), dim3(256), 0, st, n, (const int32_t*)h->rp.as<int32_t>(),
                           (const int32_t*)h->col.as<int32_t>(), (const float*)h->val.as<float>(), l,
                           tmpA.as<int32_t>(), bad);
                tphase("row order decided");
            }
            tmpB.ensure(2 * (size_t)nnz * sizeof(int32_t));  // iota | sorted perm
            tmpC.ensure((size_t)nnz * sizeof(int32_t));      // sorted keys
            int32_t* iota = tmpB.as<int32_t>();
            int32_t* perm = iota + nnz;
            launch(k_iota, dim3(1024), dim3(256), 0, st, (int32_t)nnz, iota);
            int end_bit = 1;
            while ((int64_t(1) << end_bit) <= l) ++end_bit;
            size_t tmp_bytes = 0;
            CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, h->col.as<int32_t>(), tmpC.as<int32_t>(), iota, perm,
                                               (int)nnz, 0, end_bit, st));
            DevBuf cubtmp{true};
            cubtmp.ensure(tmp_bytes + 16);
            CK(cub::DeviceRadixSort::SortPairs(cubtmp.p, tmp_bytes, h->col.as<int32_t>(), tmpC.as<int32_t>(), iota, perm,
                                               (int)nnz, 0, end_bit, st));
            g_launches.fetch_add(1);
            launch(k_gather_csc, dim3(1024), dim3(256), 0, st, (int32_t)nnz, (const int32_t*)perm,
                   (const int32_t*)tmpA.as<int32_t>(), (const float*)h->val.as<float>(), h->ridx.as<int32_t>(),
                   h->cval.as<float>());
            launch(k_col_ptr, dim3((unsigned)((l + 256) / 256)), dim3(256), 0, st, l, (int32_t)nnz,
                   (const int32_t*)tmpC.as<int32_t>(), h->cptr.as<int32_t>());
            CK(cudaStreamSynchronize(st));
            cubtmp.release();
            tphase("CSC built");
            build_blocked(h, tmpA.as<int32_t>(), st);
            tphase("row blocks built");
            // the tensor-core sparse step's S images depend on S only: built here, inside a host
            // D's upload window, instead of in the first eigs
            if (h->blocked && !d_dev) {
                ensure_sp8(h, st);
                tphase("sparse-step images built");
            }
        } else {
            CK(cudaMemsetAsync(h->cptr.p, 0, (l + 1) * sizeof(int32_t), st));
        }
        // w, column keys, spatial column order (sort columns by their median row)
        {
            DevBuf keys{true}, keys2{true}, ord0{true};
            keys.ensure(l * sizeof(int32_t));
            keys2.ensure(l * sizeof(int32_t));
            ord0.ensure(l * sizeof(int32_t));
            // (w = S^T 1 / n with the GLOBAL n: a shard's w_g = S_g^T 1 / n sums to w over the ranks)
            launch(k_colstats, dim3((unsigned)std::min<int64_t>(4096, (l + 7) / 8)), dim3(256), 0, st, l, n_global,
                   (const int32_t*)h->cptr.as<int32_t>(), (const int32_t*)h->ridx.as<int32_t>(),
                   (const float*)h->cval.as<float>(), h->w.as<double>(), keys.as<int32_t>());
            launch(k_iota, dim3(64), dim3(256), 0, st, (int32_t)l, ord0.as<int32_t>());
            int end_bit = 1;
            while ((int64_t(1) << end_bit) <= n) ++end_bit;
            size_t tmp_bytes = 0;
            CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.as<int32_t>(), keys2.as<int32_t>(),
                                               ord0.as<int32_t>(), h->order.as<int32_t>(), (int)l, 0, end_bit, st));
            DevBuf cubtmp{true};
            cubtmp.ensure(tmp_bytes + 16);
            CK(cub::DeviceRadixSort::SortPairs(cubtmp.p, tmp_bytes, keys.as<int32_t>(), keys2.as<int32_t>(),
                                               ord0.as<int32_t>(), h->order.as<int32_t>(), (int)l, 0, end_bit, st));
            g_launches.fetch_add(1);
            // rowsum deviation (diagnostic)
            DevBuf rs{true};
            rs.ensure(sizeof(unsigned long long));
            CK(cudaMemsetAsync(rs.p, 0, sizeof(unsigned long long), st));
            launch(k_rowsum_dev, dim3(1024), dim3(256), 0, st, n, (const int32_t*)h->rp.as<int32_t>(),
                   (const float*)h->val.as<float>(), rs.as<unsigned long long>());
            unsigned long long bits = 0;
            peek_to_host(&bits, rs.p, sizeof bits, st);
            double d;
            memcpy(&d, &bits, sizeof d);
            h->rowsum_dev = d;
        }
        tmpA.release();
        tmpB.release();
        tmpC.release();

        tphase("S side done");
        // the int8 D stream's schedule (host work) while D is still crossing the link
        PlanHost ph16;
        const bool pre_plan = h->dmax8_ok && !h->s8plan[1].ok;
        if (pre_plan) ph16 = plan_host(l, h->num_sms, Sym8Cfg<16>::SR, Sym8Cfg<16>::GN, true, h->rank, h->world, Sym8Cfg<16>::SC);
        // ---- D_ll: borrow (device, l % 4 == 0), copy a device D into a 16-byte-pitched buffer, or
        // join the host upload started above
        if (!d_dev) {
            CK(cudaStreamWaitEvent(st, dside_done, 0));
        } else if ((flags & SBMDS_BORROW_D) && h->ldD == l && (reinterpret_cast<uintptr_t>(D_ll) & 15) == 0) {
            h->D = const_cast<float*>(D_ll);
            h->d_borrowed = true;
        } else {
            h->Dbuf.ensure((size_t)l * h->ldD * sizeof(float));
            CK(cudaMemcpy2DAsync(h->Dbuf.p, h->ldD * sizeof(float), D_ll, l * sizeof(float), l * sizeof(float), l,
                                 cudaMemcpyDeviceToDevice, st));
            h->D = h->Dbuf.as<float>();
            h->own_D = true;
        }
        if (flags & SBMDS_VALIDATE) {
            DevBuf cb{true};
            cb.ensure(64);
            CK(cudaMemsetAsync(cb.p, 0, 64, st));
            unsigned int* md = cb.as<unsigned int>();
            const unsigned tiles = (unsigned)((l + 31) / 32);
            launch(k_check_sym, dim3(tiles, tiles), dim3(256), 0, st, l, h->ldD, (const float*)h->D, md, md + 1,
                   reinterpret_cast<int*>(md + 2));
            unsigned int hv[3];
            CK(cudaMemcpyAsync(hv, md, sizeof hv, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            float mdiff, mabs;
            memcpy(&mdiff, &hv[0], 4);
            memcpy(&mabs, &hv[1], 4);
            if (hv[2]) {
                join_dside(); destroy_ctx(h);
                return fail(SBMDS_EINVAL, "D_ll has non-finite entries");
            }
            if (mdiff > 1e-6f * mabs) {
                join_dside(); destroy_ctx(h);
                return fail(SBMDS_EINVAL, "D_ll not symmetric: max|D-D^T| = %g, max|D| = %g", mdiff, mabs);
            }
        }
        CK(cudaStreamSynchronize(st));
        tphase("S-side stream idle");
        join_dside();
        tphase("D upload joined");
        if (pre_plan) {
            dq_decide(h, st);   // the int8 stream's precision check (max |D| vs the median)
            if (h->dq_state < 0) h->Dt8.release();
        }
        if (pre_plan && h->dq_state > 0) {
            // D and max |D| have landed: upload the schedule and pack D (int8 digits of the
            // upper tiles) on a handle stream that runs on past create's return; the first
            // D-stream launch waits for it
            using C8 = Sym8Cfg<16>;
            auto& pl = h->s8plan[1];
            build_pair_plan(h, pl, h->num_sms, C8::SR, C8::GN, true, &ph16, C8::SC);
            h->Dt8.ensure((size_t)((int64_t)pl.NT * (pl.NT + 1) / 2) * C8::A_BYTES);
            unsigned int* aux = h->y16aux.as<unsigned int>();
            CK(cudaStreamCreateWithFlags(&h->pack_st, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&h->pack_ev, cudaEventDisableTiming));
            launch(k_pack_sym8, dim3((unsigned)std::min<int64_t>(pl.ntiles, 16 * (int64_t)h->num_sms)), dim3(256), 0,
                   h->pack_st, (const float*)h->D, h->ldD, h->l, (const uint32_t*)pl.tiles.p, (int64_t)pl.NT, pl.ntiles,
                   (const unsigned int*)(aux + 2), reinterpret_cast<int*>(aux + 3), h->Dt8.as<int8_t>());
            CK(cudaEventRecord(h->pack_ev, h->pack_st));
            h->dt8_ok = true;
            h->pack_pending = true;
            tphase("D pack issued");
        }
    } catch (const CudaError& e) {
        join_dside(); destroy_ctx(h);
        if (e.e == cudaErrorMemoryAllocation) return fail(SBMDS_ENOMEM, "device allocation failed (%s)", e.what);
        return fail(SBMDS_ECUDA, "%s: %s%s", e.what, cudaGetErrorString(e.e), hang_note().c_str());
    }
    *out = h;
    return SBMDS_OK;
}
}  // namespace

extern "C" sbmds_status sbmds_create(int64_t n, int64_t l, int64_t nnz, const int64_t* row_ptr,
                                     const int32_t* col_idx, const float* val, const float* D_ll, uint32_t flags,
                                     void* cuda_stream, sbmds_t* out) {
    return create_impl(n, n, 0, 0, 1, l, nnz, row_ptr, col_idx, val, D_ll, flags, cuda_stream, out);
}

extern "C" sbmds_status sbmds_create_shard(int64_t n_global, int64_t row0, int64_t n_local, int64_t l, int64_t nnz,
                                           const int64_t* row_ptr, const int32_t* col_idx, const float* val,
                                           const float* D_ll, int32_t rank, int32_t world, uint32_t flags,
                                           void* cuda_stream, sbmds_t* out) {
    if (out) *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) return fail(SBMDS_EINVAL, "need 0 <= rank < world");
    if (n_local < 1 || row0 < 0 || row0 + n_local > n_global)
        return fail(SBMDS_EINVAL, "need 0 <= row0, 1 <= n_local, row0 + n_local <= n_global");
    return create_impl(n_local, n_global, row0, rank, world, l, nnz, row_ptr, col_idx, val, D_ll, flags, cuda_stream,
                       out, true);
}

extern "C" void sbmds_destroy(sbmds_t h) {
    if (!h) return;
    DevGuard g(h->dev);
    cudaDeviceSynchronize();
    destroy_ctx(h);
}

extern "C" const char* sbmds_last_error(void) { return t_err.c_str(); }
extern "C" int64_t sbmds_launch_count(void) { return g_launches.load(); }
extern "C" int32_t sbmds_abi_version(void) { return 2; }

// ============================================================================ apply
static bool overlap(const void* a, size_t na, const void* b, size_t nb) {
    const char* x = (const char*)a;
    const char* y = (const char*)b;
    return x < y + nb && y < x + na;
}

namespace {
void shard_stage_dev(sbmds_ctx* h, int stage, int b, const float* X, const void* exch_in, void* exch_out,
                     float* Y, cudaStream_t st);
void shard_apply_nccl(sbmds_ctx* h, int b, const float* X, float* Y, cudaStream_t st);
}  // namespace

extern "C" sbmds_status sbmds_apply(sbmds_t h, int32_t b, const float* X, float* Y, void* cuda_stream) {
    Nvtx nv_apply("sbmds_apply");
    if (!h) return fail(SBMDS_EINVAL, "NULL handle");
    if (b < 1 || b > kMaxB) return fail(SBMDS_EINVAL, "need 1 <= b <= 64 (b=%d)", b);
    if (!X || !Y) return fail(SBMDS_EINVAL, "NULL X or Y");
    const size_t bytes = (size_t)h->n * b * sizeof(float);
    if (overlap(X, bytes, Y, bytes)) return fail(SBMDS_EINVAL, "X and Y overlap");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
    DevGuard g(h->dev);
    try {
        const bool xd = is_device_ptr(X), yd = is_device_ptr(Y);
        const float* Xd = X;
        float* Yd = Y;
        if (!xd) {
            h->xhost.ensure(bytes);
            CK(cudaMemcpyAsync(h->xhost.p, X, bytes, cudaMemcpyHostToDevice, st));
            Xd = h->xhost.as<float>();
        }
        if (!yd) {
            h->yhost.ensure(bytes);
            Yd = h->yhost.as<float>();
        }
        ensure_dq(h, st);   // the int8 stream's precision check (once per handle)
        float* Yuser = Yd;
        if (h->permuted) {   // caller's row order -> the handle's (and back below)
            h->xperm.ensure(bytes);
            h->yperm.ensure(bytes);
            permute_block(h, b, Xd, h->xperm.as<float>(), false, st);
            Xd = h->xperm.as<float>();
            Yd = h->yperm.as<float>();
        }
        if (h->shard) {
            if (!h->center) return fail(SBMDS_EINVAL, "a shard handle applies the centred operator only");
            if (h->comm) shard_apply_nccl(h, b, Xd, Yd, st);
            else if (h->world == 1) for (int sg = 0; sg < 4; ++sg) shard_stage_dev(h, sg, b, Xd, nullptr, nullptr, Yd, st);
            else return fail(SBMDS_EINVAL, "shard handle (world %d): attach NCCL or drive sbmds_shard_stage", h->world);
        } else if (h->center) {
            apply_device(h, b, Xd, Yd, st);
        } else {
            // uncentred E^ X = S D S^T X: the centred machinery with s = 0 and w = 0 (both rank-one
            // terms vanish) and R^-1 = -2 I folded into Y1 (cancels the -1/2; exact)
            h->w0.ensure((size_t)h->l * sizeof(double));
            h->rawR.ensure((size_t)kMaxB * kMaxB * sizeof(double));
            std::vector<double> m2((size_t)b * b, 0.0);
            for (int c = 0; c < b; ++c) m2[(size_t)c * b + c] = -2.0;
            CK(cudaMemsetAsync(h->w0.p, 0, (size_t)h->l * sizeof(double), st));
            CK(cudaMemcpyAsync(h->rawR.p, m2.data(), m2.size() * sizeof(double), cudaMemcpyHostToDevice, st));
            CK(cudaMemsetAsync(h->s.p, 0, kMaxB * sizeof(double), st));
            h->raw_now = true;
            try {
                apply_device(h, b, Xd, Yd, st, true, h->rawR.as<double>());
            } catch (...) {
                h->raw_now = false;
                throw;
            }
            h->raw_now = false;
            CK(cudaStreamSynchronize(st));   // m2 (host) must outlive its copy
        }
        if (h->permuted) permute_block(h, b, Yd, Yuser, true, st);
        if (!yd) CK(cudaMemcpyAsync(Y, Yuser, bytes, cudaMemcpyDeviceToHost, st));
        if (!xd || !yd) CK(cudaStreamSynchronize(st));
    } catch (const CudaError& e) {
        if (e.e == cudaErrorMemoryAllocation) return fail(SBMDS_ENOMEM, "device allocation failed (%s)", e.what);
        return fail(SBMDS_ECUDA, "%s: %s%s", e.what, cudaGetErrorString(e.e), hang_note().c_str());
    } catch (const NcclError& e) {
        return fail(SBMDS_ECUDA, "%s: %s", e.what, nccl_api().errorString(e.r));
    }
    return SBMDS_OK;
}

// ============================================================================ sharded apply
// rank g holds rows R_g of S (CSR S_g and its CSC copy) and streams tile range g
// of D's upper triangle. The apply is linear in every exchanged quantity, so each rank forms
// partials and a sum over ranks completes them (PAPER.md:221-222's matvec, split by rows of P
// and by tiles of W):
//   stage 0  s_g  = 1^T X_g                                   -> sum: s = 1^T X
//   stage 1  Y1_g = S_g^T X_g - w_g s^T,  w_g = S_g^T 1 / n    -> sum: Y1 = S^T X - w s^T
//   stage 2  Y2_g = sum over my tiles of D_IJ Y1_J (+ D_IJ^T Y1_I), t_g = (D w_g)^T Y1
//                                                               -> sum: Y2 = D Y1, t = w^T D Y1 = w^T Y2
//   stage 3  Y_g  = -1/2 (S_g Y2 - 1 t^T)                       (local rows, no exchange)
// With an NCCL communicator attached, sbmds_apply runs the stages with in-library allreduces
// on the call's stream; without one, the caller drives sbmds_shard_stage and sums the
// exchange buffers itself. Full-D paths (FFMA, 3xTF32: b < 5, or the precision fallback) are
// not tiled by rank: rank 0 streams all of D and the other ranks contribute zero partials.
namespace {

// out = v_g^T Y1 (b values): block partials + a fixed-order sum
void vdot(sbmds_ctx* h, int b, int bp, double* out, cudaStream_t st) {
    h->vdpart.ensure((size_t)kVdotBlocks * 64 * sizeof(double));
    launch(k_vdot, dim3(kVdotBlocks), dim3(256), 0, st, h->l, b, bp, (const double*)h->vg.as<double>(),
           (const float*)h->Y1.as<float>(), h->vdpart.as<double>());
    launch(k_vdot_sum, dim3(1), dim3(64), 0, st, kVdotBlocks, b, (const double*)h->vdpart.as<double>(), out);
}

int64_t exch_t_offset(int64_t l, int b) { return ((int64_t)4 * l * b + 7) / 8 * 8; }

// One stage on device buffers; the compact exchange layouts are those of sbmds_shard_stage.
// exch_in / exch_out may be null (the NCCL path works on the internal buffers directly).
void shard_stage_dev(sbmds_ctx* h, int stage, int b, const float* X, const void* exch_in, void* exch_out,
                     float* Y, cudaStream_t st) {
    const int bp = next_pow2(b);
    ensure_apply_ws(h, bp);
    const int64_t l = h->l;
    if (stage == 0) {
        colsum(h, b, X, st);
        if (exch_out) CK(cudaMemcpyAsync(exch_out, h->s.p, (size_t)b * sizeof(double), cudaMemcpyDeviceToDevice, st));
    } else if (stage == 1) {
        if (exch_in) CK(cudaMemcpyAsync(h->s.p, exch_in, (size_t)b * sizeof(double), cudaMemcpyDeviceToDevice, st));
        spmm_csc(h, b, bp, X, st);
        if (exch_out)
            CK(cudaMemcpy2DAsync(exch_out, (size_t)b * 4, h->Y1.p, (size_t)bp * 4, (size_t)b * 4, l,
                                 cudaMemcpyDeviceToDevice, st));
    } else if (stage == 2) {
        if (exch_in)
            CK(cudaMemcpy2DAsync(h->Y1.p, (size_t)bp * 4, exch_in, (size_t)b * 4, (size_t)b * 4, l,
                                 cudaMemcpyDeviceToDevice, st));
        if (h->dstream == 0 && h->dy_max_range < 64 && takes_sym(h, bp, false))
            ycheck(h, b, bp, st);   // (same Y1, same decision on every rank)
        if (takes_sym(h, bp, false) || h->rank == 0) {
            dstream(h, b, bp, st, nullptr);
        } else {   // full-D paths are not tiled: rank 0 owns all of D Y1
            CK(cudaMemsetAsync(h->Y2.p, 0, (size_t)l * bp * sizeof(float), st));
            CK(cudaMemsetAsync(h->t.p, 0, (size_t)b * sizeof(double), st));
        }
        h->y_fallback = false;
        // t_g: the reduce formed w_g^T (this rank's Y2 part); the plan needs sum_g t_g = w^T Y2 =
        // sum_g (D w_g)^T Y1 with the full Y1 every rank holds: overwrite t with v_g^T Y1
        if (!h->vg_ok) {
            ensure_full_d(h, st);
            h->vg.ensure((size_t)l * sizeof(double));
            launch(k_symv_rows, dim3((unsigned)std::min<int64_t>(8 * (int64_t)h->num_sms, (l + 7) / 8)), dim3(256), 0,
                   st, l, (const float*)h->D, h->ldD, (const double*)h->w.as<double>(), h->vg.as<double>());
            h->vg_ok = true;
        }
        vdot(h, b, bp, h->t.as<double>(), st);
        if (exch_out) {
            CK(cudaMemcpy2DAsync(exch_out, (size_t)b * 4, h->Y2.p, (size_t)bp * 4, (size_t)b * 4, l,
                                 cudaMemcpyDeviceToDevice, st));
            CK(cudaMemcpyAsync((char*)exch_out + exch_t_offset(l, b), h->t.p, (size_t)b * sizeof(double),
                               cudaMemcpyDeviceToDevice, st));
        }
    } else {
        if (exch_in) {
            CK(cudaMemcpy2DAsync(h->Y2.p, (size_t)bp * 4, exch_in, (size_t)b * 4, (size_t)b * 4, l,
                                 cudaMemcpyDeviceToDevice, st));
            CK(cudaMemcpyAsync(h->t.p, (const char*)exch_in + exch_t_offset(l, b), (size_t)b * sizeof(double),
                               cudaMemcpyDeviceToDevice, st));
        }
        spmm_csr(h, b, bp, Y, st);
    }
}

// The four stages with NCCL sums in between (sbmds_apply on a handle with a communicator).
void shard_apply_nccl(sbmds_ctx* h, int b, const float* X, float* Y, cudaStream_t st) {
    const NcclApi& nc = nccl_api();
    ncclComm_t comm = reinterpret_cast<ncclComm_t>(h->comm);
    const int bp = next_pow2(b);
    shard_stage_dev(h, 0, b, X, nullptr, nullptr, nullptr, st);
    NK(nc.allReduce(h->s.p, h->s.p, (size_t)b, ncclFloat64, ncclSum, comm, st));
    shard_stage_dev(h, 1, b, X, nullptr, nullptr, nullptr, st);
    NK(nc.allReduce(h->Y1.p, h->Y1.p, (size_t)h->l * bp, ncclFloat32, ncclSum, comm, st));
    shard_stage_dev(h, 2, b, nullptr, nullptr, nullptr, nullptr, st);
    NK(nc.groupStart());
    NK(nc.allReduce(h->Y2.p, h->Y2.p, (size_t)h->l * bp, ncclFloat32, ncclSum, comm, st));
    NK(nc.allReduce(h->t.p, h->t.p, (size_t)b, ncclFloat64, ncclSum, comm, st));
    NK(nc.groupEnd());
    shard_stage_dev(h, 3, b, nullptr, nullptr, nullptr, Y, st);
}

}  // namespace

extern "C" int64_t sbmds_shard_exchange_bytes(int64_t l, int32_t b, int32_t stage) {
    if (l < 1 || b < 1 || b > kMaxB) return -1;
    switch (stage) {
        case 0: return (int64_t)b * 8;                       // out: s_g
        case 1: return (int64_t)4 * l * b;                   // out: Y1_g (in: s)
        case 2: return exch_t_offset(l, b) + (int64_t)8 * b;  // out: Y2_g | t_g (in: Y1)
        case 3: return exch_t_offset(l, b) + (int64_t)8 * b;  // in: Y2 | t
        default: return -1;
    }
}

extern "C" sbmds_status sbmds_shard_stage(sbmds_t h, int32_t stage, int32_t b, const float* X, const void* exch_in,
                                          void* exch_out, float* Y, void* cuda_stream) {
    Nvtx nv("sbmds_shard_stage");
    if (!h) return fail(SBMDS_EINVAL, "NULL handle");
    if (b < 1 || b > kMaxB) return fail(SBMDS_EINVAL, "need 1 <= b <= 64 (b=%d)", b);
    if (stage < 0 || stage > 3) return fail(SBMDS_EINVAL, "stage in 0..3");
    const bool need_x = stage <= 1, need_in = stage >= 1, need_out = stage <= 2, need_y = stage == 3;
    if ((need_x && !X) || (need_in && !exch_in) || (need_out && !exch_out) || (need_y && !Y))
        return fail(SBMDS_EINVAL, "stage %d: NULL buffer", stage);
    for (const void* p : {(const void*)X, exch_in, (const void*)exch_out, (const void*)Y})
        if (p && !is_device_ptr(p)) return fail(SBMDS_EINVAL, "sbmds_shard_stage takes device buffers only");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
    DevGuard g(h->dev);
    try {
        ensure_dq(h, st);
        shard_stage_dev(h, stage, b, X, exch_in, exch_out, Y, st);
    } catch (const CudaError& e) {
        if (e.e == cudaErrorMemoryAllocation) return fail(SBMDS_ENOMEM, "device allocation failed (%s)", e.what);
        return fail(SBMDS_ECUDA, "%s: %s%s", e.what, cudaGetErrorString(e.e), hang_note().c_str());
    }
    return SBMDS_OK;
}

extern "C" sbmds_status sbmds_nccl_unique_id(void* id_out) {
    if (!id_out) return fail(SBMDS_EINVAL, "NULL id");
    const NcclApi& nc = nccl_api();
    if (!nc.ok) return fail(SBMDS_ECUDA, "NCCL unavailable: %s", nc.why.c_str());
    ncclUniqueId id;
    const ncclResult_t r = nc.getUniqueId(&id);
    if (r != ncclSuccess) return fail(SBMDS_ECUDA, "ncclGetUniqueId: %s", nc.errorString(r));
    memcpy(id_out, &id, sizeof id);
    return SBMDS_OK;
}

extern "C" sbmds_status sbmds_shard_attach_nccl(sbmds_t h, const void* unique_id) {
    if (!h || !unique_id) return fail(SBMDS_EINVAL, "NULL handle or id");
    if (h->comm) return fail(SBMDS_EINVAL, "a communicator is already attached");
    const NcclApi& nc = nccl_api();
    if (!nc.ok) return fail(SBMDS_ECUDA, "NCCL unavailable: %s", nc.why.c_str());
    DevGuard g(h->dev);
    ncclUniqueId id;
    memcpy(&id, unique_id, sizeof id);
    ncclComm_t comm = nullptr;
    const ncclResult_t r = nc.commInitRank(&comm, h->world, id, h->rank);   // collective over the ranks
    if (r != ncclSuccess) return fail(SBMDS_ECUDA, "ncclCommInitRank: %s", nc.errorString(r));
    h->comm = comm;
    return SBMDS_OK;
}

// ============================================================================ eigs
namespace {

// G = Y^T Y, s = 1^T Y (into h->s when want_s), and H = X^T Y when X != null.
void gram(sbmds_ctx* h, int b, const float* Y, const float* X, cudaStream_t st, bool want_s = false) {
    h->gpart.ensure((size_t)kRedBlocks * kGramPart * sizeof(double));
    double* cs = want_s ? h->s.as<double>() : nullptr;
    smem_attr(k_gram<true>, 80 * 1024);
    smem_attr(k_gram<false>, 80 * 1024);
    const size_t smem = gram_smem_bytes(b);
    double* Hd = h->H.as<double>();
    double* Gd = h->G.as<double>();
    double* P = h->gpart.as<double>();
    // b > 16: the block partials are summed by k_gram_sum (several blocks) instead of the last block
    const bool two_level = h->gram_tc && b > 16 && b <= 32;
    unsigned int* cnt = two_level ? nullptr : h->counters.as<unsigned int>() + CNT_GRAM;
    smem_attr(k_gram_tc<4, true>, (int)gram_tc_smem<4>());
    smem_attr(k_gram_tc<4, false>, (int)gram_tc_smem<4>());
    smem_attr(k_gram_tc<2, true>, (int)gram_tc_smem<2>());   // (48 KB of row staging + the kernel's static 1 KB)
    smem_attr(k_gram_tc<2, false>, (int)gram_tc_smem<2>());
    const size_t smem_tc = b <= 8 ? gram_tc_smem<1>() : (b <= 16 ? gram_tc_smem<2>() : gram_tc_smem<4>());
    auto tc = [&](auto kern) {
        launch(kern, dim3(kRedBlocks), dim3(256), smem_tc, st, h->n, b, Y, X, P, Gd, Hd, cs, cnt);
    };
    profiled(h->prof, PK_GRAM, st, [&] {
        if (h->gram_tc && b <= 32 && b > 4) {   // FP64 tensor cores (DMMA m8n8k4); b <= 4 (the orthogonality check of V): k_gram
            const int ncb = (b + 7) / 8;
            if (X) {
                if (ncb == 1) tc(k_gram_tc<1, true>);
                else if (ncb == 2) tc(k_gram_tc<2, true>);
                else tc(k_gram_tc<4, true>);
            } else {
                if (ncb == 1) tc(k_gram_tc<1, false>);
                else if (ncb == 2) tc(k_gram_tc<2, false>);
                else tc(k_gram_tc<4, false>);
            }
            if (two_level) {
                const int ent = b * b * (X ? 2 : 1) + (cs ? b : 0);
                launch(k_gram_sum, dim3((unsigned)((4 * ent + 255) / 256)), dim3(256), 0, st, b, kRedBlocks, (const double*)P,
                       Gd, X ? Hd : (double*)nullptr, cs);
            }
        } else if (X) {
            launch(k_gram<true>, dim3(kRedBlocks), dim3(256), smem, st, h->n, b, Y, X, P, Gd, Hd, cs, cnt);
        } else {
            launch(k_gram<false>, dim3(kRedBlocks), dim3(256), smem, st, h->n, b, Y, (const float*)nullptr, P, Gd,
                   (double*)nullptr, cs, cnt);
        }
    });
}

// out = in * M (+ addc), optionally s = 1^T out.
void rotate(sbmds_ctx* h, int b, int mo, int ldm, const float* in, const double* M, float* out, const double* addc,
            bool colsum, cudaStream_t st) {
    const int grid = (int)std::min<int64_t>(2 * 148, (h->n + 255) / 256);
    double* cp = colsum ? h->colpart.as<double>() : nullptr;
    double* co = colsum ? h->s.as<double>() : nullptr;
    unsigned int* cnt = h->counters.as<unsigned int>() + CNT_ROTATE;
    auto go = [&](auto kern) { launch(kern, dim3(grid), dim3(256), 0, st, h->n, b, mo, ldm, in, M, out, addc, cp, co, cnt); };
    profiled(h->prof, PK_ROTATE, st, [&] {
        if (b <= 4) go(k_rotate<4>);
        else if (b <= 8) go(k_rotate<8>);
        else if (b <= 16) { if (mo <= 4) go(k_rotate<16, 4>); else go(k_rotate<16>); }
        else if (b <= 32) { if (mo <= 4) go(k_rotate<32, 4>); else go(k_rotate<32>); }
        else go(k_rotate<64>);
    });
}

// R^-1 from G = Y^T Y = R^T R (status read later). The orthonormal X = Y R^-1 is never
// formed: the next apply folds R^-1 into its l x b stage.
// G = R^T R -> Rinv (b x b): the warp form up to b = 16 (also run inside the sparse step and
// the fold), the block-parallel one above
void chol_launch(int b, const double* G, double* Rinv, int* status, cudaStream_t st) {
    if (b <= 16) {
        launch(k_chol, dim3(1), dim3(256), 0, st, b, G, Rinv, status);
    } else {
        smem_attr(k_chol_par, kCholParSmem);
        launch(k_chol_par, dim3(1), dim3(256), (size_t)kCholParSmem, st, b, G, Rinv, status);
    }
}

void chol(sbmds_ctx* h, int b, cudaStream_t st) {
    profiled(h->prof, PK_CHOL, st, [&] {
        chol_launch(b, (const double*)h->G.as<double>(), h->Rinv.as<double>(), h->status.as<int>(), st);
    });
}

}  // namespace

// ---------------------------------------------------------------------------- NEXT-3: block Lanczos
// Restarted block Lanczos with full reorthogonalisation ("uses the Lanczos method";
// SPEC.md:52 full reorthogonalisation), block size b, k blocks per cycle (k b <= 64):
//   Q_0 = orth(X0); for j < k: W = B~ Q_j; CGS2 against Q_0..Q_j (coefficients -> T's column
//   block j); j < k-1: W = Q_{j+1} R_j (Cholesky-QR, R_j -> T's subdiagonal block);
//   Rayleigh-Ritz on T (k_rr, the residual ||B~y - θy|| = ||R_k E^T u|| from Gl = T T + E G_W E^T);
//   restart from the top b Ritz vectors. Every step on the device; the host reads one flag per cycle.
// Returns the number of applies; eigvals / V / Z / info as sbmds_eigs.
struct LanczosBreakdown {
    const char* what;
};

int eigs_lanczos(sbmds_ctx* h, int m, int b, int max_iters, double tol, uint64_t seed, const float* X0, double* eigvals,
                 float* V, float* Z, sbmds_info* info, cudaStream_t st, bool* converged_out) {
    const int64_t n = h->n;
    const int k = std::max(2, std::min(h->lz_blocks > 0 ? h->lz_blocks : kLzMaxKB / b, kLzMaxKB / b));
    const int kb = k * b;
    if (kb > kLzMaxKB || k < 2) throw CudaError{cudaErrorInvalidValue, "block Lanczos needs 2 blocks of b <= 32"};
    h->lzQ.ensure((size_t)k * n * b * sizeof(float));
    h->lzW.ensure((size_t)n * b * sizeof(float));
    h->lzC.ensure((size_t)kLzMaxKB * kMaxB * sizeof(double));
    h->lzT.ensure((size_t)kLzMaxKB * kLzMaxKB * sizeof(double));
    h->lzGl.ensure((size_t)kLzMaxKB * kLzMaxKB * sizeof(double));
    h->lzI.ensure((size_t)kLzMaxKB * kLzMaxKB * sizeof(double));
    h->lzR.ensure((size_t)kMaxB * kMaxB * sizeof(double));
    h->X.ensure((size_t)n * b * sizeof(float));
    float* Q = h->lzQ.as<float>();
    float* W = h->lzW.as<float>();
    float* tmp = h->X.as<float>();
    double* C = h->lzC.as<double>();
    double* T = h->lzT.as<double>();
    auto Qj = [&](int j) { return Q + (size_t)j * n * b; };
    const int grid = (int)std::min<int64_t>(4 * 148, (n + 255) / 256);
    auto combine = [&](int nq, int mo, int ldm, const double* M, const float* in0, double alpha, float* out) {
        auto go = [&](auto kern) {
            launch(kern, dim3(grid), dim3(256), 0, st, n, b, nq, (const float*)Q, mo, ldm, M, in0, alpha, out);
        };
        if (mo <= 4) go(k_combine<4>);
        else if (mo <= 8) go(k_combine<8>);
        else if (mo <= 16) go(k_combine<16>);
        else go(k_combine<32>);
    };
    auto cholqr = [&](const float* in, float* out, double* Rout) {   // out R = in (out may alias in)
        gram(h, b, in, nullptr, st);
        launch(k_chol_r, dim3(1), dim3(256), 0, st, b, (const double*)h->G.as<double>(), h->Rinv.as<double>(),
               h->status.as<int>(), Rout);
        rotate(h, b, b, b, in, (const double*)h->Rinv.as<double>(), out, (const double*)nullptr, false, st);
    };
    auto check_breakdown = [&](const char* where) {
        int hs = 0;
        CK(cudaMemcpyAsync(&hs, h->status.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (hs == 2) throw LanczosBreakdown{where};
    };
    // Q_0 = orth(X0) (Cholesky-QR twice)
    if (X0) {
        CK(cudaMemcpyAsync(W, X0, (size_t)n * b * sizeof(float), cudaMemcpyDefault, st));
        if (h->permuted) {
            h->xperm.ensure((size_t)n * b * sizeof(float));
            CK(cudaMemcpyAsync(h->xperm.p, W, (size_t)n * b * sizeof(float), cudaMemcpyDeviceToDevice, st));
            permute_block(h, b, h->xperm.as<float>(), W, false, st);
        }
    }
    else launch(k_init_philox, dim3(4 * 148), dim3(256), 0, st, n, b, seed, W, (int64_t)0);
    cholqr(W, tmp, h->lzR.as<double>());
    cholqr(tmp, Qj(0), h->lzR.as<double>());
    check_breakdown("Cholesky-QR of the initial block broke down");
    smem_attr(k_rr, kRrSmem);
    int applies = 0;
    bool converged = false;
    for (;;) {
        CK(cudaMemsetAsync(T, 0, (size_t)kb * kb * sizeof(double), st));
        for (int j = 0; j < k; ++j) {
            apply_device(h, b, Qj(j), W, st);   // W = B~ Q_j (A1-A5)
            ++applies;
            for (int pass = 0; pass < 2; ++pass) {   // CGS2: W -= Q_{0..j} (Q_{0..j}^T W)
                for (int i = 0; i <= j; ++i) {
                    gram(h, b, W, Qj(i), st);        // H = Q_i^T W
                    CK(cudaMemcpyAsync(C + (size_t)i * b * b, h->H.p, (size_t)b * b * sizeof(double),
                                       cudaMemcpyDeviceToDevice, st));
                    launch(k_tadd, dim3(1), dim3(256), 0, st, b, kb, i, j, (const double*)h->H.as<double>(), T, 0);
                }
                combine(j + 1, b, b, C, W, -1.0, W);
            }
            if (j < k - 1) {   // W = Q_{j+1} R_j
                cholqr(W, Qj(j + 1), h->lzR.as<double>());
                // T[j+1][j] = R_j (T[j][j+1] ~ R_j^T comes from step j+1's CGS coefficients)
                launch(k_tadd, dim3(1), dim3(256), 0, st, b, kb, j + 1, j, (const double*)h->lzR.as<double>(), T, 0);
            } else {   // the residual block: G_W = R_k^T R_k (for Gl) and R_k itself
                gram(h, b, W, nullptr, st);
                launch(k_chol_r, dim3(1), dim3(256), 0, st, b, (const double*)h->G.as<double>(), h->Rinv2.as<double>(),
                       h->status.as<int>() + 1, h->lzR.as<double>());
            }
        }
        launch(k_lanczos_prep, dim3(1), dim3(256), 0, st, kb, b, T, (const double*)h->G.as<double>(),
               h->lzGl.as<double>(), h->lzI.as<double>());
        launch(k_rr, dim3(1), dim3(256), (size_t)kRrSmem, st, kb, m, tol, (const double*)T,
               (const double*)h->lzGl.as<double>(), (const double*)h->lzI.as<double>(), h->rr.as<RrOut>());
        launch(k_lanczos_resid, dim3(1), dim3(64), 0, st, kb, b, m, tol, (const double*)h->lzR.as<double>(),
               h->rr.as<RrOut>());
        int conv = 0;
        CK(cudaMemcpyAsync(&conv, &h->rr.as<RrOut>()->converged, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        check_breakdown("Cholesky-QR broke down in block Lanczos");
        if ((conv && tol > 0.0) || applies + k > max_iters) {
            converged = conv != 0 && tol > 0.0;
            break;
        }
        // restart from the top b Ritz vectors (orthonormal: Q orthonormal, U orthogonal)
        const double* U = h->rr.as<RrOut>()->U;
        combine(k, b, kb, U, nullptr, 1.0, tmp);
        cholqr(tmp, Qj(0), h->lzR.as<double>());   // re-orthonormalise against drift
    }
    RrOut rr_host;
    CK(cudaMemcpyAsync(&rr_host, h->rr.p, sizeof(RrOut), cudaMemcpyDeviceToHost, st));
    // E6: V = Q U[:, :m] (top-m algebraic Ritz vectors), signs, Z
    const bool vdev = V && is_device_ptr(V), zdev = Z && is_device_ptr(Z);
    const size_t vbytes = (size_t)n * m * sizeof(float);
    float* Vd = vdev ? V : (h->vtmp.ensure(vbytes), h->vtmp.as<float>());
    float* Zd = zdev ? Z : (Z ? (h->ztmp.ensure(vbytes), h->ztmp.as<float>()) : nullptr);
    combine(k, m, kb, h->rr.as<RrOut>()->U, nullptr, 1.0, Vd);
    unpermute_v(h, m, Vd, st);
    h->sign.ensure(kMaxB * sizeof(float));
    h->apval.ensure(kRedBlocks * kMaxB * sizeof(float));
    h->apidx.ensure(kRedBlocks * kMaxB * sizeof(long long));
    launch(k_col_argmax, dim3(kRedBlocks), dim3(256), 0, st, n, m, (const float*)Vd, h->apval.as<float>(),
           h->apidx.as<long long>(), h->sign.as<float>(), h->counters.as<unsigned int>() + CNT_ARGMAX);
    const double* theta = h->rr.as<RrOut>()->theta;
    launch(k_finalize, dim3((unsigned)std::min<int64_t>(4 * 148, (n * m + 255) / 256)), dim3(256), 0, st, n, m,
           (const float*)h->sign.as<float>(), theta, Vd, Zd);
    gram(h, m, Vd, nullptr, st);
    std::vector<double> gv((size_t)m * m);
    CK(cudaMemcpyAsync(gv.data(), h->G.p, gv.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (V && !vdev) CK(cudaMemcpyAsync(V, Vd, vbytes, cudaMemcpyDeviceToHost, st));
    if (Z && !zdev) CK(cudaMemcpyAsync(Z, Zd, vbytes, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    double orth = 0.0;
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) orth = std::max(orth, std::fabs(gv[i * m + j] - (i == j ? 1.0 : 0.0)));
    int n_neg = 0;
    for (int j = 0; j < m; ++j) {
        eigvals[j] = rr_host.theta[j];
        if (rr_host.theta[j] < 0.0) ++n_neg;
    }
    if (info) {
        info->iters = applies;
        info->n_applies = applies;
        info->n_negative = n_neg;
        info->converged = converged ? 1 : 0;
        info->max_residual = rr_host.maxres;
        info->orth_error = orth;
    }
    *converged_out = converged;
    return applies;
}

// ---------------------------------------------------------------------------- sharded eigensolver
// The block subspace iteration on a shard handle (round 2): each rank holds its
// rows of the iterate. The apply is the four sharded stages with the R^{-1} fold (t_g = (v_g^T Y1)
// R^{-1}); the Grams G = Y^T Y, 1^T Y and, at Rayleigh-Ritz steps, H' = Y_k^T Y_{k+1} are local
// partials summed with ncclAllReduce, so every rank factors the same G and solves the same
// Rayleigh-Ritz problem (the same convergence decision on every rank); V's rows stay local; the
// sign rule takes the global largest |v| (ties: lowest global row) by a max-allreduce of packed
// keys. Non-fused kernels (the row-blocked / tensor-core steps are not sharded).
namespace {
sbmds_status eigs_shard(sbmds_ctx* h, int m, int b, int max_iters, double tol, uint64_t seed, const float* X0,
                        double* eigvals, float* V, float* Z, sbmds_info* info, cudaStream_t st) {
    const NcclApi* nc = h->comm ? &nccl_api() : nullptr;
    ncclComm_t comm = reinterpret_cast<ncclComm_t>(h->comm);
    auto sum = [&](void* p, size_t count, ncclDataType_t ty) {
        if (h->comm) NK(nc->allReduce(p, p, count, ty, ncclSum, comm, st));
    };
    const int64_t n = h->n;
    const int bp = next_pow2(b);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, st));
    h->X.ensure((size_t)n * b * sizeof(float));
    h->Y.ensure((size_t)n * b * sizeof(float));
    h->G.ensure(kMaxB * kMaxB * sizeof(double));
    h->H.ensure(kMaxB * kMaxB * sizeof(double));
    h->Rinv.ensure(kMaxB * kMaxB * sizeof(double));
    h->status.ensure(16);
    h->rr.ensure(sizeof(RrOut));
    h->tsave.ensure(kMaxB * sizeof(double));
    ensure_apply_ws(h, bp);
    float* Yc = h->X.as<float>();
    float* Yn = h->Y.as<float>();
    if (X0) CK(cudaMemcpyAsync(Yc, X0, (size_t)n * b * sizeof(float), cudaMemcpyDefault, st));
    else launch(k_init_philox, dim3(4 * 148), dim3(256), 0, st, n, b, seed, Yc, h->row0 * b);
    auto grams = [&](const float* Y, const float* Yprev) {   // G, s (and H') summed over the ranks
        gram(h, b, Y, Yprev, st, true);
        sum(h->G.p, (size_t)b * b, ncclFloat64);
        sum(h->s.p, (size_t)b, ncclFloat64);
        if (Yprev) sum(h->H.p, (size_t)b * b, ncclFloat64);
    };
    grams(Yc, nullptr);
    chol(h, b, st);
    int hstat = 0;
    peek_to_host(&hstat, h->status.p, sizeof(int), st);
    if (hstat == 2) return fail(SBMDS_EBREAKDOWN, "Cholesky-QR of the initial block broke down");
    smem_attr(k_rr, kRrSmem);
    const double* Rinv = h->Rinv.as<double>();
    if (!h->vg_ok) {   // v_g = D w_g (t_g = v_g^T Y1)
        ensure_full_d(h, st);
        h->vg.ensure((size_t)h->l * sizeof(double));
        launch(k_symv_rows, dim3((unsigned)std::min<int64_t>(8 * (int64_t)h->num_sms, (h->l + 7) / 8)), dim3(256), 0,
               st, h->l, (const float*)h->D, h->ldD, (const double*)h->w.as<double>(), h->vg.as<double>());
        h->vg_ok = true;
    }
    int it = 1;
    bool converged = false;
    RrOut rr_host;
    for (; it <= max_iters; ++it) {
        const bool do_rr = (it % h->rr_period == 0) || it == max_iters;
        // Y_{k+1} = B~ (Y_k R^-1): s = 1^T Y_k came with the Gram
        profiled(h->prof, PK_CSC, st, [&] { spmm_csc(h, b, bp, Yc, st); });   // Y1_g = S_g^T Y_k - w_g s^T
        sum(h->Y1.p, (size_t)h->l * bp, ncclFloat32);
        profiled(h->prof, PK_SPLIT, st, [&] {
            vdot(h, b, bp, h->tsave.as<double>(), st);   // v_g^T Y1 (before the fold)
        });
        if (takes_sym(h, bp, true) || h->rank == 0) {
            dstream(h, b, bp, st, Rinv);
        } else {
            CK(cudaMemsetAsync(h->Y2.p, 0, (size_t)h->l * bp * sizeof(float), st));
        }
        launch(k_vec_rinv, dim3(1), dim3(64), 0, st, b, (const double*)h->tsave.as<double>(), Rinv, h->t.as<double>());
        if (h->comm) {
            NK(nc->groupStart());
            NK(nc->allReduce(h->Y2.p, h->Y2.p, (size_t)h->l * bp, ncclFloat32, ncclSum, comm, st));
            NK(nc->allReduce(h->t.p, h->t.p, (size_t)b, ncclFloat64, ncclSum, comm, st));
            NK(nc->groupEnd());
        }
        profiled(h->prof, PK_CSR, st, [&] { spmm_csr(h, b, bp, Yn, st); });   // local rows of Y_{k+1}
        grams(Yn, do_rr ? Yc : nullptr);
        if (do_rr) {
            launch(k_rr, dim3(1), dim3(256), (size_t)kRrSmem, st, b, m, tol, (const double*)h->H.as<double>(),
                   (const double*)h->G.as<double>(), Rinv, h->rr.as<RrOut>());
            int conv = 0;
            CK(cudaMemcpyAsync(&conv, &h->rr.as<RrOut>()->converged, sizeof(int), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            if (conv || it == max_iters) {
                converged = conv != 0;
                break;   // Ritz vectors Y_k (R_k^-1 U): Yc and Rinv stay valid
            }
        }
        chol(h, b, st);
        std::swap(Yc, Yn);
    }
    if (it > max_iters) it = max_iters;
    CK(cudaMemcpyAsync(&rr_host, h->rr.p, sizeof(RrOut), cudaMemcpyDeviceToHost, st));
    h->vsel.ensure(((size_t)b * m + 2 * m) * sizeof(double));
    double* Msel_d = h->vsel.as<double>();
    launch(k_select, dim3(1), dim3(256), 0, st, b, m, h->n_global, (const RrOut*)h->rr.as<RrOut>(), Rinv, Msel_d,
           Msel_d + (size_t)b * m, Msel_d + (size_t)b * m + m);
    std::vector<double> theta_out(m, 0.0);
    CK(cudaMemcpyAsync(theta_out.data(), Msel_d + (size_t)b * m + m, m * sizeof(double), cudaMemcpyDeviceToHost, st));
    const bool vdev = V && is_device_ptr(V), zdev = Z && is_device_ptr(Z);
    const size_t vbytes = (size_t)n * m * sizeof(float);
    float* Vd = vdev ? V : (h->vtmp.ensure(vbytes), h->vtmp.as<float>());
    float* Zd = zdev ? Z : (Z ? (h->ztmp.ensure(vbytes), h->ztmp.as<float>()) : nullptr);
    const double* theta = Msel_d + (size_t)b * m + m;
    rotate(h, b, m, m, (const float*)Yc, (const double*)Msel_d, Vd, (const double*)(Msel_d + (size_t)b * m), false, st);
    // the sign rule over all ranks' rows
    h->apidx.ensure(kRedBlocks * kMaxB * sizeof(long long));
    h->sign.ensure(kMaxB * sizeof(float));
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(h->apidx.p);
    CK(cudaMemsetAsync(keys, 0, m * sizeof(unsigned long long), st));
    launch(k_col_key, dim3((unsigned)std::min<int64_t>(4 * 148, (n * m + 255) / 256)), dim3(256), 0, st, n, m,
           (const float*)Vd, h->row0, keys);
    if (h->comm) NK(nc->allReduce(keys, keys, (size_t)m, ncclUint64, ncclMax, comm, st));
    launch(k_key_sign, dim3(1), dim3(64), 0, st, n, m, (const float*)Vd, h->row0, (const unsigned long long*)keys,
           h->sign.as<float>());
    sum(h->sign.p, (size_t)m, ncclFloat32);
    launch(k_finalize, dim3((unsigned)std::min<int64_t>(4 * 148, (n * m + 255) / 256)), dim3(256), 0, st, n, m,
           (const float*)h->sign.as<float>(), theta, Vd, Zd);
    gram(h, m, Vd, nullptr, st);
    sum(h->G.p, (size_t)m * m, ncclFloat64);
    std::vector<double> gv((size_t)m * m);
    CK(cudaMemcpyAsync(gv.data(), h->G.p, gv.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (V && !vdev) CK(cudaMemcpyAsync(V, Vd, vbytes, cudaMemcpyDeviceToHost, st));
    if (Z && !zdev) CK(cudaMemcpyAsync(Z, Zd, vbytes, cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(e1, st));
    CK(cudaStreamSynchronize(st));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    double orth = 0.0;
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) orth = std::max(orth, std::fabs(gv[i * m + j] - (i == j ? 1.0 : 0.0)));
    int n_neg = 0;
    for (int j = 0; j < m; ++j) {
        eigvals[j] = theta_out[j];
        if (theta_out[j] < 0.0) ++n_neg;
    }
    if (info) {
        info->iters = it;
        info->n_applies = it;
        info->n_negative = n_neg;
        info->converged = converged ? 1 : 0;
        info->max_residual = rr_host.maxres;
        info->orth_error = orth;
        info->gpu_ms = ms;
    }
    if (tol > 0.0 && !converged)
        return fail(SBMDS_ENOCONV, "no convergence in %d iterations (residual %g)", max_iters, rr_host.maxres);
    return SBMDS_OK;
}
}  // namespace

extern "C" sbmds_status sbmds_eigs(sbmds_t h, int32_t m, int32_t block, int32_t max_iters, double tol, uint64_t seed,
                                   const float* X0, double* eigvals, float* V, float* Z, sbmds_info* info,
                                   void* cuda_stream) {
    // (diagnostics) SBMDS_TRACE_EIGS=1: host-clock phase times of this eigs on stderr
    static const bool trace_eigs = getenv("SBMDS_TRACE_EIGS") != nullptr;
    const auto t_eigs0 = std::chrono::steady_clock::now();
    auto ephase = [&](const char* what, cudaStream_t sst) {
        nvtxMarkA(what);   // stage boundary on the NVTX timeline
        if (!trace_eigs) return;
        cudaStreamSynchronize(sst);
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_eigs0).count();
        fprintf(stderr, "[sbmds_eigs] %8.2f ms  %s\n", ms, what);
    };

    Nvtx nv_eigs("sbmds_eigs");
    if (!h) return fail(SBMDS_EINVAL, "NULL handle");
    if (h->shard) {
        if (h->world > 1 && !h->comm)
            return fail(SBMDS_EINVAL, "sbmds_eigs on a shard handle (world %d) needs an attached communicator", h->world);
        if (h->solver == 1) return fail(SBMDS_EINVAL, "the block Lanczos solver is not sharded");
        if (block < 1 || block > kMaxB || block >= h->n_global || m < 1 || m > block || max_iters < 1 || !eigvals)
            return fail(SBMDS_EINVAL, "need 1 <= m <= block <= 64, block < n, max_iters >= 1, eigvals");
        cudaStream_t sst = reinterpret_cast<cudaStream_t>(cuda_stream);
        DevGuard gs(h->dev);
        try {
            ensure_dq(h, sst);
            return eigs_shard(h, m, block, max_iters, tol, seed, X0, eigvals, V, Z, info, sst);
        } catch (const CudaError& e) {
            if (e.e == cudaErrorMemoryAllocation) return fail(SBMDS_ENOMEM, "device allocation failed (%s)", e.what);
            return fail(SBMDS_ECUDA, "%s: %s%s", e.what, cudaGetErrorString(e.e), hang_note().c_str());
        } catch (const NcclError& e) {
            return fail(SBMDS_ECUDA, "%s: %s", e.what, nccl_api().errorString(e.r));
        }
    }
    if (block < 1 || block > kMaxB || block >= h->n) return fail(SBMDS_EINVAL, "need 1 <= block <= 64, block < n");
    if (m < 1 || m > block) return fail(SBMDS_EINVAL, "need 1 <= m <= block");
    if (max_iters < 1) return fail(SBMDS_EINVAL, "need max_iters >= 1");
    if (!eigvals) return fail(SBMDS_EINVAL, "eigvals (host) is NULL");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
    DevGuard g(h->dev);
    const int b = block;
    const int64_t n = h->n;
    sbmds_status ret = SBMDS_OK;
    try {
        ensure_dq(h, st);   // the int8 stream's precision check (once per handle)
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, st));
        h->X.ensure((size_t)n * b * sizeof(float));
        h->Y.ensure((size_t)n * b * sizeof(float));
        h->G.ensure(kMaxB * kMaxB * sizeof(double));
        h->H.ensure(kMaxB * kMaxB * sizeof(double));
        h->Rinv.ensure(kMaxB * kMaxB * sizeof(double));
        h->Rinv2.ensure(kMaxB * kMaxB * sizeof(double));
        h->status.ensure(16);
        h->rr.ensure(sizeof(RrOut));
        h->gram_deferred = false;
        if (h->solver == 1) {   // NEXT-3: restarted block Lanczos with full reorthogonalisation
            struct EvGuard {
                cudaEvent_t a, b;
                ~EvGuard() {
                    cudaEventDestroy(a);
                    cudaEventDestroy(b);
                }
            } evg{e0, e1};
            if (b > 32) return fail(SBMDS_EINVAL, "block Lanczos needs block <= 32 (two blocks per cycle)");
            bool conv = false;
            try {
                eigs_lanczos(h, m, b, max_iters, tol, seed, X0, eigvals, V, Z, info, st, &conv);
            } catch (const LanczosBreakdown& e) {
                return fail(SBMDS_EBREAKDOWN, "%s", e.what);
            }
            CK(cudaEventRecord(e1, st));
            CK(cudaStreamSynchronize(st));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (info) info->gpu_ms = ms;
            if (tol > 0.0 && !conv) return fail(SBMDS_ENOCONV, "block Lanczos: no convergence in %d applies", max_iters);
            return SBMDS_OK;
        }
        // Two n x b buffers alternate as Y_k (current, unnormalised) and Y_{k+1}; the
        // orthonormal iterate is X_k = Y_k R_k^{-1} (R from Cholesky-QR), never materialised.
        float* Yc = h->X.as<float>();
        float* Yn = h->Y.as<float>();
        // E1: initial block Y_0 (Philox N(0,1) or the warm start), G_0, s_0, R_0^{-1}
        if (X0) {
            if (h->permuted) {   // warm start in the caller's order -> the handle's
                h->xperm.ensure((size_t)n * b * sizeof(float));
                CK(cudaMemcpyAsync(h->xperm.p, X0, (size_t)n * b * sizeof(float), cudaMemcpyDefault, st));
                permute_block(h, b, h->xperm.as<float>(), Yc, false, st);
            } else
            CK(cudaMemcpyAsync(Yc, X0, (size_t)n * b * sizeof(float), cudaMemcpyDefault, st));
        } else {
            launch(k_init_philox, dim3(4 * 148), dim3(256), 0, st, n, b, seed, Yc, (int64_t)0);
        }
        gram(h, b, Yc, nullptr, st, true);
        chol(h, b, st);
        int hstat = 0;
        CK(cudaMemcpyAsync(&hstat, h->status.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (hstat == 2) return fail(SBMDS_EBREAKDOWN, "Cholesky-QR of the initial block broke down");
        h->chol_retries = hstat == 1 ? 1 : 0;
        ephase("initial block", st);

        smem_attr(k_rr, kRrSmem);
        RrOut rr_host;
        int it = 0;
        bool converged = false;
        const bool fused = fused_ok(h, b) && blocked_ok(h, b, b, Yc, Yn);
        const bool sp8 = fused && sp8_ok(h, b, st);   // tensor-core sparse step (fuse = 3)
        // b = 32 (config 3): the same kernel as two 16-column passes per step, Gram and Cholesky
        // by their own kernels
        const bool sp8h = !sp8 && fused && b == 32 && h->fuse == 3 && h->sp8_apply && sp8_ok(h, 16, st);   // (also on small
        // problems, unlike the standalone apply: config 2 at b = 32 7.5 vs 10.5 ms per 50 iterations on the fp32 fused kernels)
        // one iteration's device work: Y_{k+1} = B~ X_k = (B~ Y_k) R_k^{-1} (s = 1^T Y_k came from
        // the last Gram), the Grams, and at Rayleigh-Ritz steps the Jacobi solve (no host syncs)
        auto enqueue_iteration = [&](int itx, bool do_rr) {
            if (sp8) {
                // A5 + Grams + the next apply's S^T Y_{k+1} partials on the int8 tensor cores (k_sp8.cuh)
                // (a Rayleigh-Ritz step reads G_k (through R_k) and G_{k+1}: those two stay on the
                // FP64 Gram of the fp32 rows; the others only orthonormalise the next iterate)
                const bool rr_next = (tol > 0.0 && (itx + 1) % std::max(1, h->rr_period) == 0) || itx + 1 >= max_iters;
                const int fl = kApplyFused | kApplySp8 | kApplyChol | (itx > 1 ? kApplyY1Ready : 0) |
                               (itx == max_iters && !(h->sp8_dbg & 8) ? kApplyNoP1 : 0) |
                               (h->sp8_gram8 && ((!do_rr && !rr_next) || (h->sp8_dbg & 32)) ? kApplyGram8 : 0);   // (sp8_dbg & 32: diagnostics)
                apply_device(h, b, Yc, Yn, st, true, h->Rinv.as<double>(), fl,
                             do_rr && !(h->sp8_dbg & 16) ? Yc : nullptr);
            } else if (sp8h) {
                const bool rr_next = (tol > 0.0 && (itx + 1) % std::max(1, h->rr_period) == 0) || itx + 1 >= max_iters;
                const int fl = kApplyFused | kApplySp8 | kApplySp8Halves | (itx > 1 ? kApplyY1Ready : 0) |
                               (itx == max_iters ? kApplyNoP1 : 0) |
                               (h->sp8_gram8 && !do_rr && !rr_next ? kApplyGram8 : 0);
                apply_device(h, b, Yc, Yn, st, true, h->Rinv.as<double>(), fl, do_rr ? Yc : nullptr);
            } else if (fused) {
                // A5 fused with G = Y_{k+1}^T Y_{k+1}, s = 1^T Y_{k+1}, H' = Y_k^T Y_{k+1} (RR) and
                // (fuse = 2) the next apply's S^T Y_{k+1} partials (k_fused.cuh)
                // (fuse 3 without the tensor-core step: the partials too from b = 32 on -- config 3:
                // 39.4 vs 46.0 ms per 50 iterations)
                const bool p1 = h->fuse == 2 || (h->fuse == 3 && b >= 32);
                const int fl = kApplyFused | (p1 && itx > 1 ? kApplyY1Ready : 0) | (!p1 || itx == max_iters ? kApplyNoP1 : 0);
                apply_device(h, b, Yc, Yn, st, true, h->Rinv.as<double>(), fl, do_rr ? Yc : nullptr);
            } else {
                apply_device(h, b, Yc, Yn, st, true, h->Rinv.as<double>());
                // G = Y_{k+1}^T Y_{k+1}, s = 1^T Y_{k+1}, and H' = Y_k^T Y_{k+1} for Rayleigh-Ritz
                gram(h, b, Yn, do_rr ? Yc : nullptr, st, true);
            }
            if (do_rr) {
                // H = X_k^T B~ X_k = R_k^{-T} H'
                profiled(h->prof, PK_RR, st, [&] {
                    launch(k_rr, dim3(1), dim3(256), (size_t)kRrSmem, st, b, m, tol, (const double*)h->H.as<double>(),
                           (const double*)h->G.as<double>(), (const double*)h->Rinv.as<double>(), h->rr.as<RrOut>());
                });
            }
        };
        // CUDA graphs (option use_graph): after the first Rayleigh-Ritz segment
        // (which also warms every buffer and tensor map), a segment of rr_period iterations -- the
        // first rr_period - 1 with their Cholesky-QR, the last ending with the Jacobi solve -- is
        // captured once per buffer parity and replayed; the host only reads the convergence flag
        // between segments, exactly where the eager loop reads it. Off while kernels are profiled.
        const int R = std::max(1, h->rr_period);
        const bool graphs = h->use_graph && h->prof.mask == 0 && !(fused && h->fuse >= 2) && R >= 2;   // (the partial
        // chains of fuse 2/3 depend on the iteration index: eager only)
        cudaGraphExec_t gexec[2] = {nullptr, nullptr};
        int64_t gnodes[2] = {0, 0};
        struct GraphGuard {
            cudaGraphExec_t* g;
            ~GraphGuard() {
                for (int k = 0; k < 2; ++k)
                    if (g[k]) cudaGraphExecDestroy(g[k]);
            }
        } graph_guard{gexec};
        it = 1;
        while (it <= max_iters) {
            const bool seg = graphs && it > R && (it - 1) % R == 0 && it + R - 1 <= max_iters;
            bool do_rr;
            if (seg) {
                const int par = (Yc == h->X.as<float>()) ? 0 : 1;
                if (!h->gstream) {
                    CK(cudaStreamCreateWithFlags(&h->gstream, cudaStreamNonBlocking));
                    CK(cudaEventCreateWithFlags(&h->gev[0], cudaEventDisableTiming));
                    CK(cudaEventCreateWithFlags(&h->gev[1], cudaEventDisableTiming));
                }
                cudaStream_t const st_caller = st;
                if (!gexec[par]) {
                    float* const Yc0 = Yc;
                    float* const Yn0 = Yn;
                    st = h->gstream;   // the lambdas enqueue on `st`
                    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
                    const int64_t n0 = g_launches.load();
                    try {
                        for (int k = 0; k < R; ++k) {
                            enqueue_iteration(it + k, k == R - 1);
                            if (k < R - 1) {
                                chol(h, b, st);
                                std::swap(Yc, Yn);
                            }
                        }
                    } catch (...) {   // end (and drop) the capture, restore the caller's stream
                        cudaGraph_t gbad = nullptr;
                        cudaStreamEndCapture(h->gstream, &gbad);
                        if (gbad) cudaGraphDestroy(gbad);
                        st = st_caller;
                        throw;
                    }
                    cudaGraph_t g = nullptr;
                    CK(cudaStreamEndCapture(st, &g));
                    const cudaError_t ie = cudaGraphInstantiate(&gexec[par], g, 0);
                    cudaGraphDestroy(g);
                    CK(ie);
                    gnodes[par] = g_launches.load() - n0;   // captured, not yet run
                    g_launches.fetch_sub(gnodes[par]);
                    Yc = Yc0;
                    Yn = Yn0;
                    st = st_caller;
                }
                // replay on the graph stream, ordered after and before the caller's stream work
                CK(cudaEventRecord(h->gev[0], st));
                CK(cudaStreamWaitEvent(h->gstream, h->gev[0], 0));
                CK(cudaGraphLaunch(gexec[par], h->gstream));
                CK(cudaEventRecord(h->gev[1], h->gstream));
                CK(cudaStreamWaitEvent(st, h->gev[1], 0));
                g_launches.fetch_add(gnodes[par]);
                for (int k = 0; k < R - 1; ++k) std::swap(Yc, Yn);
                it += R - 1;   // the segment's Rayleigh-Ritz iteration
                do_rr = true;
            } else {
                // Rayleigh-Ritz only feeds the convergence test (the iterate is never rotated), so a
                // fixed-iteration solve (tol <= 0, BASELINE config 4) needs it only at the end
                do_rr = (tol > 0.0 && it % R == 0) || it == max_iters;
                enqueue_iteration(it, do_rr);
            }
            if (it <= 2) ephase(it == 1 ? "iteration 1" : "iteration 2", st);
            if (do_rr) {
                int conv = 0;
                CK(cudaMemcpyAsync(&conv, &h->rr.as<RrOut>()->converged, sizeof(int), cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                if (conv || it == max_iters) {
                    converged = conv != 0;
                    break;   // Ritz vectors are X_k U = Y_k (R_k^{-1} U): Yc and Rinv stay valid
                }
            }
            if (sp8) h->Rinv.swap(h->Rinv2);   // R_{k+1}^{-1}, factored by the step's last CTA
            else chol(h, b, st);               // R_{k+1}^{-1}
            std::swap(Yc, Yn);
            if (do_rr || it % 16 == 0) {
                CK(cudaMemcpyAsync(&hstat, h->status.p, sizeof(int), cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                if (hstat == 2) return fail(SBMDS_EBREAKDOWN, "Cholesky-QR broke down at iteration %d", it);
                if (hstat == 1) ++h->chol_retries;
            }
            ++it;
        }
        if (it > max_iters) it = max_iters;
        ephase("iterations done", st);
        CK(cudaMemcpyAsync(&rr_host, h->rr.p, sizeof(RrOut), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        // E6: select the top-m algebraic pairs. B~ 1 = 0 exactly (J 1 = 0), but the iterate
        // lives in 1^perp after the first apply, so the known pair (0, 1/sqrt(n)) is merged
        // into the Ritz list: it enters the top m when fewer than m Ritz values are >= 0 (k_select).
        h->vsel.ensure(((size_t)b * m + 2 * m) * sizeof(double));
        double* Msel_d = h->vsel.as<double>();
        launch(k_select, dim3(1), dim3(256), 0, st, b, m, n, (const RrOut*)h->rr.as<RrOut>(),
               (const double*)h->Rinv.as<double>(), Msel_d, Msel_d + (size_t)b * m, Msel_d + (size_t)b * m + m);
        std::vector<double> theta_out(m, 0.0);
        CK(cudaMemcpyAsync(theta_out.data(), Msel_d + (size_t)b * m + m, m * sizeof(double), cudaMemcpyDeviceToHost,
                           st));
        const bool vdev = V && is_device_ptr(V), zdev = Z && is_device_ptr(Z);
        const size_t vbytes = (size_t)n * m * sizeof(float);
        float* Vd = vdev ? V : (h->vtmp.ensure(vbytes), h->vtmp.as<float>());
        float* Zd = zdev ? Z : (Z ? (h->ztmp.ensure(vbytes), h->ztmp.as<float>()) : nullptr);
        const int grid = (int)std::min<int64_t>(4 * 148, (n * m + 255) / 256);
        const double* theta = Msel_d + (size_t)b * m + m;
        rotate(h, b, m, m, (const float*)Yc, (const double*)Msel_d, Vd, (const double*)(Msel_d + (size_t)b * m),
               false, st);
        unpermute_v(h, m, Vd, st);
        h->sign.ensure(kMaxB * sizeof(float));
        h->apval.ensure(kRedBlocks * kMaxB * sizeof(float));
        h->apidx.ensure(kRedBlocks * kMaxB * sizeof(long long));
        launch(k_col_argmax, dim3(kRedBlocks), dim3(256), 0, st, n, m, (const float*)Vd, h->apval.as<float>(),
               h->apidx.as<long long>(), h->sign.as<float>(), h->counters.as<unsigned int>() + CNT_ARGMAX);
        launch(k_finalize, dim3(grid), dim3(256), 0, st, n, m, (const float*)h->sign.as<float>(), theta, Vd, Zd);
        // orthogonality of the returned V (fp64 Gram)
        gram(h, m, Vd, nullptr, st);
        std::vector<double> gv((size_t)m * m);
        CK(cudaMemcpyAsync(gv.data(), h->G.p, gv.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
        if (V && !vdev) CK(cudaMemcpyAsync(V, Vd, vbytes, cudaMemcpyDeviceToHost, st));
        if (Z && !zdev) CK(cudaMemcpyAsync(Z, Zd, vbytes, cudaMemcpyDeviceToHost, st));
        CK(cudaEventRecord(e1, st));
        CK(cudaStreamSynchronize(st));
        ephase("outputs on the host", st);
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        double orth = 0.0;
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < m; ++j) orth = std::max(orth, std::fabs(gv[i * m + j] - (i == j ? 1.0 : 0.0)));
        int n_neg = 0;
        for (int j = 0; j < m; ++j) {
            eigvals[j] = theta_out[j];
            if (theta_out[j] < 0.0) ++n_neg;
        }
        if (info) {
            info->iters = it;
            info->n_applies = it;
            info->n_negative = n_neg;
            info->converged = converged ? 1 : 0;
            info->max_residual = rr_host.maxres;
            info->orth_error = orth;
            info->gpu_ms = ms;
        }
        if (tol > 0.0 && !converged) ret = fail(SBMDS_ENOCONV, "no convergence in %d iterations (residual %g)",
                                                max_iters, rr_host.maxres);
    } catch (const CudaError& e) {
        if (e.e == cudaErrorMemoryAllocation) return fail(SBMDS_ENOMEM, "device allocation failed (%s)", e.what);
        return fail(SBMDS_ECUDA, "%s: %s%s", e.what, cudaGetErrorString(e.e), hang_note().c_str());
    }
    return ret;
}

// ============================================================================ BMDS
// NEXT-3b: the paper's QR route, k_bmds.cuh. Steps (all on the device, fp64):
//   G = (J P)^T (J P) from the dense n x l J P; G = R^T R (blocked upper Cholesky, 64-wide panels);
//   M = -1/2 R W R^T; the top-m algebraic eigenpairs of the l x l M by block subspace iteration
//   with Cholesky-QR and Rayleigh-Ritz (k_chol, k_rr: the same small kernels as sbmds_eigs);
//   U = R^{-1} V~_m; V = J P U = S U - 1 (w^T U) (CSR SpMM), Z = V Λ^{1/2}, signs as sbmds_eigs.
namespace {
// fp64 GEMM dispatch: small shapes on the 64 x 64 kernel; shapes with >= 64 big tiles or a long
// K on the 128 x 128 one, splitting K (fixed-order sum of the slices) until ~2 CTAs per SM
// (ws: the caller's split-K workspace, grown on demand and reused across calls)
template <bool TA, bool TB>
void dgemm(cudaStream_t st, DevBuf& ws, int M, int N, int64_t K, double alpha, const double* A, int64_t lda,
           const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
    const int64_t tiles = (int64_t)((M + 127) / 128) * ((N + 127) / 128);
    if ((int64_t)M * N < 128 * 128 || K < 64) {
        launch(k_dgemm<TA, TB>, dim3((unsigned)((N + 63) / 64), (unsigned)((M + 63) / 64)), dim3(256), 0, st, M, N, K,
               alpha, A, lda, B, ldb, beta, C, ldc);
        return;
    }
    int splits = 1;
    while (tiles * splits < 296 && K / (splits * 2) >= 512) splits *= 2;
    if (splits > 1) {
        ws.ensure((size_t)splits * M * N * sizeof(double));
        launch(k_dgemm128<TA, TB>, dim3((unsigned)((N + 127) / 128), (unsigned)((M + 127) / 128), (unsigned)splits),
               dim3(256), 0, st, M, N, K, 1.0, A, lda, B, ldb, 0.0, C, ldc, ws.as<double>());
        launch(k_sum_splits, dim3((unsigned)std::min<int64_t>(4096, ((int64_t)M * N + 255) / 256)), dim3(256), 0, st, M,
               N, splits, alpha, (const double*)ws.as<double>(), beta, C, ldc);
    } else {
        launch(k_dgemm128<TA, TB>, dim3((unsigned)((N + 127) / 128), (unsigned)((M + 127) / 128), 1u), dim3(256), 0, st,
               M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, (double*)nullptr);
    }
}
}  // namespace

extern "C" sbmds_status sbmds_bmds(sbmds_t h, int32_t m, int32_t block, int32_t max_iters, double tol, uint64_t seed,
                                   double* eigvals, float* V, float* Z, sbmds_info* info, void* cuda_stream) {
    Nvtx nv("sbmds_bmds");
    if (!h) return fail(SBMDS_EINVAL, "NULL handle");
    if (h->shard) return fail(SBMDS_EINVAL, "sbmds_bmds on a shard handle");
    const int64_t n = h->n, l = h->l;
    if (l > kBmdsMaxL || (double)n * (double)l > 2.0e9)
        return fail(SBMDS_EINVAL, "BMDS needs l <= %d and n l <= 2e9 (dense J P and l x l factors)", kBmdsMaxL);
    if (block < 1 || block > kMaxB || block > l) return fail(SBMDS_EINVAL, "need 1 <= block <= min(64, l)");
    if (m < 1 || m > block) return fail(SBMDS_EINVAL, "need 1 <= m <= block");
    if (max_iters < 1) return fail(SBMDS_EINVAL, "need max_iters >= 1");
    if (!eigvals) return fail(SBMDS_EINVAL, "eigvals (host) is NULL");
    if ((V && !is_device_ptr(V)) || (Z && !is_device_ptr(Z))) return fail(SBMDS_EINVAL, "sbmds_bmds: V, Z on the device");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
    DevGuard g(h->dev);
    const int b = block;
    sbmds_status ret = SBMDS_OK;
    try {
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, st));
        DevBuf JP{true}, A{true}, W{true}, T{true}, X{true}, Y{true}, small{true}, gws{true};
        h->G.ensure(kMaxB * kMaxB * sizeof(double));   // (the final orthogonality Gram)
        h->status.ensure(16);
        CK(cudaMemsetAsync(h->status.p, 0, 16, st));
        int* status = h->status.as<int>();
        // J P (dense, n x l) and its Gram G (in A)
        JP.ensure((size_t)n * l * sizeof(double));
        launch(k_jp_dense, dim3((unsigned)std::min<int64_t>(n, 16 * (int64_t)h->num_sms)), dim3(256), 0, st, n, l,
               (const int32_t*)h->rp.as<int32_t>(), (const int32_t*)h->col.as<int32_t>(),
               (const float*)h->val.as<float>(), (const double*)h->w.as<double>(), JP.as<double>());
        A.ensure((size_t)l * l * sizeof(double));
        dgemm<true, false>(st, gws, (int)l, (int)l, n, 1.0, JP.as<double>(), l, JP.as<double>(), l, 0.0, A.as<double>(), l);
        JP.release();
        // G = R^T R, right-looking, 64-column panels (semi-definite: null pivots dropped)
        small.ensure((size_t)3 * kMaxB * kMaxB * sizeof(double) + 64);
        double* dmax = reinterpret_cast<double*>(small.as<char>() + (size_t)3 * kMaxB * kMaxB * sizeof(double));
        int* dropped = status + 2;
        launch(k_maxdiag, dim3(1), dim3(256), 0, st, (const double*)A.as<double>(), l, l, dmax);
        for (int64_t k0 = 0; k0 < l; k0 += 64) {
            const int nb = (int)std::min<int64_t>(64, l - k0);
            launch(k_potf2, dim3(1), dim3(256), 0, st, A.as<double>(), l, (int)k0, nb, status, (const double*)dmax,
                   dropped, 1);
            const int64_t rest = l - k0 - nb;
            if (rest > 0) {
                launch(k_trsm_rows, dim3((unsigned)((rest + 255) / 256)), dim3(256), 0, st, A.as<double>(), l, l,
                       (int)k0, nb, (const int*)status);
                // trailing A[k1:, k1:] -= R[k0:k1, k1:]^T R[k0:k1, k1:]
                const double* Rp = A.as<double>() + k0 * l + k0 + nb;
                dgemm<true, false>(st, gws, (int)rest, (int)rest, nb, -1.0, Rp, l, Rp, l, 1.0,
                                   A.as<double>() + (k0 + nb) * l + k0 + nb, l);
            }
        }
        int hst3[3] = {0, 0, 0};
        peek_to_host(hst3, status, sizeof hst3, st);
        int hstat = hst3[0];
        if (hstat == 2) return fail(SBMDS_EBREAKDOWN, "BMDS: (JP)^T JP is not positive semi-definite");
        h->bmds_dropped = hst3[2];
        launch(k_zero_lower, dim3((unsigned)std::min<int64_t>(4096, (l * l + 255) / 256)), dim3(256), 0, st,
               A.as<double>(), l, l);
        // M = -1/2 R W R^T
        ensure_full_d(h, st);
        W.ensure((size_t)l * l * sizeof(double));
        T.ensure((size_t)l * l * sizeof(double));
        launch(k_f2d_sym, dim3((unsigned)std::min<int64_t>(4096, (l * l + 255) / 256)), dim3(256), 0, st, l,
               (const float*)h->D, h->ldD, W.as<double>());
        dgemm<false, false>(st, gws, (int)l, (int)l, l, 1.0, A.as<double>(), l, W.as<double>(), l, 0.0, T.as<double>(), l);
        dgemm<false, true>(st, gws, (int)l, (int)l, l, -0.5, T.as<double>(), l, A.as<double>(), l, 0.0, W.as<double>(), l);
        double* Md = W.as<double>();
        // top-m of M: block subspace iteration (X orthonormal l x b)
        X.ensure((size_t)l * b * sizeof(double));
        Y.ensure((size_t)l * b * sizeof(double));
        double* Gs = small.as<double>();
        double* Hs = Gs + kMaxB * kMaxB;
        h->Rinv.ensure(kMaxB * kMaxB * sizeof(double));
        h->rr.ensure(sizeof(RrOut));
        launch(k_dinit, dim3(64), dim3(256), 0, st, l * b, (uint64_t)seed, Y.as<double>());
        auto orth = [&](double* Yin, double* Xout) {   // Xout = Yin R^-1, Yin^T Yin = R^T R
            dgemm<true, false>(st, gws, b, b, l, 1.0, Yin, b, Yin, b, 0.0, Gs, b);
            chol_launch(b, (const double*)Gs, h->Rinv.as<double>(), status, st);
            dgemm<false, false>(st, gws, (int)l, b, b, 1.0, Yin, b, h->Rinv.as<double>(), b, 0.0, Xout, b);
        };
        orth(Y.as<double>(), X.as<double>());
        smem_attr(k_rr, kRrSmem);
        int it = 0;
        bool converged = false;
        RrOut rr_host;
        for (it = 1; it <= max_iters; ++it) {
            dgemm<false, false>(st, gws, (int)l, b, l, 1.0, Md, l, X.as<double>(), b, 0.0, Y.as<double>(), b);
            if (it % h->rr_period == 0 || it == max_iters) {
                dgemm<true, false>(st, gws, b, b, l, 1.0, X.as<double>(), b, Y.as<double>(), b, 0.0, Hs, b);
                dgemm<true, false>(st, gws, b, b, l, 1.0, Y.as<double>(), b, Y.as<double>(), b, 0.0, Gs, b);
                launch(k_rr, dim3(1), dim3(256), kRrSmem, st, b, m, tol > 0.0 ? tol : -1.0, (const double*)Hs,
                       (const double*)Gs, (const double*)nullptr, h->rr.as<RrOut>());
                int conv = 0;
                CK(cudaMemcpyAsync(&conv, &h->rr.as<RrOut>()->converged, sizeof(int), cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                if ((tol > 0.0 && conv) || it == max_iters) {
                    converged = tol > 0.0 && conv;
                    break;
                }
            }
            orth(Y.as<double>(), X.as<double>());
        }
        if (it > max_iters) it = max_iters;
        peek_to_host(&hstat, status, sizeof(int), st);
        if (hstat == 2) return fail(SBMDS_EBREAKDOWN, "BMDS: Cholesky-QR of the l x b iterate broke down");
        CK(cudaMemcpyAsync(&rr_host, h->rr.p, sizeof(RrOut), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        // V~_m = X U[:, :m] (l x m), U_l = R^-1 V~_m, V = J P U_l
        double* Vt = Y.as<double>();                       // (reuse: l x m)
        double* Ul = T.as<double>();
        dgemm<false, false>(st, gws, (int)l, m, b, 1.0, X.as<double>(), b, h->rr.as<RrOut>()->U, b, 0.0, Vt, m);
        launch(k_backsolve, dim3((unsigned)((m + 7) / 8)), dim3(256), 0, st, l, m, (const double*)A.as<double>(), l,
               (const double*)Vt, (int64_t)m, Ul);
        const int bp = next_pow2(m);
        ensure_apply_ws(h, bp);
        launch(k_bmds_to_y2, dim3(1), dim3(256), 0, st, l, m, bp, (const double*)Ul, (const double*)h->w.as<double>(),
               h->Y2.as<float>(), h->t.as<double>());
        const size_t vbytes = (size_t)n * m * sizeof(float);
        float* Vd = V ? V : (h->vtmp.ensure(vbytes), h->vtmp.as<float>());
        spmm_csr(h, m, bp, Vd, st);
        unpermute_v(h, m, Vd, st);
        h->sign.ensure(kMaxB * sizeof(float));
        h->apval.ensure(kRedBlocks * kMaxB * sizeof(float));
        h->apidx.ensure(kRedBlocks * kMaxB * sizeof(long long));
        launch(k_col_argmax, dim3(kRedBlocks), dim3(256), 0, st, n, m, (const float*)Vd, h->apval.as<float>(),
               h->apidx.as<long long>(), h->sign.as<float>(), h->counters.as<unsigned int>() + CNT_ARGMAX);
        const double* theta = h->rr.as<RrOut>()->theta;
        launch(k_finalize, dim3((unsigned)std::min<int64_t>(4 * 148, (n * m + 255) / 256)), dim3(256), 0, st, n, m,
               (const float*)h->sign.as<float>(), theta, Vd, Z);
        gram(h, m, Vd, nullptr, st);
        std::vector<double> gv((size_t)m * m);
        CK(cudaMemcpyAsync(gv.data(), h->G.p, gv.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaEventRecord(e1, st));
        CK(cudaStreamSynchronize(st));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        double orth_err = 0.0;
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < m; ++j) orth_err = std::max(orth_err, std::fabs(gv[i * m + j] - (i == j ? 1.0 : 0.0)));
        int n_neg = 0;
        for (int j = 0; j < m; ++j) {
            eigvals[j] = rr_host.theta[j];
            if (rr_host.theta[j] < 0.0) ++n_neg;
        }
        if (info) {
            info->iters = it;
            info->n_applies = 0;   // (no operator applies: the l x l problem only)
            info->n_negative = n_neg;
            info->converged = converged ? 1 : 0;
            info->max_residual = rr_host.maxres;
            info->orth_error = orth_err;
            info->gpu_ms = ms;
        }
        if (tol > 0.0 && !converged)
            ret = fail(SBMDS_ENOCONV, "BMDS: no convergence in %d iterations (residual %g)", max_iters, rr_host.maxres);
    } catch (const CudaError& e) {
        if (e.e == cudaErrorMemoryAllocation) return fail(SBMDS_ENOMEM, "device allocation failed (%s)", e.what);
        return fail(SBMDS_ECUDA, "%s: %s%s", e.what, cudaGetErrorString(e.e), hang_note().c_str());
    }
    return ret;
}

// ============================================================================ sBHA build
// NEXT-2 (§2.2, §3, §3.1; k_sbha.cuh): the sparse interpolation operator S = P_sparse
// of a triangle mesh on the device, ready for sbmds_create.
namespace {

// Reverse Cuthill-McKee of the free vertices' graph (L's 1-ring without the landmarks): BFS from
// a pseudo-peripheral start (two sweeps from the lowest-degree vertex), neighbours visited by
// increasing degree (ties: lower index), per connected component, then reversed.
std::vector<int32_t> rcm_order(int64_t n, const std::vector<int64_t>& lp, const std::vector<int32_t>& lc,
                               const std::vector<int32_t>& lmpos) {
    std::vector<int32_t> deg(n, 0);
    for (int64_t i = 0; i < n; ++i)
        if (lmpos[i] < 0)
            for (int64_t e = lp[i]; e < lp[i + 1]; ++e)
                if (lc[e] != i && lmpos[lc[e]] < 0) ++deg[i];
    std::vector<int32_t> order, level(n, -1);
    order.reserve(n);
    std::vector<char> done(n, 0);
    std::vector<int32_t> nbr;
    auto bfs = [&](int32_t s0, std::vector<int32_t>& out, bool record) -> int32_t {
        // returns the last vertex of the deepest level (lowest degree among them)
        std::vector<int32_t> q{s0};
        std::vector<char>& seen = done;
        std::vector<int32_t> touched{s0};
        seen[s0] = 1;
        for (size_t h = 0; h < q.size(); ++h) {
            const int32_t v = q[h];
            nbr.clear();
            for (int64_t e = lp[v]; e < lp[v + 1]; ++e) {
                const int32_t j = lc[e];
                if (j != v && lmpos[j] < 0 && !seen[j]) nbr.push_back(j);
            }
            std::sort(nbr.begin(), nbr.end(), [&](int32_t a, int32_t b) { return deg[a] != deg[b] ? deg[a] < deg[b] : a < b; });
            for (int32_t j : nbr) {
                seen[j] = 1;
                q.push_back(j);
                touched.push_back(j);
            }
        }
        if (record) out.insert(out.end(), q.begin(), q.end());
        else for (int32_t v : touched) seen[v] = 0;
        int32_t last = q.back();
        return last;
    };
    for (int64_t s0 = 0; s0 < n; ++s0) {
        if (lmpos[s0] >= 0 || done[s0]) continue;
        // component's lowest-degree vertex, then two pseudo-peripheral sweeps
        int32_t start = (int32_t)s0;
        std::vector<int32_t> dummy;
        const int32_t far1 = bfs(start, dummy, false);
        const int32_t far2 = bfs(far1, dummy, false);
        bfs(far2, order, true);
    }
    std::reverse(order.begin(), order.end());
    return order;
}

}  // namespace

extern "C" int64_t sbmds_sbha_p(int64_t n, int64_t l, double p_row) {
    if (l < 1 || l >= n || !(p_row > 0.0)) return -1;
    const double v = std::ceil((double)(n - l) * p_row / (double)l);
    return std::max<int64_t>(1, std::min<int64_t>(n - l, (int64_t)v));
}

extern "C" sbmds_status sbmds_sbha_build(int64_t n, const double* verts, int64_t nf, const int32_t* faces, int64_t l,
                                         const int32_t* landmarks, double p_row, int64_t* row_ptr, int32_t* col_idx,
                                         float* val, sbmds_sbha_info* info, void* cuda_stream) {
    Nvtx nv("sbmds_sbha_build");
    const int64_t p = sbmds_sbha_p(n, l, p_row);
    if (n < 2 || nf < 1 || p < 1) return fail(SBMDS_EINVAL, "need n >= 2, nf >= 1, 1 <= l < n, p_row > 0");
    if (n >= (int64_t(1) << 31) || nf * 3 >= (int64_t(1) << 31)) return fail(SBMDS_EINVAL, "n or nf too large");
    if (!verts || !faces || !landmarks || !row_ptr || !col_idx || !val) return fail(SBMDS_EINVAL, "NULL argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
    const auto t0 = std::chrono::steady_clock::now();
    try {
        install_hang_record();
        configure_pool_once();
        int dev = 0, sms = 148;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        std::vector<int32_t> lm(l);
        CK(cudaMemcpy(lm.data(), landmarks, l * sizeof(int32_t), cudaMemcpyDefault));
        std::vector<int32_t> lmpos(n, -1);
        for (int64_t t = 0; t < l; ++t) {
            if (lm[t] < 0 || lm[t] >= n || lmpos[lm[t]] >= 0) return fail(SBMDS_EINVAL, "landmarks must be distinct, in [0, n)");
            lmpos[lm[t]] = (int32_t)t;
        }
        DevBuf dV{true}, dF{true}, cot{true}, area{true}, bad{true}, keys{true}, keys2{true}, fid{true}, fid2{true},
            vfp{true}, deg{true}, lptr{true}, lcol{true}, lval{true}, mass{true};
        dV.ensure((size_t)n * 3 * sizeof(double));
        dF.ensure((size_t)nf * 3 * sizeof(int32_t));
        CK(cudaMemcpyAsync(dV.p, verts, (size_t)n * 3 * sizeof(double), cudaMemcpyDefault, st));
        CK(cudaMemcpyAsync(dF.p, faces, (size_t)nf * 3 * sizeof(int32_t), cudaMemcpyDefault, st));
        bad.ensure(sizeof(int));
        CK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
        {   // faces index check on the host side of the copy is not needed: the incidence sort
            std::vector<int32_t> hf((size_t)nf * 3);
            CK(cudaMemcpyAsync(hf.data(), dF.p, hf.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            for (int32_t v : hf)
                if (v < 0 || v >= n) return fail(SBMDS_EINVAL, "face vertex index out of [0, n)");
        }
        cot.ensure((size_t)nf * 3 * sizeof(double));
        area.ensure((size_t)nf * sizeof(double));
        launch(k_face_geom, dim3((unsigned)std::min<int64_t>(4 * sms, (nf + 255) / 256)), dim3(256), 0, st, nf,
               (const double*)dV.as<double>(), (const int32_t*)dF.as<int32_t>(), cot.as<double>(), area.as<double>(),
               bad.as<int>());
        // vertex -> incident faces (stable radix sort of the corners by vertex keeps faces ascending)
        const int32_t nc = (int32_t)(nf * 3);
        keys2.ensure(nc * sizeof(int32_t));
        fid.ensure(nc * sizeof(int32_t));
        fid2.ensure(nc * sizeof(int32_t));
        {
            std::vector<int32_t> hf(nc);
            for (int32_t e = 0; e < nc; ++e) hf[e] = e / 3;
            CK(cudaMemcpyAsync(fid.p, hf.data(), nc * sizeof(int32_t), cudaMemcpyHostToDevice, st));
            int end_bit = 1;
            while ((int64_t(1) << end_bit) <= n) ++end_bit;
            size_t tb = 0;
            CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, dF.as<int32_t>(), keys2.as<int32_t>(), fid.as<int32_t>(),
                                               fid2.as<int32_t>(), nc, 0, end_bit, st));
            DevBuf tmp{true};
            tmp.ensure(tb + 16);
            CK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, dF.as<int32_t>(), keys2.as<int32_t>(), fid.as<int32_t>(),
                                               fid2.as<int32_t>(), nc, 0, end_bit, st));
            g_launches.fetch_add(1);
            CK(cudaStreamSynchronize(st));   // (hf)
        }
        vfp.ensure((n + 1) * sizeof(int32_t));
        launch(k_col_ptr, dim3((unsigned)std::min<int64_t>(1024, (n + 256) / 256)), dim3(256), 0, st, n, nc,
               (const int32_t*)keys2.as<int32_t>(), vfp.as<int32_t>());
        // L = V - A rows (two passes) and the lumped mass
        deg.ensure(n * sizeof(int32_t));
        const dim3 vg((unsigned)std::min<int64_t>(8 * sms, (n + 127) / 128));
        launch(k_vertex_rows, vg, dim3(128), 0, st, n, (const int32_t*)dF.as<int32_t>(), (const int32_t*)vfp.as<int32_t>(),
               (const int32_t*)fid2.as<int32_t>(), (const double*)cot.as<double>(), (const double*)area.as<double>(), 0,
               deg.as<int32_t>(), (const int64_t*)nullptr, (int32_t*)nullptr, (double*)nullptr, (double*)nullptr,
               bad.as<int>());
        std::vector<int32_t> hdeg(n);
        CK(cudaMemcpyAsync(hdeg.data(), deg.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        int hbad = 0;
        CK(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (hbad & 1) return fail(SBMDS_EINVAL, "degenerate face (zero area: non-finite cotangent)");
        if (hbad & 2) return fail(SBMDS_EINVAL, "a vertex has more than %d neighbours", kSbhaMaxDeg);
        std::vector<int64_t> hlp(n + 1, 0);
        for (int64_t i = 0; i < n; ++i) hlp[i + 1] = hlp[i] + hdeg[i];
        const int64_t nnzL = hlp[n];
        lptr.ensure((n + 1) * sizeof(int64_t));
        lcol.ensure(nnzL * sizeof(int32_t));
        lval.ensure(nnzL * sizeof(double));
        mass.ensure(n * sizeof(double));
        CK(cudaMemcpyAsync(lptr.p, hlp.data(), (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        launch(k_vertex_rows, vg, dim3(128), 0, st, n, (const int32_t*)dF.as<int32_t>(), (const int32_t*)vfp.as<int32_t>(),
               (const int32_t*)fid2.as<int32_t>(), (const double*)cot.as<double>(), (const double*)area.as<double>(), 1,
               deg.as<int32_t>(), (const int64_t*)lptr.as<int64_t>(), lcol.as<int32_t>(), lval.as<double>(),
               mass.as<double>(), bad.as<int>());
        std::vector<int32_t> hlc(nnzL);
        CK(cudaMemcpyAsync(hlc.data(), lcol.p, nnzL * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        // ordering of the free vertices (host) and the bandwidth of M_uu under it
        const int64_t nu = n - l;
        std::vector<int32_t> uvert = rcm_order(n, hlp, hlc, lmpos);   // r -> vertex
        if ((int64_t)uvert.size() != nu) return fail(SBMDS_ECUDA, "internal: RCM ordered %zu of %lld free vertices",
                                                     uvert.size(), (long long)nu);
        std::vector<int32_t> pos(n, -1), uq, qrow;
        for (int64_t r = 0; r < nu; ++r) pos[uvert[r]] = (int32_t)r;
        uq.reserve(nu);
        qrow.reserve(nu);
        for (int64_t i = 0; i < n; ++i)
            if (lmpos[i] < 0) { uq.push_back((int32_t)i); qrow.push_back(pos[i]); }
        int64_t w = 0;
        for (int64_t i = 0; i < n; ++i) {
            if (lmpos[i] >= 0) continue;
            for (int64_t e = hlp[i]; e < hlp[i + 1]; ++e) {
                const int32_t k = hlc[e];
                for (int64_t f = hlp[k]; f < hlp[k + 1]; ++f) {
                    const int32_t j = hlc[f];
                    if (lmpos[j] < 0) w = std::max<int64_t>(w, std::llabs((long long)pos[i] - pos[j]));
                }
            }
        }
        const int64_t W = std::min<int64_t>((w + 1 + 63) / 64 * 64 + 64, (nu + 63) / 64 * 64);
        DevBuf gws{true};   // split-K workspace of the GEMMs below
        DevBuf duv{true}, dpos{true}, dlm{true}, duq{true}, dqrow{true}, B{true}, Wa{true}, Wb{true}, Rp{true},
            XT{true}, selq{true}, selv{true}, cnt{true}, rp{true}, cur{true}, small{true};
        duv.ensure(nu * sizeof(int32_t));
        dpos.ensure(n * sizeof(int32_t));
        dlm.ensure(n * sizeof(int32_t));
        duq.ensure(nu * sizeof(int32_t));
        dqrow.ensure(nu * sizeof(int32_t));
        CK(cudaMemcpyAsync(duv.p, uvert.data(), nu * sizeof(int32_t), cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(dpos.p, pos.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(dlm.p, lmpos.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(duq.p, uq.data(), nu * sizeof(int32_t), cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(dqrow.p, qrow.data(), nu * sizeof(int32_t), cudaMemcpyHostToDevice, st));
        // right-hand sides -M_ub (n_u x l, permuted rows) and max diag of M
        B.ensure((size_t)nu * l * sizeof(double));
        CK(cudaMemsetAsync(B.p, 0, B.bytes, st));
        small.ensure(64);
        CK(cudaMemsetAsync(small.p, 0, 64, st));
        unsigned long long* dmaxbits = small.as<unsigned long long>();
        int* status = reinterpret_cast<int*>(small.as<char>() + 16);
        const dim3 mg((unsigned)std::min<int64_t>(8 * sms, (nu + 127) / 128));
        auto mrows = [&](int64_t r0, int64_t r1, int mode, double* out, int64_t ld, int64_t k0) {
            if (r1 <= r0) return;
            launch(k_m_rows, dim3((unsigned)std::min<int64_t>(8 * sms, (r1 - r0 + 127) / 128)), dim3(128), 0, st, r0, r1,
                   (const int32_t*)duv.as<int32_t>(), (const int32_t*)dpos.as<int32_t>(), (const int32_t*)dlm.as<int32_t>(),
                   (const int64_t*)lptr.as<int64_t>(), (const int32_t*)lcol.as<int32_t>(), (const double*)lval.as<double>(),
                   (const double*)mass.as<double>(), mode, out, ld, k0, W,
                   mode == 0 ? dmaxbits : (unsigned long long*)nullptr, bad.as<int>());
        };
        (void)mg;
        mrows(0, nu, 0, B.as<double>(), l, 0);
        // band Cholesky of M_uu in a sliding W x W window; panel p's rows of R kept in Rp
        const int64_t npan = (nu + 63) / 64;
        Wa.ensure((size_t)W * W * sizeof(double));
        Wb.ensure((size_t)W * W * sizeof(double));
        Rp.ensure((size_t)npan * 64 * W * sizeof(double));
        CK(cudaMemsetAsync(Wa.p, 0, Wa.bytes, st));
        mrows(0, std::min<int64_t>(W, nu), 1, Wa.as<double>(), W, 0);
        double* Wc = Wa.as<double>();
        double* Wn = Wb.as<double>();
        const double* dmax = reinterpret_cast<const double*>(dmaxbits);
        int* dropped = status + 1;
        for (int64_t pn = 0; pn < npan; ++pn) {
            const int64_t k0 = pn * 64;
            const int nb = (int)std::min<int64_t>(64, nu - k0);
            const int64_t Wcur = std::min<int64_t>(W, nu - k0);
            launch(k_potf2, dim3(1), dim3(256), 0, st, Wc, W, 0, nb, status, dmax, dropped, 0);
            if (Wcur > nb) {
                launch(k_trsm_rows, dim3((unsigned)((Wcur - nb + 255) / 256)), dim3(256), 0, st, Wc, W, Wcur, 0, nb,
                       (const int*)status);
                dgemm<true, false>(st, gws, (int)(Wcur - nb), (int)(Wcur - nb), nb, -1.0, Wc + nb, W, Wc + nb, W, 1.0,
                                   Wc + nb * W + nb, W);
            }
            CK(cudaMemcpyAsync(Rp.as<double>() + pn * 64 * W, Wc, (size_t)nb * W * sizeof(double),
                               cudaMemcpyDeviceToDevice, st));
            if (pn + 1 < npan) {   // shift the window by 64 and load the rows entering it
                CK(cudaMemcpy2DAsync(Wn, W * sizeof(double), Wc + 64 * W + 64, W * sizeof(double),
                                     (W - 64) * sizeof(double), W - 64, cudaMemcpyDeviceToDevice, st));
                CK(cudaMemsetAsync(Wn + (W - 64) * W, 0, 64 * W * sizeof(double), st));
                CK(cudaMemset2DAsync(Wn + (W - 64), W * sizeof(double), 0, 64 * sizeof(double), W - 64, st));
                mrows(std::min<int64_t>(nu, k0 + W), std::min<int64_t>(nu, k0 + W + 64), 2, Wn, W, k0 + 64);
                std::swap(Wc, Wn);
            }
        }
        int hs[2] = {0, 0};
        peek_to_host(hs, status, sizeof hs, st);
        if (hs[0] == 2) return fail(SBMDS_EBREAKDOWN, "sBHA: M_uu is not positive definite (a free region without landmarks?)");
        Wa.release();
        Wb.release();
        // X = M_uu^{-1} B: forward R^T Y = B, backward R X = Y, panel by panel
        const unsigned rg = (unsigned)((l + 255) / 256);
        for (int64_t pn = 0; pn < npan; ++pn) {
            const int64_t k0 = pn * 64;
            const int nb = (int)std::min<int64_t>(64, nu - k0);
            const int64_t Wcur = std::min<int64_t>(W, nu - k0);
            const double* R = Rp.as<double>() + pn * 64 * W;
            launch(k_trsm_panel<true>, dim3(rg), dim3(256), 0, st, R, W, nb, B.as<double>() + k0 * l, l, l);
            if (Wcur > nb)
                dgemm<true, false>(st, gws, (int)(Wcur - nb), (int)l, nb, -1.0, R + nb, W, B.as<double>() + k0 * l, l, 1.0,
                                   B.as<double>() + (k0 + nb) * l, l);
        }
        for (int64_t pn = npan - 1; pn >= 0; --pn) {
            const int64_t k0 = pn * 64;
            const int nb = (int)std::min<int64_t>(64, nu - k0);
            const int64_t Wcur = std::min<int64_t>(W, nu - k0);
            const double* R = Rp.as<double>() + pn * 64 * W;
            if (Wcur > nb)
                dgemm<false, false>(st, gws, nb, (int)l, Wcur - nb, -1.0, R + nb, W, B.as<double>() + (k0 + nb) * l, l, 1.0,
                                    B.as<double>() + k0 * l, l);
            launch(k_trsm_panel<false>, dim3(rg), dim3(256), 0, st, R, W, nb, B.as<double>() + k0 * l, l, l);
        }
        Rp.release();
        // per column: the p largest magnitudes over the free vertices (increasing vertex order)
        XT.ensure((size_t)nu * l * sizeof(double));
        launch(k_gather_t, dim3((unsigned)((nu + 31) / 32), (unsigned)((l + 31) / 32)), dim3(256), 0, st, nu, l,
               (const int32_t*)dqrow.as<int32_t>(), (const double*)B.as<double>(), XT.as<double>());
        B.release();
        selq.ensure((size_t)l * p * sizeof(int32_t));
        selv.ensure((size_t)l * p * sizeof(double));
        launch(k_topp, dim3((unsigned)l), dim3(256), 0, st, nu, p, (const double*)XT.as<double>(), selq.as<int32_t>(),
               selv.as<double>());
        XT.release();
        // CSR of S
        const int64_t nnz = l + l * p;
        cnt.ensure(n * sizeof(int32_t));
        CK(cudaMemsetAsync(cnt.p, 0, n * sizeof(int32_t), st));
        dlm.ensure(n * sizeof(int32_t));
        DevBuf dlml{true};
        dlml.ensure(l * sizeof(int32_t));
        CK(cudaMemcpyAsync(dlml.p, lm.data(), l * sizeof(int32_t), cudaMemcpyHostToDevice, st));
        const dim3 eg((unsigned)std::min<int64_t>(8 * sms, (nnz + 255) / 256));
        launch(k_sbha_count, eg, dim3(256), 0, st, l, p, (const int32_t*)dlml.as<int32_t>(), (const int32_t*)duq.as<int32_t>(),
               (const int32_t*)selq.as<int32_t>(), cnt.as<int32_t>());
        std::vector<int32_t> hc(n);
        CK(cudaMemcpyAsync(hc.data(), cnt.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        std::vector<int64_t> hrp(n + 1, 0);
        for (int64_t i = 0; i < n; ++i) hrp[i + 1] = hrp[i] + hc[i];
        rp.ensure((n + 1) * sizeof(int64_t));
        CK(cudaMemcpyAsync(rp.p, hrp.data(), (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        cur.ensure(n * sizeof(int32_t));
        CK(cudaMemsetAsync(cur.p, 0, n * sizeof(int32_t), st));
        DevBuf oc{true}, ov{true};
        oc.ensure(nnz * sizeof(int32_t));
        ov.ensure(nnz * sizeof(float));
        launch(k_sbha_fill, eg, dim3(256), 0, st, l, p, (const int32_t*)dlml.as<int32_t>(), (const int32_t*)duq.as<int32_t>(),
               (const int32_t*)selq.as<int32_t>(), (const double*)selv.as<double>(), (const int64_t*)rp.as<int64_t>(),
               cur.as<int32_t>(), oc.as<int32_t>(), ov.as<float>());
        launch(k_sort_rows, dim3((unsigned)std::min<int64_t>(8 * sms, (n + 255) / 256)), dim3(256), 0, st, n,
               (const int64_t*)rp.as<int64_t>(), oc.as<int32_t>(), ov.as<float>());
        CK(cudaMemcpyAsync(row_ptr, rp.p, (n + 1) * sizeof(int64_t), cudaMemcpyDefault, st));
        CK(cudaMemcpyAsync(col_idx, oc.p, nnz * sizeof(int32_t), cudaMemcpyDefault, st));
        CK(cudaMemcpyAsync(val, ov.p, nnz * sizeof(float), cudaMemcpyDefault, st));
        CK(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (hbad & 4) return fail(SBMDS_EINVAL, "a row of M has more than %d entries", kSbhaMaxRing2);
        if (info) {
            info->nnz = nnz;
            info->p = (int32_t)p;
            info->bandwidth = (int32_t)w;
            info->window = (int32_t)W;
            info->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
    } catch (const CudaError& e) {
        if (e.e == cudaErrorMemoryAllocation) return fail(SBMDS_ENOMEM, "device allocation failed (%s)", e.what);
        return fail(SBMDS_ECUDA, "%s: %s%s", e.what, cudaGetErrorString(e.e), hang_note().c_str());
    }
    return SBMDS_OK;
}

// ============================================================================ options / stats
extern "C" sbmds_status sbmds_set_option(sbmds_t h, const char* key, int64_t value) {
    if (!h || !key) return fail(SBMDS_EINVAL, "NULL handle or key");
    if (!strcmp(key, "rr_period")) {
        if (value < 1) return fail(SBMDS_EINVAL, "rr_period >= 1");
        h->rr_period = (int)value;
    } else if (!strcmp(key, "use_graph")) {
        h->use_graph = value ? 1 : 0;
    } else if (!strcmp(key, "blocked")) {
        if (value < 0 || value > 3) return fail(SBMDS_EINVAL, "blocked is a bit mask in [0, 3]");
        h->use_blocked = (int)value;
        h->blocked_auto = false;
    } else if (!strcmp(key, "csr_shfl")) {
        if (value < -1 || value > 1) return fail(SBMDS_EINVAL, "csr_shfl in {-1 auto, 0, 1}");
        h->csr_shfl = (int)value;
    } else if (!strcmp(key, "gram_tc")) {
        h->gram_tc = value ? 1 : 0;
    } else if (!strcmp(key, "order_columns")) {
        h->order_columns = value ? 1 : 0;
    } else if (!strcmp(key, "profile")) {
        h->prof.mask = (uint32_t)value;
    } else if (!strcmp(key, "profile_reset")) {
        DevGuard g(h->dev);
        h->prof.drain();
        for (int k = 0; k < PK_N; ++k) { h->prof.ns[k] = 0; h->prof.cnt[k] = 0; }
    } else if (!strcmp(key, "dstream")) {
        if (value < 0 || value > 4)
            return fail(SBMDS_EINVAL, "dstream in {0 auto, 1 ffma, 2 tcgen05, 3 symmetric int8, 4 symmetric 2xfp16 pairs}");
        h->dstream = (int)value;
        if ((value == 1 || value == 2 || value == 4) && h->dt8_ok) {
            // off the int8 stream: release its packed D (3 l^2 / 2 bytes); re-packed on return
            DevGuard g(h->dev);
            if (h->pack_st) cudaStreamSynchronize(h->pack_st);
            h->pack_pending = false;
            h->Dt8.release();
            h->dt8_ok = false;
        }
    } else if (!strcmp(key, "dq_max_range")) {
        if (value < 0 || value > 255) return fail(SBMDS_EINVAL, "dq_max_range in [0, 255] binades");
        h->dq_max_range = (int)value;
        if (h->dq_state != 0) h->dq_state = 0;   // re-decided at the next apply / eigs
    } else if (!strcmp(key, "dy_max_range")) {
        if (value < 0 || value > 255) return fail(SBMDS_EINVAL, "dy_max_range in [0, 255] binades");
        h->dy_max_range = (int)value;
    } else if (!strcmp(key, "sp8_max_range")) {
        if (value < 0 || value > 255) return fail(SBMDS_EINVAL, "sp8_max_range in [0, 255] binades");
        h->sp8_max_range = (int)value;   // (read when the sparse-step images are built)
    } else if (!strcmp(key, "center")) {
        h->center = value ? 1 : 0;
    } else if (!strcmp(key, "csr_sub_L")) {
        if (!(value == 0 || value == 1 || value == 2 || value == 4 || value == 8 || value == 16 || value == 32))
            return fail(SBMDS_EINVAL, "csr_sub_L in {0 auto, 1, 2, 4, 8, 16, 32}");
        h->csr_sub_L = (int)value;
    } else if (!strcmp(key, "solver")) {
        if (value < 0 || value > 1) return fail(SBMDS_EINVAL, "solver in {0 subspace iteration, 1 block Lanczos}");
        h->solver = (int)value;
    } else if (!strcmp(key, "lanczos_blocks")) {
        if (value < 0 || value > 32) return fail(SBMDS_EINVAL, "lanczos_blocks in [0, 32] (0: 64 / block)");
        h->lz_blocks = (int)value;
    } else if (!strcmp(key, "sp8_poll")) {
        if (value < 0 || value > 100000) return fail(SBMDS_EINVAL, "sp8_poll must be in [0, 100000] ns");
        h->sp8_poll = (int)value;
    } else if (!strcmp(key, "sp8_apply")) {
        h->sp8_apply = value != 0;
    } else if (!strcmp(key, "sp8_min_rows")) {
        if (value < 0) return fail(SBMDS_EINVAL, "sp8_min_rows must be >= 0");
        h->sp8_min_rows = value;
    } else if (!strcmp(key, "sp8_gram8")) {
        h->sp8_gram8 = value != 0;
    } else if (!strcmp(key, "sp8_pf")) {
        if (value < 0 || value > 15) return fail(SBMDS_EINVAL, "sp8_pf must be in [0, 15] blocks");
        h->sp8_pf = (int)value;
    } else if (!strcmp(key, "sp8_dbg")) {
        h->sp8_dbg = (int)value;
    } else if (!strcmp(key, "fuse")) {
        if (value < 0 || value > 3) return fail(SBMDS_EINVAL, "fuse in {0, 1 Gram, 2 Gram + S^T, 3 tensor-core step}");
        h->fuse = (int)value;
    } else if (!strcmp(key, "pair_dbg")) {
        h->pair_dbg = (int)value;   // bit 0: wait-cycle instrumentation; bits 1..: experiment modes
    } else {
        return fail(SBMDS_EINVAL, "unknown option '%s'", key);
    }
    return SBMDS_OK;
}

extern "C" sbmds_status sbmds_get_stat(sbmds_t h, const char* key, int64_t* value) {
    if (!h || !key || !value) return fail(SBMDS_EINVAL, "NULL argument");
    if (!strcmp(key, "n")) *value = h->n;
    else if (!strcmp(key, "l")) *value = h->l;
    else if (!strcmp(key, "nnz")) *value = h->nnz;
    else if (!strcmp(key, "rowsum_dev_e9")) *value = (int64_t)std::llround(h->rowsum_dev * 1e9);
    else if (!strcmp(key, "d_borrowed")) *value = h->d_borrowed ? 1 : 0;
    else if (!strcmp(key, "blocked_umax")) *value = h->blocked ? (int64_t)h->umax : -1;
    else if (!strcmp(key, "dstream_path")) *value = h->last_dpath;
    else if (!strcmp(key, "d_packed_in_create")) *value = h->pack_ev != nullptr ? 1 : 0;
    else if (!strcmp(key, "dstream_bytes")) *value = h->last_dbytes;
    else if (!strcmp(key, "h2d_bytes")) *value = h->h2d_bytes;
    else if (!strcmp(key, "d_lower_missing")) *value = h->d_lower_missing ? 1 : 0;
    else if (!strncmp(key, "pair_dbg_", 9) && (key[9] == 'N' || key[9] == 'T') && key[10] == '_') {
        const int site = atoi(key + 11);
        if (site < 0 || site > 15) return fail(SBMDS_EINVAL, "pair_dbg site in 0..15");
        *value = (int64_t)std::llround(h->pdbg_avg[key[9] == 'T'][site]);
    }
    else if (!strcmp(key, "blocked_slots")) *value = h->total_u;
    else if (!strcmp(key, "sp8_state")) *value = h->sp8_state;          // tensor-core sparse step: 1 built, -1 n/a, -2 precision check
    else if (!strcmp(key, "sp8_apply_launches")) *value = h->sp8_apply_launches;   // standalone applies whose A5 took it
    else if (!strcmp(key, "sp8_apply_t_launches")) *value = h->sp8_apply_t_launches;   // ... whose A2 took it
    else if (!strcmp(key, "sp8_splits")) *value = h->sp8_splits;   // 128-row blocks halved to fit their images
    else if (!strcmp(key, "sp8_blocks")) *value = h->s8.nblk;
    else if (!strcmp(key, "x_fallbacks")) *value = h->x_fallbacks;   // ... whose X failed the column check
    else if (!strcmp(key, "gram8_launches")) *value = h->gram8_launches;   // eigs steps with the int8 Gram
    else if (!strcmp(key, "sp8_range")) *value = h->sp8_range;          // its binade range (-1 not built)
    else if (!strcmp(key, "chol_retries")) *value = h->chol_retries;
    else if (!strcmp(key, "row_permuted")) *value = h->permuted ? 1 : 0;     // create kept a reordered S
    else if (!strcmp(key, "order_distinct_natural")) *value = h->order_distinct[0];
    else if (!strcmp(key, "order_distinct_permuted")) *value = h->order_distinct[1];
    else if (!strcmp(key, "bmds_dropped")) *value = h->bmds_dropped;  // last BMDS: rank deficiency of J P
    else if (!strcmp(key, "y_fallbacks")) *value = h->y_fallbacks;    // standalone applies sent to the fp32-grade stream  // last eigs: shifted Cholesky retries seen
    else if (!strcmp(key, "dq_state")) *value = h->dq_state;            // int8 D stream check: 1 kept, -1 fell back, 0 undecided
    else if (!strcmp(key, "dq_range")) *value = h->dq_range;            // binades between max |D| and the median |D|
    else if (!strcmp(key, "sp8_bytes")) *value = h->s8_bytes;           // its S images (HBM bytes per pass)
    else if (!strcmp(key, "sp8_umax")) *value = h->sp8_state > 0 ? (int64_t)h->s8.umax : -1;
    else if (!strcmp(key, "dstream_slots")) *value = h->s8plan[1].nslots;   // int8 D stream partial slots (b = 16)
    else if (!strcmp(key, "sp8_slots")) *value = h->sp8_state > 0 ? (int64_t)h->s8.total_u : -1;   // 128-row dictionary entries
    else if (!strncmp(key, "sp8_trace_", 10)) {   // (diagnostics, sp8_dbg & 2) event timestamps of CTA 0
        const int k = atoi(key + 10);
        if (k < 0 || k >= 2048 + 8 * 64 || !h->s8trace.p) return fail(SBMDS_EINVAL, "no sp8 trace");
        unsigned long long v = 0;
        if (cudaMemcpy(&v, h->s8trace.as<unsigned long long>() + k, sizeof v, cudaMemcpyDeviceToHost) != cudaSuccess)
            return fail(SBMDS_ECUDA, "sp8 trace read");
        *value = (int64_t)v;
    }
    else if (!strcmp(key, "csc_bytes")) *value = (int64_t)(h->cptr.bytes + h->ridx.bytes + h->cval.bytes);
    else if (!strcmp(key, "workspace_bytes"))
        *value = (int64_t)(h->Y1.bytes + h->Y2.bytes + h->P.bytes + h->X.bytes + h->Y.bytes + h->gpart.bytes);
    else {
        for (int k = 0; k < PK_N; ++k) {
            const std::string nm(kProfNames[k]);
            if (key == nm + "_ns" || key == nm + "_launches") {
                DevGuard g(h->dev);
                h->prof.drain();
                *value = (key == nm + "_ns") ? (int64_t)std::llround(h->prof.ns[k]) : h->prof.cnt[k];
                return SBMDS_OK;
            }
        }
        return fail(SBMDS_EINVAL, "unknown stat '%s'", key);
    }
    return SBMDS_OK;
}
