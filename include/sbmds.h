/*
 * sbmds.h — C ABI of the B200-native sBMDS hot path (libsbmds.so).
 *
 * Sparse biharmonic MDS (Turek & Huth, arXiv 1705.10887): classical scaling on the
 * factored squared-distance approximation  Ê = P W P^T  (Eq. 7),
 * where P = S is the n x l sparse interpolation operator (Eq. 6,
 * sparsified per PAPER.md:175-191) and W = D_ll the l x l landmark block
 * (PAPER.md:149), already squared for MDS (reading R2).
 *
 *   operator   B~ = -1/2 J S D_ll S^T J,   J = I - (1/n) 1 1^T
 *   eigs       top-m algebraic eigenpairs of B~ and Z = V_m Λ_m^{1/2},
 *              "using only matrix-vector multiplications" — here a
 *              block subspace iteration with Cholesky-QR and Rayleigh-Ritz
 *              (BASELINE.json north_star) instead of the paper's Lanczos.
 *
 * Conventions for every entry point
 *   - Pointer arguments may be HOST or DEVICE memory (detected per call with
 *     cudaPointerGetAttributes). Host inputs are staged through library-owned device
 *     buffers and the call synchronises `cuda_stream` before returning; with all
 *     pointers on the device the call is asynchronous on `cuda_stream` (eigs reads a
 *     small convergence flag back every rr_period iterations).
 *   - `cuda_stream` is a cudaStream_t (NULL = legacy default stream).
 *   - Dense blocks (X, Y, V, Z) are row-major n x b fp32: the b values of vertex i
 *     are contiguous at offset i*b.
 *   - Errors never abort: a non-OK status is returned and sbmds_last_error() gives a
 *     thread-local message. Invalid arguments leave the handle unchanged.
 *   - One handle serialises its own calls (shared workspace); distinct handles are
 *     independent and may be used from different threads.
 */
#ifndef SBMDS_H
#define SBMDS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sbmds_ctx* sbmds_t; /* opaque handle */

typedef enum {
    SBMDS_OK = 0,
    SBMDS_EINVAL = 1,     /* bad argument (sizes, ranges, NULL, overlap, asymmetric D) */
    SBMDS_ENOMEM = 2,     /* device allocation failed */
    SBMDS_ECUDA = 3,      /* CUDA runtime/driver error (message in sbmds_last_error) */
    SBMDS_ENOCONV = 4,    /* eigs hit max_iters with tol > 0; outputs and info still filled */
    SBMDS_EBREAKDOWN = 5  /* Cholesky-QR broke down even after the shifted retry */
} sbmds_status;

enum {
    /* Keep a reference to the caller's DEVICE D_ll instead of copying it (the caller
       keeps it alive and unchanged until sbmds_destroy). Ignored for host D, or when
       l % 4 != 0 (TMA needs 16-byte row pitch; the library then copies). */
    SBMDS_BORROW_D = 1u << 0,
    /* Full input checks at create: row_ptr monotone with row_ptr[0] = 0 and
       row_ptr[n] = nnz, 0 <= col_idx < l, all values finite, D symmetric
       (|D_ij - D_ji| <= 1e-6 max|D|). Without it only sizes are checked. */
    SBMDS_VALIDATE = 1u << 1
};

typedef struct {
    int32_t iters;        /* subspace iterations run */
    int32_t n_applies;    /* operator applies (= iters) */
    int32_t n_negative;   /* negative eigenvalues among the top m (their Z column is 0) */
    int32_t converged;    /* 1 if max_i<m r_i <= tol*|θ|max (always 0 when tol <= 0) */
    double max_residual;  /* max_i<m ||B~v_i - θ_i v_i|| / max_j |θ_j| at the last RR */
    double orth_error;    /* max |V^T V - I| of the returned V (fp64 Gram)           */
    double gpu_ms;        /* device time of the whole call (CUDA events)             */
} sbmds_info;

/*
 * sbmds_create — build a handle from S (CSR) and D_ll.
 *   n, l, nnz   : S is n x l with nnz stored entries; 1 <= l <= n, 0 <= nnz < 2^31.
 *   row_ptr     : int64[n+1], row_ptr[0] = 0, row_ptr[n] = nnz, nondecreasing.
 *   col_idx     : int32[nnz], 0 <= col < l; any order within a row; duplicates summed.
 *   val         : float[nnz]. No sign or row-sum assumption (the paper's thresholded
 *                 P_sparse has neither).
 *   D_ll        : float[l*l], row-major, symmetric ("d_M is symmetric";
 *                 W_ij = d(b_i, b_j)), squared distances (R2).
 *                 The kernels read D as D^T, which equals D for symmetric input.
 *   flags       : SBMDS_BORROW_D | SBMDS_VALIDATE.
 * The library copies S (and D unless borrowed) into device memory it owns, builds a
 * row-sorted CSC copy of S on the device (for S^T X without atomics) and the vector
 * w = S^T 1 / n used by the rank-one centring (J S = S - 1 w^T).
 * Returns SBMDS_OK and *out, or an error with *out = NULL.
 */
sbmds_status sbmds_create(int64_t n, int64_t l, int64_t nnz, const int64_t* row_ptr,
                          const int32_t* col_idx, const float* val, const float* D_ll,
                          uint32_t flags, void* cuda_stream, sbmds_t* out);

/*
 * sbmds_apply — Y = -1/2 J S D_ll S^T J X.
 *   b    : block width, 1 <= b <= 64.
 *   X, Y : n x b row-major fp32, host or device; must not overlap. X is not modified.
 * Computed as s = 1^T X, Y1 = S^T X - w s^T, Y2 = D Y1, t = w^T Y2,
 * Y = -1/2 (S Y2 - 1 t^T): no n-length centred copy is formed.
 */
sbmds_status sbmds_apply(sbmds_t h, int32_t b, const float* X, float* Y, void* cuda_stream);

/*
 * sbmds_eigs — top-m algebraic eigenpairs of B~ and the embedding Z = V_m Λ_m^{1/2}
 * ("truncating its decomposition to the biggest m eigenvalues").
 *   m          : 1 <= m <= block.
 *   block      : subspace width b, m <= b <= 64, b < n. Subspace iteration converges to
 *                the largest |λ|, so b must also cover the negative eigenvalues with
 *                |λ| > λ_m (reading R1).
 *   max_iters  : >= 1 subspace iterations (one apply each).
 *   tol        : > 0: stop when max_i<m ||B~v_i - θ_i v_i|| <= tol * max_j |θ_j|
 *                (SPEC.md:52 form), checked every rr_period (default 5) iterations;
 *                <= 0: run exactly max_iters iterations (status OK); Rayleigh-Ritz then runs
 *                once, after the last iteration (it only feeds the convergence test).
 *   seed       : initial block X0 ~ N(0,1) from a counter-based Philox generator.
 *   X0         : optional n x block warm start (host or device), or NULL.
 *   eigvals    : HOST double[m], descending.
 *   V, Z       : n x m fp32 (host or device), or NULL to skip. V orthonormal columns;
 *                each column's largest-|v_i| entry is positive (ties: lowest i);
 *                Z column j = sqrt(max(θ_j, 0)) V_j (negative θ_j -> zero column).
 *   info       : HOST sbmds_info*, or NULL.
 * Returns SBMDS_OK, SBMDS_ENOCONV (results filled), SBMDS_EBREAKDOWN, or an error.
 */
sbmds_status sbmds_eigs(sbmds_t h, int32_t m, int32_t block, int32_t max_iters, double tol,
                        uint64_t seed, const float* X0, double* eigvals, float* V, float* Z,
                        sbmds_info* info, void* cuda_stream);

/* Frees everything the library allocated (not borrowed D). NULL-safe. */
void sbmds_destroy(sbmds_t h);

/* Thread-local message for the last non-OK status on this thread ("" if none). */
const char* sbmds_last_error(void);

/*
 * Tuning / introspection (tests and bench). Options change how, never what, is computed.
 *   sbmds_set_option keys:
 *     "rr_period"      (>= 1) Rayleigh-Ritz every r iterations (default 5)
 *     "use_graph"      (0/1)
 *     "order_columns"  (0/1) spatial CSC column order for the S^T X gathers
 *     "dstream"        D-stream kernel for A3: 0 auto (symmetric half as 24-bit fixed point on
 *                      the int8 tensor cores when b in 5..32 and D has >= 8 tiles per 2 SMs,
 *                      else full-D tcgen05 for b >= 5, else FFMA), 1 FFMA, 2 full-D tcgen05
 *                      3xTF32, 3 symmetric half int8 (k_dstream_sym8), 4 symmetric half 2xFP16
 *                      on CTA pairs (k_dstream_pair; b in 5..32, else as 2)
 *     "blocked"        bit mask: 1 = S Y2 through the row-blocked kernel, 2 = S^T X too
 *     "gram_tc"        (0/1) Gram on the FP64 tensor cores (b <= 32)
 *     "center"         (0/1, default 1) 0: sbmds_apply returns the uncentred E^ X = S D S^T X
 *                      (the BHA approximation of the squared-distance matrix;
 *                      its rows are what the error estimate of PAPER.md:309/317 compares);
 *                      sbmds_eigs always uses the centred operator
 *     "fuse"           eigs: 0 separate kernels, 1 A5 fused with the Gram, 2 also the next
 *                      apply's S^T partials, 3 (default) the tensor-core sparse step
 *                      (k_sp8.cuh: A5 + Grams + next A2 on the int8 tensor cores from dense
 *                      128-row digit images of S) where it applies -- b = 16 and every
 *                      128-row block touching <= 128 landmarks -- else as 1
 *     "solver"         eigs: 0 (default) block subspace iteration; 1 restarted block Lanczos with
 *                      full reorthogonalisation (block <= 32, k
 *                      blocks of b per cycle with k b <= 64; max_iters counts block applies)
 *     "lanczos_blocks" blocks per Lanczos cycle (0 = 64 / block, at least 2)
 *     "sp8_dbg"        diagnostics of the tensor-core step (timing only; bits 1, 4, 8, 16 make
 *                      results invalid): 1 skip the T product, 2 record a timeline of CTA 0
 *                      (stats "sp8_trace_<event * 64 + block>"; entries 768 + c / 1024 + c /
 *                      1280 + c: CTA c's start / roles done / Gram partials written, 1277-1279
 *                      the last CTA's Gram sums and Cholesky), 4 stream the images only,
 *                      8 T product in the last iteration too, 16 no H' term; valid-result
 *                      switches: 64 Y2's digit planes by a separate k_y2_digits instead of the
 *                      cooperative reduce, 128 Gram sums + Cholesky in the step's last CTA on
 *                      every step (not deferred to the next fold)
 *     "use_graph"      (0/1, default 0) eigs: replay Rayleigh-Ritz segments from CUDA graphs
 *     "profile"        bit mask of kernel families timed with CUDA events on the launching
 *                      stream (bit k = family k of: colsum csc dstream dreduce csr gram chol
 *                      rotate rr split); "profile_reset" (any value) zeroes the counters
 *     "pair_dbg"       diagnostics of k_dstream_pair: bit 0 per-role wait-cycle counters
 *                      (stats "pair_dbg_N_<site>", "pair_dbg_T_<site>"), higher bits disable
 *                      parts of the kernel for experiments (results then invalid)
 *   sbmds_get_stat keys: "n", "l", "nnz", "rowsum_dev_e9" (max |row sum - 1| * 1e9),
 *     "d_borrowed", "csc_bytes", "workspace_bytes", "blocked_umax" (largest per-block
 *     landmark dictionary, -1 if the row-blocked structure is off), "blocked_slots",
 *     "dstream_path" (1 FFMA, 2 full-D tcgen05, 3 symmetric half; of the last apply),
 *     "d_packed_in_create" (1: a host D was packed for the int8 stream by create, on a handle
 *     stream the first D-stream launch waits for),
 *     "dstream_bytes" (its algorithmic bytes per launch), "sp8_state" (tensor-core step: 1
 *     built, -1 not applicable, 0 not tried yet), "sp8_bytes" (its S images), "sp8_umax"
 *     (largest 128-row dictionary), "<family>_ns" / "<family>_launches"
 *     (profiled device time in ns / launch count per family since the last reset).
 * Both return SBMDS_EINVAL for an unknown key.
 */
sbmds_status sbmds_set_option(sbmds_t h, const char* key, int64_t value);
sbmds_status sbmds_get_stat(sbmds_t h, const char* key, int64_t* value);

/* Number of kernels this library has launched in this process (graph replays count
   each captured kernel). Monotone; for bench.py's gpu_launches. */
int64_t sbmds_launch_count(void);

/* Diagnostics (host only, no GPU needed): builds the symmetric-half D-stream schedule for l,
   block edge S (1..16), row-accumulator group gN (>= 1), at most max_ctas CTAs (or CTA pairs),
   contiguous slot layout (0/1), replays the kernels' accumulate/flush rules against it and
   returns the number of violated invariants (0 = consistent; < 0 = bad arguments). Used by the
   CPU tests; see k_dstream_sym8.cuh / k_dstream_pair.cuh and DESIGN.md §4. */
int64_t sbmds_plan_selfcheck(int64_t l, int32_t S, int32_t gN, int32_t max_ctas, int32_t contiguous);

/* ABI version: 1. */
int32_t sbmds_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SBMDS_H */
