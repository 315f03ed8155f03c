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
 *     small convergence flag back every rr_period iterations; the first call of a handle
 *     reads D's precision check back once; a standalone apply on the int8 stream reads
 *     its Y1 column check back, and at b = 16 on the tensor-core sparse kernels X's column
 *     check, unless "dy_max_range" >= 64).
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
    SBMDS_VALIDATE = 1u << 1,
    /* Let create reorder S's rows: sorted by their two smallest column indices, the order is
       kept internally when sampled 128-row blocks then touch < 3/4 of the landmarks (stat
       "row_permuted"); X, Y, X0, V and Z keep the caller's order (the handle permutes at the
       boundary). Off by default: measured slower with the current sparse kernels on every
       config (DESIGN.md §4 "Row order"). */
    SBMDS_REORDER_ROWS = 1u << 2
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
 * With a host D large enough for the int8 stream, create returns while that stream's packing of
 * D (and max |D|) may still run on a handle-owned stream: every later D-stream launch waits on its
 * event until it has completed, and a fault in it is reported by the call that first waits.
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

/*
 * sbmds_bmds — BMDS, the paper's QR route to the same eigenpairs (§3.3):
 * Q R = J P, -1/2 R W R^T = V~ Λ V~^T, Z = Q V~_m Λ_m^{1/2}, for small l (SURVEY §8(f) NEXT-3b;
 * SPEC.md:455 asks for the BMDS / sBMDS path equivalence). On the device in fp64: the Gram
 * (J P)^T J P from the dense n x l J P (the O(nl) memory the paper notes), its upper Cholesky
 * factor R (= the R of QR = J P up to column signs), M = -1/2 R W R^T, the top-m algebraic
 * eigenpairs of the l x l M by block subspace iteration (block, max_iters, tol, seed as in
 * sbmds_eigs, Rayleigh-Ritz every rr_period iterations), then V = J P R^{-1} V~_m (Q is never
 * stored) and Z = V Λ^{1/2} with sbmds_eigs' sign rule. M has the nonzero spectrum of B~ (the
 * rest of B~'s spectrum is 0), so the top-m agree with sbmds_eigs whenever B~ has >= m
 * positive eigenvalues.
 *   Limits: l <= 8192, n l <= 2e9, 1 <= m <= block <= min(64, l). V, Z DEVICE (or NULL).
 *   info->n_applies = 0 (no operator applies). SBMDS_EBREAKDOWN when J P is rank-deficient
 *   (e.g. a landmark column of S with no entries); SBMDS_ENOCONV as sbmds_eigs.
 */
sbmds_status sbmds_bmds(sbmds_t h, int32_t m, int32_t block, int32_t max_iters, double tol, uint64_t seed,
                        double* eigvals, float* V, float* Z, sbmds_info* info, void* cuda_stream);

/*
 * sBHA build: the sparse biharmonic interpolation operator
 * S = P_sparse of a triangle mesh, the input of sbmds_create (§2.2, §3, §3.1):
 *   A_ij = (cot α_ij + cot β_ij) / 2 (a boundary edge: its one cotangent / 2),
 *   D_ii = 1/3 of the area of the faces incident on i, V = diag(A 1),
 *   M = (V - A)^T D^{-1} (V - A),
 *   P = [I_l ; P_u], P_u = -M_uu^{-1} M_ub (Eq. 6; landmark rows are e_t),
 *   each column of P_u keeps its p largest magnitudes (PAPER.md:175-191 thresholding; ties to
 *   the lowest vertex index, kept values unchanged), p = sbmds_sbha_p(n, l, p_row)
 *   = clamp(ceil((n - l) p_row / l), 1, n - l) (ceiling per SPEC.md:380).
 * Computed on the device in fp64: cotangents and masses per face / vertex, M's rows on the fly,
 * a band Cholesky of M_uu after a reverse Cuthill-McKee ordering of the free vertices (host),
 * the l right-hand sides solved panel by panel, a radix select per column.
 *   verts   : double[n*3] (host or device), faces: int32[nf*3] (host or device), vertex
 *             indices in [0, n), no zero-area face (SBMDS_EINVAL otherwise).
 *   landmarks: int32[l], distinct, in [0, n), 1 <= l < n.
 *   row_ptr : int64[n+1], col_idx: int32[nnz], val: float[nnz] (host or device) receive S in
 *             CSR (columns ascending per row), nnz = l + l p exactly (info->nnz).
 * SBMDS_EBREAKDOWN when M_uu is not positive definite (a connected region of free vertices
 * without a landmark); SBMDS_EINVAL when a vertex has more than 64 neighbours or a row of M
 * more than 256 entries.
 */
typedef struct {
    int64_t nnz;        /* stored entries of S = l + l p */
    int32_t p;          /* kept entries per column of P_u */
    int32_t bandwidth;  /* half-bandwidth of M_uu under the ordering */
    int32_t window;     /* rows of the dense band-Cholesky window */
    double seconds;     /* host wall time of the call */
} sbmds_sbha_info;
int64_t sbmds_sbha_p(int64_t n, int64_t l, double p_row);
sbmds_status sbmds_sbha_build(int64_t n, const double* verts, int64_t nf, const int32_t* faces, int64_t l,
                              const int32_t* landmarks, double p_row, int64_t* row_ptr, int32_t* col_idx,
                              float* val, sbmds_sbha_info* info, void* cuda_stream);

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
 *                      digit images of blocks of <= 128 consecutive rows of S) where it applies
 *                      -- b = 16, or b = 32 as two 16-column passes, and every block touching
 *                      <= 128 landmarks after the build has halved the blocks that do not (stat
 *                      "sp8_splits") -- else as 1
 *     "sp8_gram8"      (0/1, default 1) eigs on the tensor-core step: steps whose Gram only feeds
 *                      the next Cholesky-QR (neither a Rayleigh-Ritz step nor the one before it)
 *                      take G = Y^T Y and 1^T Y from Y's 24-bit digits on the int8 tensor cores
 *                      (exact integer sums) instead of the FP64 Gram of the fp32 rows (stat
 *                      "gram8_launches")
 *     "sp8_apply"      (0/1, default 1) standalone sbmds_apply at b = 16 where the tensor-core
 *                      step applies: A2 = S^T X as its T products (unless X fails the column
 *                      check of "dy_max_range": stat "x_fallbacks") and A5 as its N products
 *                      (stats "sp8_apply_t_launches", "sp8_apply_launches"); 0 keeps the fp32
 *                      CSC / row-blocked CSR kernels
 *     "sp8_min_rows"   (default 303,104 = 16 blocks of 128 rows per SM) the standalone apply takes
 *                      the tensor-core sparse kernels only from this many rows on: their fixed
 *                      costs per launch lose to the fp32 SpMMs on small problems (config 2,
 *                      n = 100,000: 0.125 vs 0.087 ms per apply at b = 32); 0 = always where they
 *                      apply (sbmds_eigs takes them at any size: there they replace several kernels)
 *     "csr_shfl"       (-1 auto / 0 / 1) fp32 CSR SpMM at b in {4, 8, 16, 32, 64}: a group's (column,
 *                      value) pairs loaded once and broadcast by shuffles (same sums bit for bit);
 *                      auto: b <= 16 or a mean row of >= b entries (measured on config 5)
 *     "sp8_pf"         (blocks, default 0) tensor-core step: L2 prefetch distance of the images
 *                      (measured: no gain)
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
 *     "dq_max_range"   (binades, default 6) precision check of the int8 D stream: auto keeps it only
                      while the median |D| over the upper tiles lies within this many binades of
                      max |D| (stat "dq_range"); otherwise the full D on 3xTF32 (stat "dq_state" -1)
     "dy_max_range"   (binades, default 3) standalone apply on the int8 stream: a Y1 column whose
                      max |y| exceeds 2^range times its rms sends that apply to the fp32-grade
                      stream (stat "y_fallbacks"); likewise a column of X for the tensor-core A2
                      (stat "x_fallbacks": that apply's S^T X stays on the fp32 CSC kernel); each
                      check reads 0.8 KB back (a stream sync), >= 64 turns both off (no host
                      sync: the apply can then be graph-captured; A2 then stays on the CSC kernel)
     "sp8_max_range"  (binades, default 7) tensor-core sparse step: a 128-row block whose smallest
                      nonzero row maximum sits more than this many binades below the block's max
                      keeps the eigs step on the fp32 sparse kernels (stat "sp8_state" -2,
                      "sp8_range"); read when the images are built
     "pair_dbg"       diagnostics of k_dstream_pair: bit 0 per-role wait-cycle counters
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
/* The same for blocks of SR x SC tiles (k_dstream_sym8 walks SR = 9, SC = 1 at b = 16: a column
   accumulator becomes a partial once per SR tiles, so tall one-tile-wide blocks write the fewest
   partials) and for the tile range of `rank` in `world` (sharded apply). */
int64_t sbmds_plan_selfcheck_rect(int64_t l, int32_t SR, int32_t SC, int32_t gN, int32_t max_ctas, int32_t contiguous,
                                  int32_t rank, int32_t world);

/* Host logic of the tensor-core sparse kernels' blocks (no GPU; used by the CPU tests; DESIGN.md §4
   "Blocks as row ranges"): one round of splitting. Block B is the row range [r0[B], r0[B + 1]) of S
   (the operator is local, so consecutive vertices share landmarks) and touches
   dsize[B] distinct landmarks; a block over `limit` (128 in the library: one image holds 128
   landmark columns) is halved at a multiple of 4 rows from its start. r0_out receives the new
   boundaries (at most `capacity` entries); returns the new block count, -1 when a block over the
   limit has fewer than 8 rows, -2 for bad arguments or too small a capacity. */
int64_t sbmds_sparse_split_rows(int64_t n, int64_t nblk, const int32_t* r0, const int32_t* dsize, int32_t limit,
                             int32_t* r0_out, int64_t capacity);

/*
 * Sharded apply. The matvec of PAPER.md:221-222 splits by rows of P (= S)
 * and by tiles of W (= D_ll): rank g of `world` holds rows [row0, row0 + n_local) of S and
 * streams the contiguous range g of D's upper 128 x 128 tiles in walk order (sbmds_shard_tiles).
 * Every exchanged quantity is linear, so the apply is four stages with a SUM over ranks after
 * each of the first three:
 *   stage 0  in: X_g (n_local x b)          out: s_g = 1^T X_g              (double[b])
 *   stage 1  in: X_g, s (summed, double[b])  out: Y1_g = S_g^T X_g - w_g s^T (float[l*b]),
 *            w_g = S_g^T 1 / n_global (the w_g sum to w = S^T 1 / n)
 *   stage 2  in: Y1 (summed, float[l*b])     out: Y2_g (float[l*b]) and, at byte offset
 *            8*ceil(4lb/8), t_g = (D w_g)^T Y1 (double[b]; sums to t = w^T D Y1 = w^T Y2
 *            with no further exchange; D w_g is formed once): this rank's tiles' D_IJ Y1_J and
 *            D_IJ^T Y1_I terms (full-D kernels -- b < 5, or the precision fallback -- run
 *            on rank 0 only; the other ranks return zeros)
 *   stage 3  in: Y2 | t (summed, stage 2's layout)   out: Y_g = -1/2 (S_g Y2 - 1 t^T) (n_local x b)
 * Layouts are compact row-major (float[l*b]: row j of Y1 at j*b). sbmds_shard_exchange_bytes
 * gives each stage's exchange size (stage 1: its output; 2, 3: the Y2 | t buffer).
 *
 * sbmds_create_shard — as sbmds_create for the local rows (row_ptr is local: row_ptr[0] = 0,
 *   row_ptr[n_local] = nnz); D_ll is the full l x l matrix on every rank. 1 <= l <= n_global,
 *   0 <= row0, row0 + n_local <= n_global, 0 <= rank < world. sbmds_apply and sbmds_eigs on a
 *   shard handle need an attached communicator when world > 1 (SBMDS_EINVAL otherwise). On a
 *   shard, sbmds_eigs runs the block subspace iteration on the rank's rows (X0, V, Z are the
 *   rank's n_local x b / x m rows): the sharded apply with the R^{-1} fold, the Grams summed over
 *   the ranks (every rank factors and solves the same small problems), the sign rule over all
 *   rows; every rank must call it with the same arguments. The Lanczos solver and sbmds_bmds
 *   reject shard handles.
 * sbmds_shard_stage — one stage on DEVICE buffers, stream-ordered (a standalone stage 2 on the
 *   int8 stream reads a small Y1 check back). X for stages 0-1, exch_in for 1-3, exch_out for
 *   0-2, Y for 3; the others may be NULL.
 * sbmds_nccl_unique_id / sbmds_shard_attach_nccl — NCCL (dlopen'ed "libnccl.so.2" on first use):
 *   rank 0 creates the 128-byte id, the caller broadcasts it, and every rank attaches
 *   (collective: ncclCommInitRank(world, id, rank) blocks until all ranks have joined). After
 *   that sbmds_apply runs all four stages with ncclAllReduce(sum) on the call's stream. The
 *   handle owns the communicator (freed by sbmds_destroy). SBMDS_ECUDA when NCCL is missing.
 * sbmds_shard_plan_selfcheck / sbmds_shard_tiles (host only, no GPU): rank's schedule checked as
 *   sbmds_plan_selfcheck does; rank's tiles (I << 16 | J) into tiles_out[capacity] (may be NULL),
 *   returning their count (< 0: bad arguments).
 */
sbmds_status sbmds_create_shard(int64_t n_global, int64_t row0, int64_t n_local, int64_t l, int64_t nnz,
                                const int64_t* row_ptr, const int32_t* col_idx, const float* val,
                                const float* D_ll, int32_t rank, int32_t world, uint32_t flags,
                                void* cuda_stream, sbmds_t* out);
sbmds_status sbmds_shard_stage(sbmds_t h, int32_t stage, int32_t b, const float* X, const void* exch_in,
                               void* exch_out, float* Y, void* cuda_stream);
int64_t sbmds_shard_exchange_bytes(int64_t l, int32_t b, int32_t stage);
sbmds_status sbmds_nccl_unique_id(void* id_out /* 128 bytes */);
sbmds_status sbmds_shard_attach_nccl(sbmds_t h, const void* unique_id /* 128 bytes */);
int64_t sbmds_shard_plan_selfcheck(int64_t l, int32_t S, int32_t gN, int32_t max_ctas, int32_t contiguous,
                                   int32_t rank, int32_t world);
int64_t sbmds_shard_tiles(int64_t l, int32_t S, int32_t rank, int32_t world, uint32_t* tiles_out,
                          int64_t capacity);

/* ABI version: 2 (1 + the sharded apply). */
int32_t sbmds_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SBMDS_H */
