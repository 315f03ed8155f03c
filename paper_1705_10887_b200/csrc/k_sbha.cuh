// sBHA build on the GPU: the sparse biharmonic interpolation operator
// S = P_sparse from a triangle mesh and its landmarks (§2.2, §3, §3.1):
//   A_ij = (cot α_ij + cot β_ij) / 2, D_ii = 1/3 incident area,
//   L = V - A, M = L^T D^{-1} L,
//   P_u = -M_uu^{-1} M_ub (Eq. 6), each column thresholded to its p largest
//   magnitudes, p = ceil((n - l) p_row / l).
// The solve is a direct band (envelope) Cholesky of M_uu in fp64 after a reverse Cuthill-McKee
// ordering of the free vertices (host, sbmds.cu): a sliding dense window of W = w + 64 rows
// (w = the ordered bandwidth of M_uu) is factored 64 columns at a time with the BMDS panel
// kernels (k_potf2 / k_trsm_rows / k_dgemm, k_bmds.cuh) and each panel's 64 x W rows of R are
// kept; the l right-hand sides are then solved panel by panel (forward and backward, a GEMM
// against the stored rows plus a 64 x 64 triangular solve). Kernels here:
//   k_face_geom     per face: the three corner cotangents and the area (degenerate -> flag)
//   k_vertex_rows   per vertex, incident faces in face order: A's row (sorted neighbours), mass,
//                   V_i = sum_j A_ij (pass 0 counts, pass 1 writes L = V - A with the diagonal)
//   k_m_rows        rows of M = L D^{-1} L (per row, k then j ascending: deterministic, symmetric)
//                   scattered into the window (and its mirror) or the right-hand sides -M_ub
//   k_trsm_panel    64 x 64 triangular solves with R_kk (forward / backward) for all l right-hand sides
//   k_gather_t      X (permuted rows x l) -> XT (l x free vertices in increasing order)
//   k_topp          per column: radix select of the p-th largest |x|, ties to the lowest row
//   k_sbha_count / k_sbha_fill / k_sort_rows   the CSR of S (landmark rows e_t + kept entries)
#pragma once
#include "common.cuh"

namespace sbmds {

constexpr int kSbhaMaxDeg = 64;     // 1-ring neighbours per vertex
constexpr int kSbhaMaxRing2 = 256;  // 2-ring entries of one row of M

__global__ void __launch_bounds__(256) k_face_geom(int64_t nf, const double* __restrict__ V,
                                                   const int32_t* __restrict__ F, double* __restrict__ cot,
                                                   double* __restrict__ area, int* __restrict__ bad) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
        const int32_t t[3] = {F[3 * f], F[3 * f + 1], F[3 * f + 2]};
        // corner k opposite edge (i, j): (a, b | c), (b, c | a), (c, a | b) -> cot[0] for edge ab, ...
        for (int e = 0; e < 3; ++e) {
            const int32_t i = t[e], j = t[(e + 1) % 3], k = t[(e + 2) % 3];
            const double ux = V[3 * i] - V[3 * k], uy = V[3 * i + 1] - V[3 * k + 1], uz = V[3 * i + 2] - V[3 * k + 2];
            const double wx = V[3 * j] - V[3 * k], wy = V[3 * j + 1] - V[3 * k + 1], wz = V[3 * j + 2] - V[3 * k + 2];
            const double cx = uy * wz - uz * wy, cy = uz * wx - ux * wz, cz = ux * wy - uy * wx;
            const double c = (ux * wx + uy * wy + uz * wz) / sqrt(cx * cx + cy * cy + cz * cz);
            if (!isfinite(c)) atomicOr(bad, 1);
            cot[3 * f + e] = c;
            if (e == 0) area[f] = 0.5 * sqrt(cx * cx + cy * cy + cz * cz);
        }
    }
}

// One thread per vertex i. pass 0: deg[i] = number of distinct neighbours (+ 1 for the diagonal);
// pass 1: L row i at lptr[i] (columns ascending, the diagonal V_i = sum_j A_ij in ascending j),
// mass[i] = sum of area / 3 over incident faces in face order.
__global__ void __launch_bounds__(128) k_vertex_rows(int64_t n, const int32_t* __restrict__ F,
                                                     const int32_t* __restrict__ vf_ptr, const int32_t* __restrict__ vf,
                                                     const double* __restrict__ cot, const double* __restrict__ area,
                                                     int pass, int32_t* __restrict__ deg, const int64_t* __restrict__ lptr,
                                                     int32_t* __restrict__ lcol, double* __restrict__ lval,
                                                     double* __restrict__ mass, int* __restrict__ bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t nb[kSbhaMaxDeg];
        double w[kSbhaMaxDeg];
        int cnt = 0;
        double m = 0.0;
        for (int32_t q = vf_ptr[i]; q < vf_ptr[i + 1]; ++q) {
            const int32_t f = vf[q];
            const int32_t t[3] = {F[3 * f], F[3 * f + 1], F[3 * f + 2]};
            m += area[f] / 3.0;
            for (int e = 0; e < 3; ++e) {   // edge e = (t[e], t[e+1]) carries cot[3f + e] / 2
                const int32_t a = t[e], b = t[(e + 1) % 3];
                int32_t j = -1;
                if (a == i) j = b;
                else if (b == i) j = a;
                if (j < 0) continue;
                const double half = cot[3 * f + e] / 2.0;
                int s = 0;
                while (s < cnt && nb[s] != j) ++s;
                if (s == cnt) {
                    if (cnt == kSbhaMaxDeg) { atomicOr(bad, 2); break; }
                    nb[cnt] = j;
                    w[cnt] = 0.0;
                    ++cnt;
                }
                w[s] += half;
            }
        }
        if (pass == 0) {
            deg[i] = cnt + 1;
            continue;
        }
        // insertion sort by column
        for (int a = 1; a < cnt; ++a) {
            const int32_t kj = nb[a];
            const double kw = w[a];
            int b = a - 1;
            while (b >= 0 && nb[b] > kj) { nb[b + 1] = nb[b]; w[b + 1] = w[b]; --b; }
            nb[b + 1] = kj;
            w[b + 1] = kw;
        }
        double vi = 0.0;
        for (int a = 0; a < cnt; ++a) vi += w[a];
        int64_t o = lptr[i];
        bool diag_done = false;
        for (int a = 0; a < cnt; ++a) {
            if (!diag_done && nb[a] > i) { lcol[o] = (int32_t)i; lval[o] = vi; ++o; diag_done = true; }
            lcol[o] = nb[a];
            lval[o] = -w[a];
            ++o;
        }
        if (!diag_done) { lcol[o] = (int32_t)i; lval[o] = vi; }
        mass[i] = m;
    }
}

// Rows of M for the free vertices at permuted positions [r0, r1) (one thread per row):
//   M_ij = sum_k (L_ik L_kj) / m_k, k over row i of L, then j over row k, both ascending.
// mode 0: right-hand sides B[r][t] = -M_{i, b_t} (landmark columns, lmpos[j] = t >= 0)
// mode 1: window rows: Win[r - k0][c - k0] = M_ij for free j with c = pos[j] in [k0, k0 + W)
// mode 2: as 1 and the mirror Win[c - k0][r - k0] (rows entering a shifted window)
// dmax (mode 0): max over the rows of M_ii (atomicMax on the bits of a non-negative double)
__global__ void __launch_bounds__(128) k_m_rows(int64_t r0, int64_t r1, const int32_t* __restrict__ uvert,
                                                const int32_t* __restrict__ pos, const int32_t* __restrict__ lmpos,
                                                const int64_t* __restrict__ lptr, const int32_t* __restrict__ lcol,
                                                const double* __restrict__ lval, const double* __restrict__ mass,
                                                int mode, double* __restrict__ out, int64_t ld, int64_t k0, int64_t W,
                                                unsigned long long* __restrict__ dmax, int* __restrict__ bad) {
    for (int64_t r = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < r1; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = uvert[r];
        int32_t cj[kSbhaMaxRing2];
        double cv[kSbhaMaxRing2];
        int cnt = 0;
        for (int64_t e = lptr[i]; e < lptr[i + 1]; ++e) {
            const int32_t k = lcol[e];
            const double lik = lval[e], mk = mass[k];
            for (int64_t f = lptr[k]; f < lptr[k + 1]; ++f) {
                const int32_t j = lcol[f];
                const double v = (lik * lval[f]) / mk;
                int s = 0;
                while (s < cnt && cj[s] != j) ++s;
                if (s == cnt) {
                    if (cnt == kSbhaMaxRing2) { atomicOr(bad, 4); break; }
                    cj[cnt] = j;
                    cv[cnt] = 0.0;
                    ++cnt;
                }
                cv[s] += v;
            }
        }
        for (int s = 0; s < cnt; ++s) {
            const int32_t j = cj[s];
            if (mode == 0) {
                const int32_t t = lmpos[j];
                if (t >= 0) out[r * ld + t] = -cv[s];
                if (j == i && dmax) atomicMax(dmax, (unsigned long long)__double_as_longlong(fmax(cv[s], 0.0)));
            } else {
                if (lmpos[j] >= 0) continue;
                const int64_t c = pos[j];
                if (c < k0 || c >= k0 + W) continue;
                out[(r - k0) * ld + (c - k0)] = cv[s];
                if (mode == 2) out[(c - k0) * ld + (r - k0)] = cv[s];
            }
        }
    }
}

// 64 x 64 triangular solves with R_kk (upper, ldr) for nrhs columns of B (rows k0.. of B, ldb):
// forward R_kk^T Y = B, backward R_kk X = B, in place; one thread per right-hand side.
template <bool FWD>
__global__ void __launch_bounds__(256) k_trsm_panel(const double* __restrict__ R, int64_t ldr, int nb,
                                                    double* __restrict__ B, int64_t ldb, int64_t nrhs) {
    __shared__ double T[64][65];
    for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) T[e / nb][e % nb] = R[(e / nb) * ldr + e % nb];
    __syncthreads();
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= nrhs) return;
    double x[64];
    if (FWD) {
#pragma unroll 1
        for (int i = 0; i < nb; ++i) {
            double acc = B[i * ldb + c];
            for (int p = 0; p < i; ++p) acc = fma(-T[p][i], x[p], acc);
            x[i] = acc / T[i][i];
            B[i * ldb + c] = x[i];
        }
    } else {
#pragma unroll 1
        for (int i = nb - 1; i >= 0; --i) {
            double acc = B[i * ldb + c];
            for (int p = i + 1; p < nb; ++p) acc = fma(-T[i][p], x[p], acc);
            x[i] = acc / T[i][i];
            B[i * ldb + c] = x[i];
        }
    }
}

// XT[c][q] = X[pos[u_q]][c]: free vertex q (increasing vertex order) of column c; 32 x 32 tiles
__global__ void __launch_bounds__(256) k_gather_t(int64_t nu, int64_t l, const int32_t* __restrict__ qrow,
                                                  const double* __restrict__ X, double* __restrict__ XT) {
    __shared__ double t[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t q0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
    for (int k = ty; k < 32; k += 8) {
        const int64_t q = q0 + k, c = c0 + tx;
        t[k][tx] = (q < nu && c < l) ? X[(int64_t)qrow[q] * l + c] : 0.0;
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
        const int64_t c = c0 + k, q = q0 + tx;
        if (c < l && q < nu) XT[c * nu + q] = t[tx][k];
    }
}

// One block per column c of XT (nu values): the p entries of largest |x| (ties: lowest q) as
// (q, x) in increasing q into sel_q / sel_v [c * p ...]. Radix select on the 64-bit pattern of
// |x| (monotone for non-negative doubles), 8 bits per pass from the top.
__global__ void __launch_bounds__(256) k_topp(int64_t nu, int64_t p, const double* __restrict__ XT,
                                              int32_t* __restrict__ sel_q, double* __restrict__ sel_v) {
    __shared__ unsigned int hist[256];
    __shared__ unsigned long long s_prefix;
    __shared__ long long s_need;
    __shared__ int s_scan[256];
    __shared__ long long s_base[2];
    const int64_t c = blockIdx.x;
    const double* x = XT + c * nu;
    auto key = [&](int64_t q) { return (unsigned long long)__double_as_longlong(fabs(x[q])); };
    unsigned long long prefix = 0, mask = 0;
    long long need = p;   // entries still to take among those matching prefix (from the top)
    for (int shift = 56; shift >= 0; shift -= 8) {
        hist[threadIdx.x] = 0;
        __syncthreads();
        for (int64_t q = threadIdx.x; q < nu; q += blockDim.x) {
            const unsigned long long k = key(q);
            if ((k & mask) == prefix) atomicAdd(&hist[(k >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            long long acc = 0;
            int d = 255;
            for (; d > 0; --d) {
                if (acc + hist[d] >= need) break;
                acc += hist[d];
            }
            s_prefix = prefix | ((unsigned long long)d << shift);
            s_need = need - acc;
        }
        __syncthreads();
        prefix = s_prefix;
        need = s_need;
        mask |= 255ull << shift;
        __syncthreads();
    }
    // prefix = the p-th largest key K; take all keys > K and the first `need` keys == K (q order)
    if (threadIdx.x == 0) { s_base[0] = 0; s_base[1] = 0; }
    __syncthreads();
    for (int64_t q0 = 0; q0 < nu; q0 += blockDim.x) {
        const int64_t q = q0 + threadIdx.x;
        unsigned long long k = 0;
        bool gt = false, eq = false;
        if (q < nu) {
            k = key(q);
            gt = k > prefix;
            eq = k == prefix;
        }
        // exclusive scans of eq (tie rank) and of taken (output slot), block-wide in q order
        s_scan[threadIdx.x] = eq ? 1 : 0;
        __syncthreads();
        for (int o = 1; o < 256; o <<= 1) {
            const int v = threadIdx.x >= o ? s_scan[threadIdx.x - o] : 0;
            __syncthreads();
            s_scan[threadIdx.x] += v;
            __syncthreads();
        }
        const long long tie_rank = s_base[1] + s_scan[threadIdx.x] - (eq ? 1 : 0);
        const bool take = gt || (eq && tie_rank < need);
        __syncthreads();
        const int ties_here = s_scan[255];
        __syncthreads();   // (every thread has read the tie total before the array is reused)
        s_scan[threadIdx.x] = take ? 1 : 0;
        __syncthreads();
        for (int o = 1; o < 256; o <<= 1) {
            const int v = threadIdx.x >= o ? s_scan[threadIdx.x - o] : 0;
            __syncthreads();
            s_scan[threadIdx.x] += v;
            __syncthreads();
        }
        if (take) {
            const long long slot = s_base[0] + s_scan[threadIdx.x] - 1;
            sel_q[c * p + slot] = (int32_t)q;
            sel_v[c * p + slot] = x[q];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            s_base[0] += s_scan[255];
            s_base[1] += ties_here;
        }
        __syncthreads();
    }
}

// CSR of S: count per row (landmark rows 1, free rows their kept entries), fill, sort each row
__global__ void k_sbha_count(int64_t l, int64_t p, const int32_t* __restrict__ lm, const int32_t* __restrict__ uvert_q,
                             const int32_t* __restrict__ sel_q, int32_t* __restrict__ cnt) {
    const int64_t total = l + l * p;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int32_t row = e < l ? lm[e] : uvert_q[sel_q[e - l]];
        atomicAdd(&cnt[row], 1);
    }
}

__global__ void k_sbha_fill(int64_t l, int64_t p, const int32_t* __restrict__ lm, const int32_t* __restrict__ uvert_q,
                            const int32_t* __restrict__ sel_q, const double* __restrict__ sel_v,
                            const int64_t* __restrict__ rp, int32_t* __restrict__ cursor, int32_t* __restrict__ col,
                            float* __restrict__ val) {
    const int64_t total = l + l * p;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        int32_t row, c;
        float v;
        if (e < l) { row = lm[e]; c = (int32_t)e; v = 1.0f; }
        else {
            const int64_t s = e - l;
            row = uvert_q[sel_q[s]];
            c = (int32_t)(s / p);
            v = (float)sel_v[s];
        }
        const int32_t o = atomicAdd(&cursor[row], 1);
        col[rp[row] + o] = c;
        val[rp[row] + o] = v;
    }
}

__global__ void k_sort_rows(int64_t n, const int64_t* __restrict__ rp, int32_t* __restrict__ col, float* __restrict__ val) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        for (int64_t a = rp[i] + 1; a < rp[i + 1]; ++a) {
            const int32_t kc = col[a];
            const float kv = val[a];
            int64_t b = a - 1;
            while (b >= rp[i] && col[b] > kc) { col[b + 1] = col[b]; val[b + 1] = val[b]; --b; }
            col[b + 1] = kc;
            val[b + 1] = kv;
        }
}

}  // namespace sbmds
