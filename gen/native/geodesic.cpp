// Input-generator helper (NOT the method): exact edge-graph geodesics on meshes.
//
// This file builds the synthetic inputs that stand in for the paper's meshes
// (BASELINE.json configs 1-5; SURVEY.md §8(c) reading 10). It holds
// none of the sBMDS arithmetic. Both the CUDA path and the oracle consume its
// outputs; neither links it.
//
//   gen_dijkstra_rows    full single-source shortest paths,
//                        many sources in parallel (OpenMP).
//   gen_fps              farthest-point landmark selection
//                        (Eq. 5), ties to the lowest vertex index.
//                        Exact: an incremental Dijkstra from each new landmark
//                        that only descends where it lowers min_dist.
//   gen_knearest         k nearest landmarks of each vertex by graph distance
//                        (BASELINE.json config 1), ties to the lowest landmark
//                        index; exact via radius-truncated searches + a check.
//   gen_landmark_sqdist  D_ll = squared exact landmark-to-landmark distances.
//   gen_landmark_graph_sqdist
//                        config-4 stand-in: squared shortest paths
//                        on the landmark graph whose edges join landmarks within
//                        a radius, weighted by exact mesh-graph distance.
//   gen_random_rows / gen_random_sym   config-5 random structure.
//
// Shortest paths use a bucket queue of width delta <= min edge weight: every
// vertex in the lowest non-empty bucket is final (a relaxation adds >= delta, so
// it cannot land in the same bucket), which gives exactly the same fixed point
// as binary-heap Dijkstra at O(1) per operation.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <queue>
#include <vector>
#include <omp.h>

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

struct CsrGraph {
    int64_t n;
    const int64_t* ptr;
    const int32_t* idx;
    const double* w;
};

struct EdgeStats {
    double wmin, wmax;
};

EdgeStats edge_stats(const CsrGraph& g) {
    double lo = kInf, hi = 0.0;
    const int64_t m = g.ptr[g.n];
    for (int64_t e = 0; e < m; ++e) {
        lo = std::min(lo, g.w[e]);
        hi = std::max(hi, g.w[e]);
    }
    return {lo, hi};
}

// Bucket-queue SSSP. dist must be all +inf on entry (restored for touched vertices
// by reset()); settled vertices are appended to `order` in settle order.
class BucketSssp {
   public:
    BucketSssp(const CsrGraph& g, EdgeStats es) : g_(g) {
        delta_ = es.wmin * (1.0 - 1e-9);
        if (!(delta_ > 0.0)) delta_ = 1e-300;
        nb_ = (int64_t)std::ceil(es.wmax / delta_) + 2;
        if (nb_ > (1 << 24)) nb_ = 1 << 24;  // guard; falls back to correct but slower scans
        buckets_.resize(nb_);
        dist.assign(g.n, kInf);
        settled_.assign(g.n, 0);
    }
    std::vector<double> dist;
    std::vector<int32_t> order;

    void reset() {
        for (int32_t v : touched_) {
            dist[v] = kInf;
            settled_[v] = 0;
        }
        touched_.clear();
        order.clear();
    }

    // Settle every vertex with dist <= radius (all of them when radius = inf).
    void run(int32_t src, double radius = kInf) {
        reset();
        dist[src] = 0.0;
        touched_.push_back(src);
        int64_t pending = 1;
        buckets_[0].push_back(src);
        int64_t k = 0;
        while (pending > 0) {
            std::vector<int32_t>& B = buckets_[k % nb_];
            if (B.empty()) {
                ++k;
                continue;
            }
            // process bucket k; it cannot grow while being processed
            for (size_t q = 0; q < B.size(); ++q) {
                const int32_t v = B[q];
                --pending;
                if (settled_[v]) continue;
                const double dv = dist[v];
                if ((int64_t)(dv / delta_) != k) continue;  // stale copy (moved to a lower bucket)
                if (dv > radius) continue;
                settled_[v] = 1;
                order.push_back(v);
                for (int64_t e = g_.ptr[v]; e < g_.ptr[v + 1]; ++e) {
                    const int32_t u = g_.idx[e];
                    if (settled_[u]) continue;
                    const double nd = dv + g_.w[e];
                    if (nd < dist[u]) {
                        if (dist[u] == kInf) touched_.push_back(u);
                        dist[u] = nd;
                        if (nd <= radius) {
                            buckets_[((int64_t)(nd / delta_)) % nb_].push_back(u);
                            ++pending;
                        }
                    }
                }
            }
            B.clear();
            ++k;
        }
    }

   private:
    const CsrGraph& g_;
    double delta_;
    int64_t nb_;
    std::vector<std::vector<int32_t>> buckets_;
    std::vector<uint8_t> settled_;
    std::vector<int32_t> touched_;
};

struct HeapItem {
    double d;
    int32_t v;
    bool operator>(const HeapItem& o) const { return d > o.d || (d == o.d && v > o.v); }
};
using MinHeap = std::priority_queue<HeapItem, std::vector<HeapItem>, std::greater<HeapItem>>;

inline uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

void mirror_upper(int64_t l, float* D) {
    const int64_t B = 64;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t ib = 0; ib < l; ib += B)
        for (int64_t jb = 0; jb <= ib; jb += B)
            for (int64_t i = ib; i < std::min(ib + B, l); ++i)
                for (int64_t j = jb; j < std::min(jb + B, i); ++j) D[i * l + j] = D[j * l + i];
}

}  // namespace

extern "C" {

int gen_num_threads() { return omp_get_max_threads(); }

// out[s * nt + t] = dist(sources[s], targets[t]).
int gen_dijkstra_rows(int64_t n, const int64_t* ptr, const int32_t* idx, const double* w,
                      int64_t ns, const int32_t* sources, int64_t nt, const int32_t* targets,
                      double* out) {
    const CsrGraph g{n, ptr, idx, w};
    const EdgeStats es = edge_stats(g);
#pragma omp parallel
    {
        BucketSssp sp(g, es);
#pragma omp for schedule(dynamic, 1)
        for (int64_t s = 0; s < ns; ++s) {
            sp.run(sources[s]);
            double* row = out + s * nt;
            for (int64_t t = 0; t < nt; ++t) row[t] = sp.dist[targets[t]];
        }
    }
    return 0;
}

// Farthest-point sampling (Eq. 5). landmarks[0] = first; min_dist (n) returned.
// Returns 0, or -1 if the graph is disconnected (an unreachable vertex is picked).
int gen_fps(int64_t n, const int64_t* ptr, const int32_t* idx, const double* w, int64_t l,
            int32_t first, int32_t* landmarks, double* min_dist) {
    for (int64_t i = 0; i < n; ++i) min_dist[i] = kInf;
    // segment tree over (min_dist, -index): argmax with ties to the lowest index
    int64_t size = 1;
    while (size < n) size <<= 1;
    std::vector<int32_t> tree(2 * size, -1);
    auto better = [&](int32_t a, int32_t b) -> int32_t {
        if (a < 0) return b;
        if (b < 0) return a;
        if (min_dist[a] > min_dist[b]) return a;
        if (min_dist[b] > min_dist[a]) return b;
        return a < b ? a : b;
    };
    for (int64_t i = 0; i < n; ++i) tree[size + i] = (int32_t)i;
    for (int64_t i = size - 1; i >= 1; --i) tree[i] = better(tree[2 * i], tree[2 * i + 1]);
    auto update = [&](int32_t v) {
        int64_t p = (size + v) >> 1;
        while (p >= 1) {
            tree[p] = better(tree[2 * p], tree[2 * p + 1]);
            p >>= 1;
        }
    };
    std::vector<int32_t> touched;
    MinHeap heap;
    int32_t cur = first;
    for (int64_t j = 0; j < l; ++j) {
        if (j > 0) {
            cur = tree[1];
            if (!(min_dist[cur] < kInf)) return -1;
        }
        landmarks[j] = cur;
        touched.clear();
        min_dist[cur] = 0.0;
        touched.push_back(cur);
        heap.push({0.0, cur});
        while (!heap.empty()) {
            HeapItem it = heap.top();
            heap.pop();
            if (it.d > min_dist[it.v]) continue;
            for (int64_t e = ptr[it.v]; e < ptr[it.v + 1]; ++e) {
                const int32_t u = idx[e];
                const double nd = it.d + w[e];
                if (nd < min_dist[u]) {
                    min_dist[u] = nd;
                    touched.push_back(u);
                    heap.push({nd, u});
                }
            }
        }
        for (int32_t v : touched) update(v);
    }
    return 0;
}

// k nearest landmarks of each vertex, sorted by (d, label); exact whenever the
// return value is 0. Candidates come from searches truncated at `radius`; a vertex
// whose k-th candidate is farther than radius (or that has < k candidates) may be
// missing a nearer landmark, so those vertices are counted and the caller retries
// with a larger radius (radius = inf gives the plain exact answer).
int64_t gen_knearest(int64_t n, const int64_t* ptr, const int32_t* idx, const double* w,
                     int64_t l, const int32_t* landmarks, int32_t k, double radius,
                     int32_t* out_lab, double* out_dist) {
    const CsrGraph g{n, ptr, idx, w};
    const EdgeStats es = edge_stats(g);
    struct Cand {
        int32_t v, lab;
        double d;
    };
    const int nt = omp_get_max_threads();
    std::vector<std::vector<Cand>> per(nt);
#pragma omp parallel
    {
        BucketSssp sp(g, es);
        auto& mine = per[omp_get_thread_num()];
#pragma omp for schedule(dynamic, 4)
        for (int64_t j = 0; j < l; ++j) {
            sp.run(landmarks[j], radius);
            for (int32_t v : sp.order) mine.push_back({v, (int32_t)j, sp.dist[v]});
        }
    }
    std::vector<int64_t> cnt(n + 1, 0);
    for (auto& P : per)
        for (auto& c : P) cnt[c.v + 1]++;
    for (int64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
    std::vector<Cand> all(cnt[n]);
    {
        std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
        for (auto& P : per) {
            for (auto& c : P) all[pos[c.v]++] = c;
            std::vector<Cand>().swap(P);
        }
    }
    int64_t bad = 0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(+ : bad)
    for (int64_t v = 0; v < n; ++v) {
        Cand* b = all.data() + cnt[v];
        Cand* e = all.data() + cnt[v + 1];
        const int64_t c = e - b;
        const int64_t kk = std::min<int64_t>(k, c);
        std::partial_sort(b, b + kk, e, [](const Cand& x, const Cand& y) {
            return x.d < y.d || (x.d == y.d && x.lab < y.lab);
        });
        for (int64_t q = 0; q < k; ++q) {
            out_lab[v * k + q] = q < kk ? b[q].lab : -1;
            out_dist[v * k + q] = q < kk ? b[q].d : kInf;
        }
        if (c < k || (radius < kInf && b[k - 1].d >= radius)) bad++;
    }
    return bad;
}

// D_ll (BASELINE.json config 1: "D_ll holds the squared Dijkstra distances between
// landmarks"): D[i*l + j] = float(d(b_i, b_j)^2). Entry (i, j) with i < j comes
// from the SSSP of source b_i and is mirrored to (j, i), so D is exactly symmetric
// with a zero diagonal. Returns -1 if some landmark pair is unreachable.
int gen_landmark_sqdist(int64_t n, const int64_t* ptr, const int32_t* idx, const double* w,
                        int64_t l, const int32_t* landmarks, float* D) {
    const CsrGraph g{n, ptr, idx, w};
    const EdgeStats es = edge_stats(g);
    int bad = 0;
#pragma omp parallel reduction(| : bad)
    {
        BucketSssp sp(g, es);
#pragma omp for schedule(dynamic, 1)
        for (int64_t s = 0; s < l; ++s) {
            sp.run(landmarks[s]);
            float* row = D + s * l;
            for (int64_t t = s; t < l; ++t) {
                const double d = sp.dist[landmarks[t]];
                if (!(d < kInf)) bad = 1;
                row[t] = (t == s) ? 0.0f : (float)(d * d);
            }
        }
    }
    mirror_upper(l, D);
    return bad ? -1 : 0;
}

// Config-4 stand-in for D_ll: exact mesh-graph distances between
// landmarks closer than `radius` become edges of a landmark graph; D holds the
// squared shortest paths of that graph (>= the mesh-graph geodesic, equal for
// pairs within radius). Returns -1 if the landmark graph is disconnected.
int gen_landmark_graph_sqdist(int64_t n, const int64_t* ptr, const int32_t* idx,
                              const double* w, int64_t l, const int32_t* landmarks, double radius,
                              float* D) {
    const CsrGraph g{n, ptr, idx, w};
    const EdgeStats es = edge_stats(g);
    std::vector<int32_t> lm_of(n, -1);
    for (int64_t j = 0; j < l; ++j) lm_of[landmarks[j]] = (int32_t)j;
    std::vector<std::vector<std::pair<int32_t, double>>> adj(l);
#pragma omp parallel
    {
        BucketSssp sp(g, es);
#pragma omp for schedule(dynamic, 4)
        for (int64_t j = 0; j < l; ++j) {
            sp.run(landmarks[j], radius);
            for (int32_t v : sp.order)
                if (lm_of[v] >= 0 && lm_of[v] != j) adj[j].push_back({lm_of[v], sp.dist[v]});
            std::sort(adj[j].begin(), adj[j].end());
        }
    }
    // symmetric landmark graph: keep (a,b) with weight min(d_ab, d_ba)
    std::vector<int64_t> lp(l + 1, 0);
    for (int64_t a = 0; a < l; ++a) lp[a + 1] = lp[a] + (int64_t)adj[a].size();
    std::vector<int32_t> li(lp[l]);
    std::vector<double> lw(lp[l]);
    for (int64_t a = 0; a < l; ++a) {
        for (size_t q = 0; q < adj[a].size(); ++q) {
            const int32_t b = adj[a][q].first;
            double d = adj[a][q].second;
            auto it = std::lower_bound(adj[b].begin(), adj[b].end(),
                                       std::make_pair((int32_t)a, -kInf));
            if (it != adj[b].end() && it->first == a) d = std::min(d, it->second);
            li[lp[a] + q] = b;
            lw[lp[a] + q] = d;
        }
    }
    std::vector<std::vector<std::pair<int32_t, double>>>().swap(adj);
    const CsrGraph lg{l, lp.data(), li.data(), lw.data()};
    const EdgeStats les = edge_stats(lg);
    int bad = 0;
#pragma omp parallel reduction(| : bad)
    {
        BucketSssp sp(lg, les);
#pragma omp for schedule(dynamic, 1)
        for (int64_t s = 0; s < l; ++s) {
            sp.run((int32_t)s);
            float* row = D + s * l;
            for (int64_t t = s; t < l; ++t) {
                const double d = sp.dist[t];
                if (!(d < kInf)) bad = 1;
                row[t] = (t == s) ? 0.0f : (float)(d * d);
            }
        }
    }
    mirror_upper(l, D);
    return bad ? -1 : 0;
}

// Config-5 D (SURVEY.md §8(c) reading 10): D = (U + U^T)/2 with U_ij ~ U[0,100]
// fp32 drawn from a counter-based hash of (seed, i, j); diagonal left as U_ii.
int gen_random_sym(int64_t l, uint64_t seed, float* D) {
    auto u01 = [&](int64_t i, int64_t j) {
        const uint64_t h =
            splitmix64(splitmix64(seed ^ 0xD1B54A32D192ED03ull) + (uint64_t)(i * l + j));
        return (float)((double)(h >> 40) * (1.0 / 16777216.0));
    };
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < l; ++i) {
        for (int64_t j = i; j < l; ++j) {
            const float a = 100.0f * u01(i, j), b = 100.0f * u01(j, i);
            const float v = (i == j) ? a : 0.5f * (a + b);
            D[i * l + j] = v;
            D[j * l + i] = v;
        }
    }
    return 0;
}

// Config 5 (BASELINE.json configs[4]; SURVEY.md §8(c) reading 10): row i has a
// centre c_i ~ U{0..l-window} and k distinct offsets from [0, window), sorted,
// with weights U(0,1] normalised to sum 1. row_ptr is i*k. Deterministic in seed.
int gen_random_rows(int64_t n, int64_t l, int32_t k, int32_t window, uint64_t seed,
                    int32_t* col_idx, float* val) {
    if (window > l || k > window) return -1;
#pragma omp parallel
    {
        std::vector<int32_t> pool(window);
        std::vector<double> wv(k);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            uint64_t st = splitmix64(seed * 0x100000001B3ull + (uint64_t)i);
            auto next = [&]() {
                st = splitmix64(st);
                return st;
            };
            const int64_t c = (int64_t)(next() % (uint64_t)(l - window + 1));
            for (int32_t q = 0; q < window; ++q) pool[q] = q;
            for (int32_t q = 0; q < k; ++q) {  // partial Fisher-Yates
                const int32_t r = q + (int32_t)(next() % (uint64_t)(window - q));
                std::swap(pool[q], pool[r]);
            }
            std::sort(pool.begin(), pool.begin() + k);
            double s = 0.0;
            for (int32_t q = 0; q < k; ++q) {
                // U(0,1]: 53 random bits, shifted off zero
                wv[q] = ((double)(next() >> 11) + 1.0) * (1.0 / 9007199254740992.0);
                s += wv[q];
            }
            for (int32_t q = 0; q < k; ++q) {
                col_idx[i * k + q] = (int32_t)(c + pool[q]);
                val[i * k + q] = (float)(wv[q] / s);
            }
        }
    }
    return 0;
}

}  // extern "C"
