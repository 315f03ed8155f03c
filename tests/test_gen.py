"""Pins for the input generators (gen/): counts, Dijkstra vs SciPy / brute force, FPS, k-nearest."""
import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import dijkstra as sp_dijkstra

from gen import _native, configs
from gen.mesh import icosphere, mesh_edges, torus_grid


@pytest.mark.parametrize("s", [0, 1, 2, 3, 4])
def test_icosphere_counts(s):
    """n = 10*4^s + 2; Euler characteristic V - E + F = 2."""
    v, f = icosphere(s)
    assert len(v) == 10 * 4 ** s + 2
    assert len(v) - len(mesh_edges(f)) + len(f) == 2
    assert np.allclose(np.linalg.norm(v, axis=1), 1.0)


def torus_graph(nu=10, nv=12, seed=0):
    v, f, e = torus_grid(nu, nv, seed=seed)
    w = np.linalg.norm(v[e[:, 0]] - v[e[:, 1]], axis=1)
    return _native.Graph(len(v), e, w), e, w, len(v)


def test_torus_mesh_structure():
    v, f, e = torus_grid(10, 12)
    assert len(v) == 120 and len(f) == 240 and len(e) == 360
    assert len(mesh_edges(f)) == 360           # every edge belongs to faces, no duplicates


def test_dijkstra_matches_scipy():
    g, e, w, n = torus_graph()
    A = sp.coo_matrix((w, (e[:, 0], e[:, 1])), shape=(n, n)).tocsr()
    ref = sp_dijkstra(A, directed=False, indices=[0, 7, 55])
    got = g.dijkstra_rows([0, 7, 55])
    assert np.allclose(got, ref, rtol=0, atol=1e-12)


def test_dijkstra_floyd_warshall_tiny():
    """agreement with Floyd-Warshall (brute force) on a tiny graph."""
    rng = np.random.default_rng(0)
    n = 9
    edges = np.array([(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < 0.4] +
                     [(i, i + 1) for i in range(n - 1)])
    w = rng.uniform(0.5, 2.0, size=len(edges))
    Dm = np.full((n, n), np.inf)
    np.fill_diagonal(Dm, 0)
    for (a, b), ww in zip(edges, w):
        Dm[a, b] = Dm[b, a] = min(Dm[a, b], ww)
    for k in range(n):
        Dm = np.minimum(Dm, Dm[:, k:k + 1] + Dm[k:k + 1, :])
    g = _native.Graph(n, edges, w)
    assert np.allclose(g.dijkstra_rows(range(n)), Dm, atol=1e-12)


def test_fps_path_example():
    """5 equally spaced points on a path, first=0 -> landmarks 0, 4, 2."""
    e = np.array([(0, 1), (1, 2), (2, 3), (3, 4)])
    g = _native.Graph(5, e, np.ones(4))
    lm, md = g.fps(3, 0)
    assert list(lm) == [0, 4, 2]
    assert np.allclose(md, [0, 1, 0, 1, 0])


def test_fps_brute_force():
    """Eq. 5 by brute force (argmax of min distance, ties lowest index) on a small torus."""
    g, e, w, n = torus_graph(8, 9, seed=3)
    K = g.dijkstra_rows(range(n))
    lm, _ = g.fps(12, 5)
    ref = [5]
    for _ in range(11):
        md = K[ref].min(axis=0)
        ref.append(int(np.flatnonzero(md == md.max())[0]))
    assert list(lm) == ref


def test_knearest_exact_and_truncated():
    g, e, w, n = torus_graph(20, 24, seed=1)
    lm, md = g.fps(30, 0)
    K = g.dijkstra_rows(lm)                  # l x n
    lab, dist = g.knearest(lm, 6)
    lab2, dist2 = g.knearest(lm, 6, radius=0.5 * md.max())   # forces retries
    assert np.array_equal(lab, lab2) and np.allclose(dist, dist2)
    for v in range(n):
        order = np.lexsort((np.arange(30), K[:, v]))[:6]      # by (dist, label)
        assert list(lab[v]) == list(order)
        assert np.allclose(dist[v], K[order, v])


def test_landmark_sqdist_and_graph_variant():
    g, e, w, n = torus_graph(30, 36, seed=2)
    lm, md = g.fps(40, 0)
    D = g.landmark_sqdist(lm)
    K = g.dijkstra_rows(lm, lm)
    iu = np.triu_indices(40, 1)
    assert np.array_equal(D, D.T) and np.all(np.diag(D) == 0)
    assert np.allclose(D[iu], (K ** 2).astype(np.float32)[iu], rtol=1e-6)
    Dg = g.landmark_graph_sqdist(lm, 3 * md.max())
    assert np.array_equal(Dg, Dg.T)
    assert np.all(Dg >= D * (1 - 1e-6))                    # paths through landmarks are longer
    near = K < 3 * md.max()
    assert np.allclose(Dg[near], D[near], rtol=1e-5)       # exact inside the radius


def test_config1_structure():
    """BASELINE.json config 1: rows sum to 1, landmark rows are unit vectors, k=8 otherwise,
    D symmetric with zero diagonal, nnz = (n - l) k + l."""
    p = configs.config(1)
    assert (p.n, p.l, p.nnz) == (2000, 100, 15300)
    lens = np.diff(p.row_ptr)
    is_lm = np.zeros(p.n, bool)
    is_lm[p.landmarks] = True
    assert np.all(lens[is_lm] == 1) and np.all(lens[~is_lm] == 8)
    rs = np.add.reduceat(p.val, p.row_ptr[:-1])
    assert np.allclose(rs, 1.0, atol=1e-14)
    assert np.all(p.col_idx[p.row_ptr[:-1][p.landmarks]] == np.arange(p.l))
    assert np.array_equal(p.D, p.D.T) and np.all(np.diag(p.D) == 0)


def test_random_rows_structure():
    col, val = _native.random_rows(1000, 600, 16, 256, seed=3)
    col = col.reshape(1000, 16)
    val = val.reshape(1000, 16)
    assert np.all(np.diff(col, axis=1) > 0)                   # distinct, sorted
    assert np.all(col.max(1) - col.min(1) < 256)              # window
    assert np.allclose(val.sum(1), 1.0, atol=1e-6) and np.all(val > 0)
    D = _native.random_sym(300, 4)
    assert np.array_equal(D, D.T) and D.min() >= 0 and D.max() <= 100


def test_bumpy_sphere_morton_order_is_a_renumbering():
    """Config 3's vertex order (Morton) renumbers the same mesh: the same triangles in space, and
    blocks of 128 consecutive vertices are compact (median bounding-box diagonal far below the
    subdivision order's)."""
    import numpy as np
    from gen.mesh import bumpy_sphere
    v, f = bumpy_sphere(6)
    v0, f0 = bumpy_sphere(6, order="subdivision")
    key = lambda V, F: np.sort(np.sort(np.round(V[F], 12).reshape(-1, 9), axis=1), axis=0)   # noqa: E731
    assert np.array_equal(key(v, f), key(v0, f0))
    def spread(V, rb=128):      # median bounding-box diagonal of consecutive 128-vertex blocks
        return np.median([np.linalg.norm(V[i:i + rb].max(0) - V[i:i + rb].min(0)) for i in range(0, len(V), rb)])
    assert spread(v) < 0.3 * spread(v0)
