"""Pins of the oracle's triangle count (oracle/tc_oracle.c) to things other than itself.

* brute force: the O(n^3) definition (SPEC acceptance 1: 50 ER + 20 R-MAT, n <= 200);
* closed forms (verified with networkx there);
* library routines: scipy trace(A^3)/6, networkx.triangles;
* invariants: sum t(v) = 3T, vertex relabelling, tuple noise, disjoint-union additivity.
"""
from math import comb

import networkx as nx
import numpy as np
import pytest
import scipy.sparse as sp

import gen
import oracle


def T(g):
    return oracle.count(*g)


def brute(g):
    return oracle.brute(*g)


# ---- brute force is itself pinned by closed forms --------------------------------
@pytest.mark.parametrize("n", [3, 4, 5, 9, 30])
def test_brute_complete(n):
    assert brute(gen.complete(n)) == comb(n, 3)


def test_brute_zero_families():
    assert brute(gen.cycle(10)) == 0
    assert brute(gen.cycle(3)) == 1
    assert brute(gen.random_tree(50, 2)) == 0
    assert brute(gen.complete_bipartite(5, 7)) == 0


# ---- node iterator vs brute force (SPEC acceptance 1 shape) -----------------------
def test_node_iterator_vs_brute_random():
    rng = np.random.default_rng(0)
    for k in range(50):
        n = int(rng.integers(5, 200))
        g = gen.er_small(n, float(rng.uniform(0.02, 0.4)), seed=k)
        assert T(g) == brute(g), k
    for k in range(20):
        scale = int(rng.integers(3, 8))
        g = gen.rmat(scale, 8, seed=100 + k)
        assert T(g) == brute(g), k


def test_node_iterator_vs_brute_messy():
    g = gen.messy(gen.er_small(150, 0.2, seed=9), seed=4)
    assert T(g) == brute(g)


# ---- closed forms ----------------------------------------------------------------
@pytest.mark.parametrize("n", [1, 2, 3, 4, 10, 57, 300])
def test_complete(n):
    assert T(gen.complete(n)) == comb(n, 3)


@pytest.mark.parametrize("n", [4, 5, 17, 1000])
def test_cycle_path_star_tree_zero(n):
    assert T(gen.cycle(n)) == 0
    assert T(gen.path(n)) == 0
    assert T(gen.star(n)) == 0
    assert T(gen.random_tree(n, 5)) == 0


def test_c3():
    assert T(gen.cycle(3)) == 1


@pytest.mark.parametrize("n", [5, 6, 11, 500])
def test_wheel(n):
    assert T(gen.wheel(n)) == n - 1


def test_wheel4_is_k4():
    # SURVEY §8(c) reading 11: W_4 = K_4 -> 4
    assert T(gen.wheel(4)) == 4


@pytest.mark.parametrize("k,m", [(1, 4), (3, 5), (10, 6)])
def test_windmill(k, m):
    assert T(gen.windmill(k, m)) == k * comb(m, 3)


def test_clique_union():
    sizes = [3, 7, 50, 120, 1, 2]
    assert T(gen.clique_union(sizes)) == sum(comb(s, 3) for s in sizes)


@pytest.mark.parametrize("a,b", [(2, 2), (3, 4), (6, 9)])
def test_rook(a, b):
    assert T(gen.rook(a, b)) == b * comb(a, 3) + a * comb(b, 3)


@pytest.mark.parametrize("r,c", [(2, 2), (3, 5), (20, 31)])
def test_king(r, c):
    assert T(gen.king(r, c)) == 4 * (r - 1) * (c - 1)


def test_complete_bipartite_zero():
    assert T(gen.complete_bipartite(20, 30)) == 0


@pytest.mark.parametrize("side,f", [(2, 1.0), (64, 0.0), (128, 0.1), (300, 0.5)])
def test_grid_diagonals(side, f):
    # one diagonal per cell adds exactly 2 triangles; none span cells
    g = gen.grid(side, f, seed=11)
    assert T(g) == 2 * gen.grid_ndiag(side, f, seed=11)


# ---- library routines ------------------------------------------------------------
def _scipy_T(n, s, d):
    A = sp.coo_matrix((np.ones(s.size), (s, d)), shape=(n, n)).tocsr()
    A = ((A + A.T) > 0).astype(np.int64)
    A.setdiag(0)
    A.eliminate_zeros()
    return int((A @ A).multiply(A).sum()) // 6


@pytest.mark.parametrize("scale", [10, 12, 14])
def test_rmat_vs_scipy(scale):
    g = gen.rmat(scale, 16, seed=1)
    assert T(g) == _scipy_T(*g)


def test_er_vs_scipy():
    g = gen.er(1 << 14, 32, seed=2)
    assert T(g) == _scipy_T(*g)


def test_per_vertex_vs_networkx():
    n, s, d = gen.rmat(9, 8, seed=4)
    G = nx.Graph()
    G.add_nodes_from(range(n))
    G.add_edges_from((int(a), int(b)) for a, b in zip(s, d) if a != b)
    Tn, tv = oracle.count(n, s, d, per_vertex=True)
    ref = nx.triangles(G)
    assert [int(x) for x in tv] == [ref[v] for v in range(n)]
    assert Tn == sum(ref.values()) // 3


# ---- invariants ------------------------------------------------------------------
def test_sum_tv_is_3T():
    for g in (gen.rmat(12, 16, 3), gen.er(5000, 20, 3), gen.king(10, 10)):
        t, tv = oracle.count(*g, per_vertex=True)
        assert int(tv.sum()) == 3 * t


def test_relabel_and_noise_invariance():
    g = gen.rmat(11, 16, seed=6)
    t0 = T(g)
    assert T(gen.relabel(g, seed=2)) == t0
    assert T(gen.messy(g, seed=3)) == t0


def test_disjoint_union_additive():
    g, h = gen.rmat(10, 16, 1), gen.er(3000, 16, 2)
    assert T(gen.disjoint_union(g, h)) == T(g) + T(h)


def test_m_edges_vs_set():
    n, s, d = gen.messy(gen.rmat(9, 8, 2), seed=1)
    ref = {(min(int(a), int(b)), max(int(a), int(b))) for a, b in zip(s, d) if a != b}
    with oracle.Graph(n, s, d) as g:
        assert g.m_edges == len(ref)
        deg = np.zeros(n, np.int64)
        for a, b in ref:
            deg[a] += 1
            deg[b] += 1
        assert (g.degrees() == deg).all()


def test_wedges_are_dag_two_paths():
    # W = number of directed 2-paths u->v->w in the degree-ordered DAG = sum(A+ @ A+)
    n, s, d = gen.rmat(10, 16, 5)
    with oracle.Graph(n, s, d) as g:
        deg = g.degrees().astype(np.int64)
        W = g.wedges()
    E = {(min(int(a), int(b)), max(int(a), int(b))) for a, b in zip(s, d) if a != b}
    key = lambda v: (deg[v], v)
    rows, cols = zip(*[(a, b) if key(a) < key(b) else (b, a) for a, b in E])
    Ap = sp.coo_matrix((np.ones(len(rows), np.int64), (rows, cols)), shape=(n, n)).tocsr()
    assert W == int((Ap @ Ap).sum())


def test_count_range_partitions_T():
    g = gen.rmat(11, 16, seed=8)
    with oracle.Graph(*g) as o:
        full = o.count()
        parts = [o.count_range(r, g[0], 4) for r in range(4)]
        assert sum(t for t, _ in parts) == full
        assert sum(e for _, e in parts) == o.m_edges


def test_bad_ids_rejected():
    with pytest.raises(ValueError):
        oracle.Graph(3, np.array([0, 5], np.uint32), np.array([1, 1], np.uint32))


def test_empty_graph():
    assert oracle.count(0, np.zeros(0, np.uint32), np.zeros(0, np.uint32)) == 0
    assert oracle.count(5, np.zeros(0, np.uint32), np.zeros(0, np.uint32)) == 0


# ---- local clustering coefficient (NEXT-1) -------------------
def test_clustering_vs_networkx():
    for n, s, d in (gen.rmat(9, 8, seed=5), gen.er_small(200, 0.08, seed=6), gen.king(7, 9)):
        G = nx.Graph()
        G.add_nodes_from(range(n))
        G.add_edges_from((int(a), int(b)) for a, b in zip(s, d) if a != b)
        _, cc = oracle.clustering(n, s, d)
        ref = nx.clustering(G)
        # both are one correctly rounded division of the same integers
        assert [float(x) for x in cc] == [float(ref[v]) for v in range(n)]


def test_clustering_closed_forms():
    _, cc = oracle.clustering(*gen.complete(12))
    assert (cc == 1.0).all()                          # every neighbourhood of K_n is a clique
    n = 40
    tv, cc = oracle.clustering(*gen.wheel(n))         # hub 0 + (n-1)-cycle
    assert tv[0] == n - 1 and (tv[1:] == 2).all()
    assert cc[0] == 2.0 * (n - 1) / ((n - 1) * (n - 2)) and (cc[1:] == 2.0 * 2 / (3 * 2)).all()
    for g in (gen.random_tree(300, 2), gen.cycle(50), gen.complete_bipartite(5, 8)):
        _, cc = oracle.clustering(*g)
        assert (cc == 0.0).all()
    e = np.zeros(0, np.uint32)
    tv, cc = oracle.clustering(5, e, e)               # isolated vertices: deg < 2 -> 0
    assert (tv == 0).all() and (cc == 0.0).all()


# ---- connected components (NEXT-4) --------------------------
def _bfs_components(n, s, d):
    adj = [[] for _ in range(n)]
    for a, b in zip(s, d):
        if a != b:
            adj[int(a)].append(int(b))
            adj[int(b)].append(int(a))
    lab = [-1] * n
    for v in range(n):           # ascending v: the first vertex reached is the smallest id
        if lab[v] >= 0:
            continue
        lab[v] = v
        stack = [v]
        while stack:
            x = stack.pop()
            for y in adj[x]:
                if lab[y] < 0:
                    lab[y] = v
                    stack.append(y)
    return lab


def test_components_vs_bfs_and_scipy():
    from scipy.sparse.csgraph import connected_components
    for n, s, d in (gen.er_small(300, 0.004, seed=1), gen.rmat(9, 2, seed=2),
                    gen.disjoint_union(gen.path(30), gen.complete(5), gen.star(9), gen.cycle(7))):
        lab, nc = oracle.components(n, s, d)
        assert [int(x) for x in lab] == _bfs_components(n, s, d)
        A = sp.coo_matrix((np.ones(s.size), (s, d)), shape=(n, n))
        k, sl = connected_components(A, directed=False)
        assert nc == k
        # same partition: labels and scipy's component ids are in bijection
        assert len(set(zip(lab.tolist(), sl.tolist()))) == k


def test_components_closed_forms():
    lab, nc = oracle.components(*gen.path(100))
    assert nc == 1 and (lab == 0).all()
    g = gen.clique_union([3, 9, 1, 64])          # 4 cliques, one a single vertex
    lab, nc = oracle.components(*g)
    assert nc == 4 and sorted(set(lab.tolist())) == [0, 3, 12, 13]
    e = np.zeros(0, np.uint32)
    lab, nc = oracle.components(6, e, e)          # isolated ids label themselves
    assert nc == 6 and lab.tolist() == list(range(6))
    lab, nc = oracle.components(*gen.messy(gen.cycle(50), seed=3))   # noise does not change G_s
    assert nc == 1


# ---- per-vertex counts by role (DESIGN R24) --------------------------------------
def test_roles_sum_and_closed_form():
    for g in (gen.rmat(10, 16, seed=8), gen.king(8, 9), gen.er_small(150, 0.1, seed=9)):
        T, lo, mi, hi = oracle.count_roles(*g)
        T2, tv = oracle.count(*g, per_vertex=True)
        assert T == T2
        assert np.array_equal(lo + mi + hi, tv)
        assert int(lo.sum()) == int(mi.sum()) == int(hi.sum()) == T   # one vertex of each role
    # K_n: all degrees equal, so the order is by id; vertex r is lowest in C(n-1-r, 2)
    # triangles, middle in r(n-1-r), highest in C(r, 2)
    n = 13
    T, lo, mi, hi = oracle.count_roles(*gen.complete(n))
    r = np.arange(n)
    assert (lo == (n - 1 - r) * (n - 2 - r) // 2).all()
    assert (mi == r * (n - 1 - r)).all()
    assert (hi == r * (r - 1) // 2).all()
