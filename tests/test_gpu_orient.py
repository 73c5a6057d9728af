"""GPU parity of the task orientations (DESIGN R25) through the C ABI.

LOW holds A_ix[u] per row u and streams A_jx[v]; MID holds A_jx[v] per row v of
part j and streams the ids w > v of A_ix[u] for every u in column v of A_ij (the
suffix after v when x == j); AUTO picks per task.  Every orientation must give
the oracle's T, per-task counts and t(v) bit-exactly, through every kernel path:
light rows (thread per row), heavy rows split into neighbour chunks (a hub whose
column holds > kChunkNbrs u's), the dense-row probe and AND paths (narrow dense
parts), the warp bitmap and hash sets (wide parts), binary search, streaming
residency and logical ranks.
"""
from math import comb

import numpy as np
import pytest

import gen
import oracle
import oracle.blocks as ob

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2209_04541_b200 as pg  # noqa: E402

ORIENTS = ["auto", "low", "mid"]


def hub_graph():
    # two adjacent hubs 0, 1, both adjacent to 6000 leaves 2..6001 paired by an edge
    # (2k+2, 2k+3), plus a separate K_80.  Triangles: (leaf, 0, 1) x 6000, (pair, 0)
    # and (pair, 1) x 3000 each, C(80,3): T = 12000 + C(80,3), t(0) = 9000.  Hub 0
    # ranks below hub 1 (degree tie, id order), so its MID row holds {1} and its
    # column holds 6000 u's: > kChunkNbrs, several heavy items of one row
    s, d = [0], [1]
    for L in range(2, 6002):
        s += [0, 1]
        d += [L, L]
    for k in range(3000):
        s.append(2 + 2 * k)
        d.append(3 + 2 * k)
    base = 6002
    for a in range(80):
        for b in range(a + 1, 80):
            s.append(base + a)
            d.append(base + b)
    return base + 80, np.array(s, np.uint32), np.array(d, np.uint32)


@pytest.mark.parametrize("orient", ORIENTS)
@pytest.mark.parametrize("p", [1, 2, 5, 16])
def test_families(orient, p):
    cases = [gen.rmat(14, 16, seed=61), gen.er(1 << 13, 24, seed=62), gen.grid(120, 0.4, seed=63),
             gen.complete(90), gen.wheel(500), hub_graph(),
             gen.disjoint_union(gen.rmat(16, 8, seed=64), gen.complete(700), gen.clique_union([40] * 30))]
    for g in cases:
        with pg.build_blocks(*g, p=p, orient=orient) as b:
            assert b.triangle_count() == oracle.count(*g), (g[0], p, orient)


def test_hub_chunks_and_closed_form():
    g = hub_graph()
    want = 12000 + comb(80, 3)
    assert oracle.count(*g) == want
    for orient in ORIENTS:
        for p in (1, 3):
            with pg.build_blocks(*g, p=p, orient=orient) as b:
                assert b.triangle_count() == want
                tv, T = b.vertex_triangles()
                assert T == want and int(tv.sum()) == 3 * want and int(tv[0]) == int(tv[1]) == 9000


@pytest.mark.parametrize("orient", ORIENTS)
@pytest.mark.parametrize("scale,p", [(10, 1), (13, 4), (15, 8)])
def test_task_counts_and_vertex(orient, scale, p):
    g = gen.rmat(scale, 16, seed=70 + scale)
    P = ob.Plan(*g, p=p, orient={"auto": 0, "low": 1, "mid": 2}[orient])
    T0, tv0 = oracle.count(*g, per_vertex=True)
    with pg.build_blocks(*g, p=p, orient=orient) as b:
        T, tc = b.triangle_count(task_counts=True)
        assert T == T0
        assert list(map(int, tc)) == P.task_counts()
        tv, T1 = b.vertex_triangles()
        assert T1 == T0 and np.array_equal(tv, tv0)


@pytest.mark.parametrize("orient", ORIENTS)
def test_roles(orient):
    g = gen.rmat(12, 16, seed=81)
    T, lo, mi, hi = oracle.count_roles(*g)
    with pg.build_blocks(*g, p=4, orient=orient) as b:
        t_lo, T1 = b.vertex_triangles(roles="low")
        t_lm, T2 = b.vertex_triangles(roles="low+mid")
        t_all, T3 = b.vertex_triangles()
    assert T1 == T2 == T3 == T
    assert np.array_equal(t_lo, lo)
    assert np.array_equal(t_lm - t_lo, mi)
    assert np.array_equal(t_all, lo + mi + hi)


@pytest.mark.parametrize("orient", ["auto", "mid"])
def test_streaming(orient):
    g = gen.rmat(13, 16, seed=9)
    T0, tv0 = oracle.count(*g, per_vertex=True)
    with pg.build_blocks(*g, p=8, orient=orient) as ref:
        mt = ref.stats()["max_task_bytes"]
    with pg.build_blocks(*g, p=8, orient=orient, residency=pg.RESIDENT_HOST, device_budget_bytes=3 * mt) as b:
        nw = b.stats()["waves"]
        assert nw > 1
        assert b.triangle_count(trace=True) == T0
        tr = b.wave_trace()                                  # copy/compute timeline (S9)
        assert tr.shape == (nw, 4)
        assert (tr[:, 0] <= tr[:, 1]).all() and (tr[:, 2] <= tr[:, 3]).all()
        assert (tr[:, 1] <= tr[:, 2] + 1e-3).all()           # each wave computes after its copy
        assert b.triangle_count() == T0
        tv, _ = b.vertex_triangles()
        assert np.array_equal(tv, tv0)
    with pg.build_blocks(*g, p=8, orient=orient, residency=pg.RESIDENT_HOST) as b:   # no budget
        assert b.triangle_count() == T0


@pytest.mark.parametrize("orient", ["auto", "mid"])
@pytest.mark.parametrize("G", [2, 3])
def test_logical_ranks(orient, G):
    g = gen.rmat(12, 16, seed=10)
    T0 = oracle.count(*g)
    total = 0
    for r in range(G):
        with pg.build_blocks(*g, p=4, rank=r, world_size=G, orient=orient) as b:
            total += b.triangle_count()
    assert total == T0


def test_auto_picks_mid_on_rmat():
    g = gen.rmat(14, 16, seed=61)
    with pg.build_blocks(*g, p=8) as b:
        d, sl, sm = b.task_orient()
        assert (d == 1).sum() > 0
        ijx, _, _ = b.tasks()
        visits = [b.block(int(i), int(j))[1].size for i, j, _ in ijx]
        assert all((dd == 1) == (int(m) + 2 * nv < int(l) and 4 * int(m) < 3 * int(l))
                   for dd, l, m, nv in zip(d, sl, sm, visits))
    with pg.build_blocks(*g, p=8, orient="low") as b:
        d, sl, sm = b.task_orient()
        assert (d == 0).all() and (sm == 0).all()


def test_bad_orient():
    g = gen.rmat(6, 8, seed=1)
    with pytest.raises(pg.PgabbError) as e:
        pg.build_blocks(*g, orient=3)
    assert e.value.name == "EINVAL"
