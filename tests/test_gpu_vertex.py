"""GPU parity of the per-vertex path: t(v) for every
vertex and the local clustering coefficient (§1), through the
C ABI (pgabb_vertex_triangles, pgabb_local_clustering), against the oracle.

t(v) is integer: bit-exact.  cc(v) is one correctly rounded fp64 division of
the same two integers on both sides, so it is compared bit-exactly as well.
The cases steer every intersection path of k_tc_rows: dense bitmap rows
(probe_dense_row and the AND path), the warp bitmap set (narrow parts), the
hash set (parts wider than 32768) and lane-parallel binary search
(|A_ix[u]| > 512 in a wide part), plus streaming residency and logical ranks.
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
from paper_2209_04541_b200 import dist as pgd  # noqa: E402


def check(g, **kw):
    want_T, want_tv = oracle.count(*g, per_vertex=True)
    with pg.build_blocks(*g, **kw) as b:
        tv, T = b.vertex_triangles()
        assert T == want_T
        assert tv.dtype == np.uint64 and tv.shape == (g[0],)
        assert np.array_equal(tv, want_tv)
        assert int(tv.sum()) == 3 * T
        # the per-vertex kernel leaves the counting path unchanged
        assert b.triangle_count() == want_T
    return tv


@pytest.mark.parametrize("p", [1, 2, 3, 8])
def test_closed_forms_per_vertex(p):
    tv = check(gen.complete(40), p=p)
    assert (tv == comb(39, 2)).all()
    tv = check(gen.wheel(300), p=p)
    assert tv[0] == 299 and (tv[1:] == 2).all()
    tv = check(gen.windmill(7, 6), p=p)
    assert tv[0] == 7 * comb(5, 2)
    check(gen.king(17, 23), p=p)
    check(gen.clique_union([3, 9, 200, 2, 1, 64]), p=p)
    tv = check(gen.random_tree(500, 3), p=p)
    assert (tv == 0).all()


@pytest.mark.parametrize("scale,p", [(8, 1), (10, 2), (12, 5), (14, 8), (16, 16)])
def test_rmat_per_vertex(scale, p):
    check(gen.rmat(scale, 16, seed=scale + 1), p=p)


def test_er_grid_per_vertex():
    check(gen.er(1 << 14, 32, seed=3), p=4)
    check(gen.grid(300, 0.3, seed=4), p=6)


@pytest.mark.parametrize("light_held", [8, 15])
def test_per_vertex_light_held(light_held):
    # medium thread-per-row items (R29) credit u, v and w like the light ones
    check(gen.er(1 << 14, 32, seed=5), p=2, light_held=light_held)
    check(gen.rmat(13, 16, seed=6), p=4, light_held=light_held)


def test_wide_parts_hash_and_search_paths():
    # p=1 over n > 32768 ids: the column part is wider than the warp bitmap, so
    # rows use the hash set (|A_ix[u]| <= 512) or binary search (> 512: K_700)
    big = gen.rmat(16, 8, seed=7)
    g = gen.disjoint_union(big, gen.complete(700), gen.clique_union([40] * 30))
    check(g, p=1)
    check(g, p=2)


def test_degenerate_per_vertex():
    e = np.zeros(0, np.uint32)
    with pg.build_blocks(7, e, e, p=3) as b:
        tv, T = b.vertex_triangles()
        assert T == 0 and tv.shape == (7,) and (tv == 0).all()
        assert (b.local_clustering(tv) == 0.0).all()
    check((3, np.array([0, 1, 2], np.uint32), np.array([1, 2, 0], np.uint32)), p=2)


def test_streaming_per_vertex():
    g = gen.rmat(13, 16, seed=9)
    _, want = oracle.count(*g, per_vertex=True)
    with pg.build_blocks(*g, p=8) as ref:
        mt = ref.stats()["max_task_bytes"]
    with pg.build_blocks(*g, p=8, residency=pg.RESIDENT_HOST, device_budget_bytes=3 * mt) as b:
        assert b.stats()["waves"] > 1
        tv, _ = b.vertex_triangles()
        assert np.array_equal(tv, want)


@pytest.mark.parametrize("G", [2, 3])
def test_logical_ranks_sum(G):
    g = gen.rmat(12, 16, seed=10)
    _, want = oracle.count(*g, per_vertex=True)
    total = np.zeros(g[0], np.uint64)
    for r in range(G):
        with pg.build_blocks(*g, p=4, rank=r, world_size=G) as b:
            tv, _ = b.vertex_triangles()
            total += tv
    assert np.array_equal(total, want)


def test_device_output_and_clustering():
    g = gen.rmat(12, 16, seed=11)
    want_tv, want_cc = oracle.clustering(*g)
    with pg.build_blocks(*g, p=4) as b:
        out = torch.full((g[0],), -1, dtype=torch.int64, device="cuda")
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            t_dev = pgd.vertex_triangles_allreduce(b, out=out)     # world size 1: no collective
            cc_dev = b.local_clustering(t_dev, stream=s)
        s.synchronize()
        assert np.array_equal(t_dev.cpu().numpy().astype(np.uint64), want_tv)
        assert np.array_equal(cc_dev.cpu().numpy(), want_cc)        # bit-exact fp64
        cc_host = b.local_clustering(want_tv)
        assert np.array_equal(cc_host, want_cc)


def test_per_vertex_messy_input():
    g = gen.rmat(10, 16, seed=12)
    m = gen.messy(g, seed=5)
    _, want = oracle.count(*g, per_vertex=True)
    with pg.build_blocks(*m, p=3) as b:
        tv, _ = b.vertex_triangles()
    assert np.array_equal(tv, want)


# ---- roles and the two-pass route (DESIGN R24) -------------------------------------
@pytest.mark.parametrize("p", [1, 3, 8])
def test_roles_vs_oracle(p):
    for g in (gen.rmat(12, 16, seed=30 + p), gen.disjoint_union(gen.complete(60), gen.king(20, 30))):
        T, lo, mi, hi = oracle.count_roles(*g)
        with pg.build_blocks(*g, p=p) as b:
            t_lo, T1 = b.vertex_triangles(roles="low")
            t_lm, T2 = b.vertex_triangles(roles="low+mid")
        assert T1 == T2 == T
        assert np.array_equal(t_lo, lo)
        assert np.array_equal(t_lm - t_lo, mi)
        with pg.build_blocks(*g, p=p, reverse_order=True) as r:
            assert r.triangle_count() == T                       # reversal keeps T
            rt_lo, _ = r.vertex_triangles(roles="low")
            rt_all, _ = r.vertex_triangles()
        assert np.array_equal(rt_lo, hi)                          # lowest in reverse = highest
        assert np.array_equal(rt_all, lo + mi + hi)


def test_two_pass_vertex_triangles():
    for g, p in ((gen.rmat(14, 16, seed=41), 8), (gen.er(1 << 13, 24, seed=42), 4), (gen.grid(150, 0.4, seed=43), 5)):
        _, want = oracle.count(*g, per_vertex=True)
        tv, T = pg.vertex_triangles_two_pass(*g, p=p)
        assert np.array_equal(tv, want) and int(tv.sum()) == 3 * T


def test_reverse_order_steps_parity():
    g = gen.rmat(9, 16, seed=44)
    P = ob.Plan(*g, p=3, reverse=True, orient=0)
    with pg.build_blocks(*g, p=3, reverse_order=True) as b:
        assert (b.rank() == P.rank).all()
        assert list(b.cuts()) == list(P.cuts)
        ijx, cost, alg = b.tasks()
        assert [tuple(map(int, t)) for t in ijx] == P.tasks
        assert list(map(int, cost)) == P.costs
        T, tc = b.triangle_count(task_counts=True)
        assert list(map(int, tc)) == P.task_counts()


def test_bad_roles_rejected():
    g = gen.rmat(8, 8, seed=45)
    with pg.build_blocks(*g, p=2) as b:
        o = pg._abi.CountOpts()
        o.flags = pg._abi.ROLE_MID
        tv = np.zeros(g[0], np.uint64)
        import ctypes
        assert pg._lib.pgabb_vertex_triangles(b._h, ctypes.byref(o), tv.ctypes.data, None) == 1
