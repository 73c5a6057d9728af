"""GPU parity: the CUDA path (through the C ABI) against the oracle, bit-exact.

All arithmetic is integer, so the bar is exact equality for every step:
rank (S2), cuts (S4), block CSR (S5), tasks (S6), costs and algorithmic bytes
(S7), pieces and LPT owners (S8), per-task counts (S10) and the total (S11).
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


def gpu_T(g, **kw):
    with pg.build_blocks(*g, **kw) as b:
        return b.triangle_count()


# ---------------------------------------------------------------- closed forms
@pytest.mark.parametrize("p", [1, 2, 3, 8])
def test_closed_forms(p):
    cases = [
        (gen.complete(3), 1), (gen.complete(4), 4), (gen.complete(57), comb(57, 3)),
        (gen.cycle(3), 1), (gen.cycle(100), 0), (gen.path(50), 0), (gen.star(40), 0),
        (gen.wheel(4), 4), (gen.wheel(5), 4), (gen.wheel(300), 299),
        (gen.windmill(7, 6), 7 * comb(6, 3)), (gen.rook(5, 7), 7 * comb(5, 3) + 5 * comb(7, 3)),
        (gen.king(17, 23), 4 * 16 * 22), (gen.complete_bipartite(9, 13), 0),
        (gen.clique_union([3, 9, 200, 2, 1, 64]), sum(comb(s, 3) for s in [3, 9, 200, 2, 1, 64])),
        (gen.random_tree(500, 3), 0),
    ]
    for g, want in cases:
        assert gpu_T(g, p=p) == want, (g[0], want)


def test_grid_diagonals_closed_form():
    for side, f in [(64, 0.0), (200, 0.1), (513, 0.5), (33, 1.0)]:
        g = gen.grid(side, f, seed=2)
        assert gpu_T(g, p=5) == 2 * gen.grid_ndiag(side, f, seed=2)


def test_degenerate_inputs():
    e = np.zeros(0, np.uint32)
    assert gpu_T((0, e, e), p=4) == 0
    assert gpu_T((10, e, e), p=4) == 0
    loops = np.arange(5, dtype=np.uint32)
    assert gpu_T((5, loops, loops), p=2) == 0                    # only self-loops
    assert gpu_T((2, np.array([0, 1, 0], np.uint32), np.array([1, 0, 1], np.uint32)), p=2) == 0
    assert gpu_T((1, np.array([0], np.uint32), np.array([0], np.uint32)), p=3) == 0


def test_errors():
    with pytest.raises(pg.PgabbError) as e:
        pg.build_blocks(3, np.array([0, 3], np.uint32), np.array([1, 1], np.uint32))
    assert e.value.name == "EINVAL"
    with pytest.raises(pg.PgabbError) as e:
        pg.build_blocks(3, np.array([0], np.uint32), np.array([1], np.uint32), rank=2, world_size=2)
    assert e.value.name == "EINVAL"
    with pytest.raises(pg.PgabbError):
        pg.build_blocks(3, np.array([0], np.uint32), np.array([1], np.uint32), cut_rule=4)


# ---------------------------------------------------------------- totals vs oracle
@pytest.mark.parametrize("scale", [6, 10, 13, 16])
@pytest.mark.parametrize("p", [1, 2, 3, 5, 8, 16])
def test_rmat_total_vs_oracle(scale, p):
    g = gen.rmat(scale, 16, seed=scale)
    assert gpu_T(g, p=p) == oracle.count(*g)


@pytest.mark.parametrize("rule", [0, 1])
def test_er_grid_total_vs_oracle(rule):
    for g in (gen.er(1 << 15, 32, seed=3), gen.er(1000, 8, seed=4), gen.grid(300, 0.2, seed=5)):
        assert gpu_T(g, p=7, cut_rule=rule) == oracle.count(*g)


def test_messy_and_relabel_invariance():
    g = gen.rmat(12, 16, seed=9)
    want = oracle.count(*g)
    assert gpu_T(gen.messy(g, seed=1), p=4) == want
    assert gpu_T(gen.relabel(g, seed=2), p=4) == want


def test_device_inputs():
    g = gen.rmat(12, 16, seed=10)
    s = torch.from_numpy(g[1].view(np.int32)).cuda()
    d = torch.from_numpy(g[2].view(np.int32)).cuda()
    with pg.build_blocks(g[0], s, d, p=6) as b:
        assert b.triangle_count() == oracle.count(*g)


def test_repeat_deterministic():
    g = gen.rmat(14, 16, seed=11)
    with pg.build_blocks(*g, p=8) as b:
        r = [b.triangle_count(task_counts=True) for _ in range(3)]
    assert all(x[0] == r[0][0] for x in r)
    assert all((x[1] == r[0][1]).all() for x in r)


def test_host_residency():
    g = gen.rmat(13, 16, seed=12)
    with pg.build_blocks(*g, p=4, residency=pg.RESIDENT_HOST) as b:
        assert b.triangle_count() == oracle.count(*g)
        assert b.stats()["h2d_bytes_last"] > 0


@pytest.mark.parametrize("factor", [1.5, 3.0, 40.0])
def test_streaming_budget(factor):
    # SPEC acceptance 5 shape: budget = 1.5x the largest block-list footprint
    # (here per staging half, x2 for the two arenas); counts must not change.
    g = gen.rmat(14, 16, seed=13)
    with pg.build_blocks(*g, p=8) as ref:
        T_ref, tc_ref = ref.triangle_count(task_counts=True)
        mt = ref.stats()["max_task_bytes"]
    with pg.build_blocks(*g, p=8, residency=pg.RESIDENT_HOST, device_budget_bytes=int(2 * factor * mt)) as b:
        st = b.stats()
        assert st["waves"] >= 1
        if factor < 3:
            assert st["waves"] > 1
        for _ in range(2):   # re-use of the arenas across calls
            T, tc = b.triangle_count(task_counts=True)
            assert T == T_ref == oracle.count(*g)
            assert (tc == tc_ref).all()
        assert b.stats()["h2d_bytes_last"] > 0
        # introspection still works with the pools in host memory only
        rp, col = b.block(0, 1)
        with pg.build_blocks(*g, p=8) as ref2:
            rp2, col2 = ref2.block(0, 1)
        assert (rp == rp2).all() and (col == col2).all()


def test_streaming_budget_too_small():
    g = gen.rmat(12, 16, seed=14)
    with pg.build_blocks(*g, p=4) as ref:
        mt = ref.stats()["max_task_bytes"]
    with pytest.raises(pg.PgabbError) as e:
        pg.build_blocks(*g, p=4, residency=pg.RESIDENT_HOST, device_budget_bytes=mt)   # half < footprint
    assert e.value.name == "EBUDGET"


def test_streaming_multirank():
    g = gen.rmat(12, 16, seed=15)
    want = oracle.count(*g)
    with pg.build_blocks(*g, p=6) as ref:
        mt = ref.stats()["max_task_bytes"]
    total = 0
    for r in range(3):
        with pg.build_blocks(*g, p=6, rank=r, world_size=3, residency=pg.RESIDENT_HOST,
                             device_budget_bytes=4 * mt) as b:
            total += b.triangle_count()
    assert total == want


# ---------------------------------------------------------------- step-by-step parity
SMALL = [
    ("rmat9", lambda: gen.rmat(9, 16, seed=1)),
    ("er", lambda: gen.er_small(300, 0.05, seed=2)),
    ("king", lambda: gen.king(9, 11)),
    ("messy", lambda: gen.messy(gen.rmat(8, 8, seed=3), seed=3)),
]


@pytest.mark.parametrize("orient", [0, 1, 2])   # R25: auto, low, mid
@pytest.mark.parametrize("name,mk", SMALL)
@pytest.mark.parametrize("p,rule", [(1, 0), (2, 0), (3, 1), (5, 0), (8, 1), (4, 2), (6, 3)])
def test_steps_parity(name, mk, p, rule, orient):
    g = mk()
    P = ob.Plan(*g, p=p, rule=rule, orient=orient)
    with pg.build_blocks(*g, p=p, cut_rule=rule, orient=orient) as b:
        st = b.stats()
        assert st["m_edges"] == len(P.E)
        assert st["p"] == P.p
        assert (b.rank() == P.rank).all()                                    # S2
        assert list(b.cuts()) == list(P.cuts)                                # S4
        for (i, j), (rp, col) in P.B.items():                                # S5
            grp, gcol = b.block(i, j)
            assert list(gcol) == list(col), (i, j)
            if col.size:
                assert list(grp) == list(rp), (i, j)
        ijx, cost, alg = b.tasks()                                           # S6, S7
        assert [tuple(map(int, t)) for t in ijx] == P.tasks
        assert list(map(int, cost)) == P.costs
        assert list(map(int, alg)) == P.alg_bytes
        dirs, s_low, s_mid = b.task_orient()                                 # R25
        assert list(map(int, dirs)) == P.dirs
        if orient != 1:
            assert [(int(a), int(c)) for a, c in zip(s_low, s_mid)] == [ob.task_streams(P.B, t) for t in P.tasks]
        assert st["wedges"] == ob.wedges_dag(g[0], P.D)
        T, tc = b.triangle_count(task_counts=True)                           # S10, S11
        assert list(map(int, tc)) == P.task_counts()
        assert T == oracle.count(*g)


@pytest.mark.parametrize("orient", [0, 1, 2])
@pytest.mark.parametrize("G", [2, 3, 8])
def test_pieces_lpt_and_rank_sum(G, orient):
    g = gen.rmat(10, 16, seed=21)
    P = ob.Plan(*g, p=4, G=G, orient=orient)
    total = 0
    for r in range(G):   # logical-rank simulation on one GPU
        with pg.build_blocks(*g, p=4, rank=r, world_size=G, orient=orient) as b:
            pcs, owner = b.pieces()
            assert pcs == P.pieces                                           # S8 pieces
            assert owner == P.owner                                          # S8 LPT
            T_r, tc = b.triangle_count(task_counts=True)
            want = sum(ob.piece_count(P.B, P.tasks[pc[0]], pc[1], pc[2], P.dirs[pc[0]])
                       for pc, o in zip(P.pieces, P.owner) if o == r)
            assert T_r == want
            total += T_r
    assert total == oracle.count(*g)


# ---------------------------------------------------------------- S8 with task weights (R22)
@pytest.mark.parametrize("G", [2, 4])
def test_weighted_pieces_and_rank_sum(G):
    g = gen.rmat(11, 16, seed=22)
    with pg.build_blocks(*g, p=5) as b1:
        nt = b1.ntasks
    rng = np.random.default_rng(G)
    w = rng.integers(0, 10 ** 9, nt).astype(np.uint64)
    P = ob.Plan(*g, p=5, G=G, weights=[int(x) for x in w], orient=0)
    total = 0
    for r in range(G):
        with pg.build_blocks(*g, p=5, rank=r, world_size=G, task_weights=w, orient=0) as b:
            pcs, owner = b.pieces()
            assert pcs == P.pieces and owner == P.owner
            total += b.triangle_count()
    assert total == oracle.count(*g)


def test_task_times_drive_a_balanced_plan():
    g = gen.rmat(14, 16, seed=23)
    with pg.build_blocks(*g, p=8) as b1:
        ns = b1.task_times()
        st = b1.stats()
        T1 = b1.triangle_count()
    assert ns.shape == (b1.ntasks,) and ns.sum() > 0
    # the estimates add up to the measured kernel time (ns), up to rounding
    assert abs(int(ns.sum()) - 1e6 * st["ms_main_kernel_last"]) <= 1e6 * st["ms_main_kernel_last"] * 0.01 + b1.ntasks
    total = 0
    for r in range(4):
        with pg.build_blocks(*g, p=8, rank=r, world_size=4, task_weights=ns) as b:
            total += b.triangle_count()
    assert total == T1 == oracle.count(*g)
    with pytest.raises(pg.PgabbError) as e:
        pg.build_blocks(*g, p=8, task_weights=ns[:-1])
    assert e.value.name == "EINVAL"


# ---------------------------------------------------------------- size limits
def test_max_parts_and_clamp():
    g = gen.rmat(12, 16, seed=51)
    T = oracle.count(*g)
    with pg.build_blocks(*g, p=64) as b:                 # kMaxParts: C(66,3) = 45760 candidate triples
        assert b.stats()["p"] == 64
        assert b.triangle_count() == T
        ijx, _, _ = b.tasks()
        assert all(i <= j <= x < 64 for i, j, x in ijx)
    with pytest.raises(pg.PgabbError) as e:
        pg.build_blocks(*g, p=65)
    assert e.value.name == "EINVAL"
    small = gen.complete(5)
    with pg.build_blocks(*small, p=40) as b:             # p > n is clamped to n (R7)
        assert b.stats()["p"] == 5 and b.triangle_count() == 10


# ------------------------------------------- medium thread-per-row items (R29)
@pytest.mark.parametrize("p", [2, 4])
def test_light_held_classes(p):
    # ER at p = 2 / 4 holds many rows with 9..15 ids per block row: with
    # light_held = 15 they run in the medium kernel instead of heavy warp items
    for g in (gen.er(1 << 15, 32, seed=21), gen.rmat(13, 16, seed=22)):
        want = oracle.count(*g)
        res = {}
        for lh in (8, 15, 0):
            with pg.build_blocks(*g, p=p, light_held=lh) as b:
                T, tc = b.triangle_count(task_counts=True)
                st = b.stats()
            assert T == want
            res[lh] = (tc, st["items_heavy"], st["items_light"])
        assert (res[8][0] == res[15][0]).all()
        assert res[15][2] >= res[8][2] and res[15][1] <= res[8][1]
    # the ER case really moves rows into the medium list
    g = gen.er(1 << 15, 32, seed=21)
    with pg.build_blocks(*g, p=p, light_held=8) as b8, pg.build_blocks(*g, p=p, light_held=15) as b15:
        s8, s15 = b8.stats(), b15.stats()
        assert s15["items_light"] > s8["items_light"] and s8["items_medium"] == 0
        assert s15["items_light"] - s15["items_medium"] == s8["items_light"]
        assert (s8["light_held"], s15["light_held"]) == (8, 15)
        # R30 slots only with medium rows on a device-resident handle
        assert s8["ell_bytes"] == 0 and s15["ell_bytes"] > 0


def test_light_held_streaming_and_rejects():
    g = gen.er(1 << 14, 32, seed=23)
    want = oracle.count(*g)
    with pg.build_blocks(*g, p=4, light_held=15) as ref:
        mt = ref.stats()["max_task_bytes"]
    with pg.build_blocks(*g, p=4, light_held=15, residency=pg.RESIDENT_HOST, device_budget_bytes=int(5 * mt)) as b:
        assert b.stats()["waves"] > 1 and b.stats()["ell_bytes"] == 0
        assert b.triangle_count() == want
    with pg.build_blocks(*g, p=4, light_held=15, residency=pg.RESIDENT_HOST) as b:
        assert b.stats()["ell_bytes"] == 0
        assert b.triangle_count() == want


@pytest.mark.parametrize("p", [1, 3])
def test_ell_slots_long_rows(p):
    # R30: rows longer than a slot continue in the col pool (scanned or binary-
    # searched); ER d = 48 at p = 1 / 3 puts many rows past 15 ids
    g = gen.er(1 << 14, 48, seed=24)
    want = oracle.count(*g)
    with pg.build_blocks(*g, p=p, light_held=15) as b:
        T, tc = b.triangle_count(task_counts=True)
        st = b.stats()
    with pg.build_blocks(*g, p=p, light_held=8) as b8:
        T8, tc8 = b8.triangle_count(task_counts=True)
    assert T == T8 == want and (tc == tc8).all()
    if p == 3:   # blocks of ~8 ids per row get 16-word slots (p = 1: ~24 per row, none)
        assert st["items_medium"] > 0 and st["ell_bytes"] > 0
    with pytest.raises(pg.PgabbError) as e:
        pg.build_blocks(*g, p=4, light_held=9)
    assert e.value.name == "EINVAL"
