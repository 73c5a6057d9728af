"""Pins of oracle/blocks.py (the block method's intermediate objects).

Hand-derived examples (worked in the comments, SPEC.md-style), the block method's
correctness theorem (sum of per-task counts = T from the node iterator and brute
force), and structural invariants.
"""
import itertools
from math import comb

import numpy as np
import pytest

import gen
import oracle
import oracle.blocks as ob


# ---- S1 canonicalise ---------------------------------------------------------------
def test_canonical_vs_set():
    n, s, d = gen.messy(gen.rmat(8, 8, 3), seed=2)
    E = ob.canonical_edges(n, s, d)
    ref = sorted({(min(int(a), int(b)), max(int(a), int(b))) for a, b in zip(s, d) if a != b})
    assert [tuple(map(int, e)) for e in E] == ref


# ---- S2 degree order (SPEC.md degree_relabel examples) ------------------------------
def test_rank_star_hub_last():
    n, s, d = gen.star(5)
    E = ob.canonical_edges(n, s, d)
    r = ob.degree_rank(n, ob.degrees(n, E))
    assert r[0] == n - 1


def test_rank_ring_identity():
    n, s, d = gen.cycle(7)
    E = ob.canonical_edges(n, s, d)
    assert (ob.degree_rank(n, ob.degrees(n, E)) == np.arange(7)).all()


def test_rank_p4_ties_by_id():
    # P4 degrees [1,2,2,1] -> order 0,3,1,2 -> rank = [0,2,3,1]
    n, s, d = gen.path(4)
    E = ob.canonical_edges(n, s, d)
    assert list(ob.degree_rank(n, ob.degrees(n, E))) == [0, 2, 3, 1]


# ---- S3 orient -------------------------------------------------------------------
def test_dag_half_edges_low_to_high():
    g = gen.rmat(9, 16, 1)
    E = ob.canonical_edges(*g)
    rank = ob.degree_rank(g[0], ob.degrees(g[0], E))
    D = ob.dag(E, rank)
    assert D.shape == E.shape
    assert (D[:, 0] < D[:, 1]).all()
    assert len({tuple(x) for x in D}) == len(D)


# ---- S4 cuts: hand examples ----------------------------------------------------------
def _plan_objs(g, p, rule=0):
    n = g[0]
    E = ob.canonical_edges(*g)
    rank = ob.degree_rank(n, ob.degrees(n, E))
    D = ob.dag(E, rank)
    return n, D, ob.cuts(n, D, p, rule)


def test_cuts_p4_hand():
    # P4: DAG (rank space) (0,2),(1,3),(2,3); d+=[1,1,1,0], d-=[0,0,1,2]
    # rule 0 weights [1,1,2,0], P=[0,1,2,4,4]: p=2 -> [0,2,4]; p=3 -> [0,2,3,4]
    # rule 1 weights [1,1,1,0], P=[0,1,2,3,3]: p=2 -> 2P>=3 -> c=2
    # rule 2 weights deg [1,1,2,2], P=[0,1,2,4,6]: p=2 -> 2P>=6 -> c=3 -> [0,3,4]
    # rule 3 weights d+ + C(d+,2) = [1,1,1,0] (C(1,2) = 0): as rule 1
    g = gen.path(4)
    assert list(_plan_objs(g, 2, 0)[2]) == [0, 2, 4]
    assert list(_plan_objs(g, 3, 0)[2]) == [0, 2, 3, 4]
    assert list(_plan_objs(g, 2, 1)[2]) == [0, 2, 4]
    assert list(_plan_objs(g, 2, 2)[2]) == [0, 3, 4]
    assert list(_plan_objs(g, 2, 3)[2]) == [0, 2, 4]


def test_cut_weights_rules_2_3_k4():
    # K4: d+ = [3,2,1,0], d- = [0,1,2,3]: degree 3 each; d+ + C(d+,2) = [6,3,1,0]
    n, D, _ = _plan_objs(gen.complete(4), 1)
    assert [int(x) for x in ob.cut_weights(n, D, 2)] == [3, 3, 3, 3]
    assert [int(x) for x in ob.cut_weights(n, D, 3)] == [6, 3, 1, 0]


def test_cuts_p1_and_clamp():
    g = gen.rmat(7, 8, 1)
    assert list(_plan_objs(g, 1)[2]) == [0, g[0]]
    n, D, c = _plan_objs(gen.complete(3), 10)
    assert len(c) == 4 and c[0] == 0 and c[-1] == 3   # p clamped to n


def test_cuts_balance_property():
    # prefix cuts: every part's weight <= W/p + max single weight
    g = gen.rmat(10, 16, 2)
    for rule in (0, 1, 2, 3):
        for p in (2, 3, 5, 8):
            n, D, c = _plan_objs(g, p, rule)
            w = np.array([int(x) for x in ob.cut_weights(n, D, rule)], dtype=np.int64)
            assert (np.diff(c) >= 0).all()
            parts = [w[c[k]:c[k + 1]].sum() for k in range(p)]
            assert max(parts) <= w.sum() / p + w.max()


# ---- S5 blocks -------------------------------------------------------------------
def test_blocks_k3_hand():
    # K3: rank = id; DAG (0,1),(0,2),(1,2); rule 0 w=[2,2,0] -> cuts [0,1,3]
    # A_00 empty; A_01 row0 -> local cols {0,1}; A_11 row0 -> {1}
    n, D, c = _plan_objs(gen.complete(3), 2)
    assert list(c) == [0, 1, 3]
    B = ob.blocks(D, c)
    assert B[(0, 0)][1].size == 0
    assert list(B[(0, 1)][0]) == [0, 2] and list(B[(0, 1)][1]) == [0, 1]
    assert list(B[(1, 1)][0]) == [0, 1, 1] and list(B[(1, 1)][1]) == [1]


def test_blocks_edge_cover():
    g = gen.rmat(10, 16, 4)
    for p in (1, 2, 3, 5, 8):
        n, D, c = _plan_objs(g, p)
        B = ob.blocks(D, c)
        assert sum(v[1].size for v in B.values()) == len(D)
        got = set()
        for (i, j), (rp, col) in B.items():
            for r in range(rp.size - 1):
                for v in col[rp[r]:rp[r + 1]]:
                    got.add((int(r + c[i]), int(v + c[j])))
        assert got == {tuple(map(int, e)) for e in D}


# ---- S6 tasks + S10 counts: the block method's correctness theorem ------------------
def test_tasks_k3_hand_and_counts():
    # tasks (0,1,1), (1,1,1); counts: edge (0->1) finds {2}; others 0 -> [1, 0]
    P = ob.Plan(*gen.complete(3), p=2)
    assert P.tasks == [(0, 1, 1), (1, 1, 1)]
    assert P.task_counts() == [1, 0]


def test_tasks_dense_is_all_triples():
    P = ob.Plan(*gen.complete(40), p=4)
    assert len(P.tasks) == comb(4 + 2, 3)


def test_p4_tasks_hand():
    P = ob.Plan(*gen.path(4), p=2)
    assert P.tasks == [(0, 1, 1), (1, 1, 1)]
    assert P.task_counts() == [0, 0]


@pytest.mark.parametrize("p", [1, 2, 3, 5, 8])
def test_sum_task_counts_is_T(p):
    for g in (gen.rmat(8, 16, 1), gen.er_small(120, 0.15, 3), gen.king(6, 7), gen.wheel(30)):
        P = ob.Plan(*g, p=p)
        tc = P.task_counts()
        assert sum(tc) == oracle.count(*g) == oracle.brute(*g)


def test_p1_single_task():
    g = gen.rmat(8, 16, 5)
    P = ob.Plan(*g, p=1)
    assert P.tasks == [(0, 0, 0)]
    assert P.task_counts() == [oracle.count(*g)]


# ---- S7 cost and algorithmic bytes: hand examples ----------------------------------
def test_cost_k4_hand():
    # K4, p=1: d+ = [3,2,1,0]; cost = sum over DAG edges (d+(u)+d+(v))
    #   = 5+4+3+3+2+1 = 18; alg elements = (3+2+1) + (2+1+0+1+0+0) = 10 -> 40 + 12*6
    P = ob.Plan(*gen.complete(4), p=1)
    assert P.costs == [18]
    assert P.alg_bytes == [4 * 10 + 12 * 6]


def test_cost_k3_p2_hand():
    # (0,1,1): edges (0,0): 2+1, (0,1): 2+0 -> 5; (1,1,1): edge (0,1): 1+0 -> 1
    # alg: (0,1,1): 2 + (1+0) = 3 el, 2 edges -> 36; (1,1,1): 1 + 0 el, 1 edge -> 16
    P = ob.Plan(*gen.complete(3), p=2)
    assert P.costs == [5, 1]
    assert P.alg_bytes == [36, 16]


def test_alg_bytes_skip_rows_without_x_neighbours():
    # star with centre c and leaves; ranks: leaves first (deg 1), centre last.  Add a
    # triangle among three leaves to create DAG rows with edges into some parts only.
    # Pinned against an independent restatement over the DAG (no block CSR):
    #   sum over tasks (i,j,x), over u in part i with N+_j(u), N+_x(u) both non-empty, of
    #   4*(|N+_x(u)| + sum_{v in N+_j(u)} |N+_x(v)|) + 12*|N+_j(u)|.
    for g, p in ((gen.rmat(8, 8, seed=7), 3), (gen.er_small(120, 0.06, seed=8), 4), (gen.king(6, 7), 5)):
        P = ob.Plan(*g, p=p)
        part = np.searchsorted(np.asarray(P.cuts), np.arange(g[0]), side="right") - 1
        nplus = {}
        for a_, b_ in P.D:
            nplus.setdefault(int(a_), []).append(int(b_))
        def nx_(u, x):
            return [w for w in nplus.get(u, []) if part[w] == x]
        want = []
        for (i, j, x) in P.tasks:
            tot = 0
            for u in range(g[0]):
                if part[u] != i:
                    continue
                nj, nxu = nx_(u, j), nx_(u, x)
                if nj and nxu:
                    tot += 4 * (len(nxu) + sum(len(nx_(v, x)) for v in nj)) + 12 * len(nj)
            want.append(tot)
        assert P.alg_bytes == want
        # rows without x-neighbours really occur here (the old all-rows model differs)
        old = 0
        for (i, j, x) in P.tasks:
            for u in range(g[0]):
                nj = nx_(u, j) if part[u] == i else []
                if nj:
                    old += 4 * (len(nx_(u, x)) + sum(len(nx_(v, x)) for v in nj)) + 12 * len(nj)
        assert sum(want) < old


# ---- S8 pieces and LPT -------------------------------------------------------------
def test_pieces_k4_hand():
    # G=2: cap = ceil(18/8) = 3, k = 6; row costs [12,5,1,0], R=[0,12,17,18,18]
    # boundaries q=1..5 -> [1,1,1,1,2]; pieces [0,1):12, [1,2):5, [2,4):1
    P = ob.Plan(*gen.complete(4), p=1, G=2)
    assert P.pieces == [(0, 0, 1, 12), (0, 1, 2, 5), (0, 2, 4, 1)]
    assert P.owner == [0, 1, 1]
    assert P.loads == [12, 6]


def test_weighted_pieces_k4_hand():
    # E = [36] (reading R22): cap = ceil(36/8) = 5, k = ceil(36/5) = 8; boundaries
    # rho_q = min{rho : 8 R[rho] >= 18 q}, R = [0,12,17,18,18] -> q=1..5: 1, q=6,7: 2.
    # Ranges [0,1) c=12, [1,2) c=5, [2,4) c=1; weights floor(36 c / 18) = 24, 10, 2.
    P = ob.Plan(*gen.complete(4), p=1, G=2, weights=[36])
    assert P.pieces == [(0, 0, 1, 24), (0, 1, 2, 10), (0, 2, 4, 2)]
    assert P.owner == [0, 1, 1] and P.loads == [24, 12]


def test_weights_equal_to_costs_change_nothing():
    g = gen.rmat(9, 16, seed=3)
    for G in (1, 2, 5):
        A = ob.Plan(*g, p=4, G=G)
        B = ob.Plan(*g, p=4, G=G, weights=A.costs)
        assert A.pieces == B.pieces and A.owner == B.owner


def test_weights_steer_lpt():
    # two equal-cost tasks made unequal by E: the heavier one gets a rank of its own
    g = gen.rmat(9, 16, seed=4)
    A = ob.Plan(*g, p=3, G=3)
    w = [0] * len(A.tasks)
    heavy = int(np.argmax(A.costs))
    w[heavy] = 10 ** 12
    B = ob.Plan(*g, p=3, G=3, weights=w)
    owners_heavy = {o for pc, o in zip(B.pieces, B.owner) if pc[0] == heavy}
    owners_rest = {o for pc, o in zip(B.pieces, B.owner) if pc[0] != heavy}
    # E of the heavy task is above the cap: it is split over all ranks; every task is still assigned
    assert len(owners_heavy) == 3
    assert {pc[0] for pc in B.pieces} == {t for t, c in enumerate(A.costs) if c > 0}
    assert owners_rest


def test_lpt_hand():
    pcs = [(0, 0, 1, 5), (1, 0, 1, 4), (2, 0, 1, 3), (3, 0, 1, 3), (4, 0, 1, 3)]
    owner, loads = ob.lpt(pcs, 2)
    assert owner == [0, 1, 1, 0, 1] and loads == [8, 10]


def test_lpt_within_graham_bound():
    rng = np.random.default_rng(1)
    for _ in range(30):
        G = int(rng.integers(2, 4))
        costs = [int(x) for x in rng.integers(1, 50, size=int(rng.integers(3, 8)))]
        pcs = [(k, 0, 1, c) for k, c in enumerate(costs)]
        _, loads = ob.lpt(pcs, G)
        opt = min(max(sum(c for c, a in zip(costs, asg) if a == g) for g in range(G))
                  for asg in itertools.product(range(G), repeat=len(costs)))
        assert max(loads) <= (4 / 3 - 1 / (3 * G)) * opt + 1e-9


@pytest.mark.parametrize("G", [2, 3, 8])
def test_pieces_partition_tasks(G):
    g = gen.rmat(9, 16, 7)
    P = ob.Plan(*g, p=3, G=G)
    tc = P.task_counts()
    for ti, t in enumerate(P.tasks):
        mine = [pc for pc in P.pieces if pc[0] == ti]
        assert sum(pc[3] for pc in mine) == P.costs[ti]
        assert sum(ob.piece_count(P.B, t, pc[1], pc[2]) for pc in mine) == tc[ti]
        for a, b in zip(mine, mine[1:]):
            assert a[2] <= b[1]
    per_rank = [0] * G
    for pc, o in zip(P.pieces, P.owner):
        per_rank[o] += ob.piece_count(P.B, P.tasks[pc[0]], pc[1], pc[2])
    assert sum(per_rank) == oracle.count(*g)


# ---- R25 orientation: MID holds A_jx[v] and streams only ids w > v ------------------
def _wedge_counts(P, t):
    """Direct enumeration over the DAG (not the blocks): S_low = #{(u,v,w): (u,v) in
    A_ij, (v,w) in the DAG with w in part x}; S_mid = #{(u,v,w): (u,v), (u,w) in the
    DAG, v < w, u in part i, v in part j, w in part x}."""
    i, j, x = t
    out = {}
    for a, b in P.D:
        out.setdefault(int(a), []).append(int(b))
    part = lambda r: int(ob.part_of(P.cuts, r))
    s_low = s_mid = 0
    for u, vs in out.items():
        if part(u) != i:
            continue
        for v in vs:
            if part(v) != j:
                continue
            s_low += sum(1 for w in out.get(v, []) if part(w) == x)
            s_mid += sum(1 for w in vs if w > v and part(w) == x)
    return s_low, s_mid


@pytest.mark.parametrize("g", [gen.rmat(7, 8, 1), gen.er(150, 12, 2), gen.complete(9), gen.king(6, 7)])
def test_mid_streams_p1_out_out_wedges(g):
    # p = 1: MID streams every pair v < w of out-neighbours of u once: sum_u C(d+(u), 2);
    # LOW streams d+(v) per DAG edge (u,v): W = sum_v d-(v) d+(v)
    P = ob.Plan(*g, p=1)
    if not P.tasks:
        return
    s_low, s_mid = ob.task_streams(P.B, P.tasks[0])
    assert s_mid == ob.out_out_wedges(P.n, P.D)
    assert s_low == ob.wedges_dag(P.n, P.D)


@pytest.mark.parametrize("p", [2, 3, 5])
def test_mid_streams_vs_wedge_enumeration(p):
    g = gen.rmat(7, 8, 5)
    P = ob.Plan(*g, p=p)
    for t in P.tasks:
        assert ob.task_streams(P.B, t) == _wedge_counts(P, t)


def test_mid_costs_k4_by_hand():
    # K4, p = 1: DAG 0->{1,2,3}, 1->{2,3}, 2->{3}.  Rows v of MID:
    #   v=1: column {0}; |A[1]| = 2 + ids of A[0] after 1 = {2,3}: 2      -> 4
    #   v=2: column {0,1}; |A[2]| = 1 + {3} + {3}                         -> 3
    #   v=3: column {0,1,2}; |A[3]| = 0 + nothing after 3                 -> 0
    # cost 7; bytes: v=1 4*(2+2)+12, v=2 4*(1+2)+24 (v=3 holds nothing) = 64.
    # Streams: S_low = sum over edges of |A[v]| = 2+1+0+1+0+0 = 4, S_mid = C(3,2)+C(2,2) = 4:
    # no saving, so auto keeps LOW.
    P = ob.Plan(*gen.complete(4), p=1, orient=2)
    t = P.tasks[0]
    assert list(ob.row_costs_mid(P.B, t)) == [0, 4, 3, 0]
    assert P.costs == [7] and P.alg_bytes == [64] and P.dirs == [ob.MID]
    assert ob.task_streams(P.B, t) == (4, 4)
    assert ob.Plan(*gen.complete(4), p=1, orient=0).dirs == [ob.LOW]


def test_auto_orientation_picks_fewer_streams():
    g = gen.rmat(9, 16, 3)
    P = ob.Plan(*g, p=4, orient=0)
    assert ob.MID in P.dirs
    for t, d in zip(P.tasks, P.dirs):
        s_low, s_mid = ob.task_streams(P.B, t)
        assert d == (ob.MID if s_mid + 2 * P.B[(t[0], t[1])][1].size < s_low and 4 * s_mid < 3 * s_low
                     else ob.LOW)


@pytest.mark.parametrize("orient", [0, 2])
@pytest.mark.parametrize("G", [1, 3])
def test_mid_pieces_partition_tasks(orient, G):
    g = gen.rmat(9, 16, 7)
    P = ob.Plan(*g, p=3, G=G, orient=orient)
    tc = P.task_counts()
    for ti, t in enumerate(P.tasks):
        d = P.dirs[ti]
        mine = [pc for pc in P.pieces if pc[0] == ti]
        assert sum(pc[3] for pc in mine) == P.costs[ti]
        assert sum(ob.piece_count(P.B, t, pc[1], pc[2], d) for pc in mine) == tc[ti]
        nrows = int(P.cuts[t[0] + 1] - P.cuts[t[0]]) if d == ob.LOW else int(P.cuts[t[1] + 1] - P.cuts[t[1]])
        assert mine[0][1] == 0 and mine[-1][2] == nrows
        for a, b in zip(mine, mine[1:]):
            assert a[2] <= b[1]
    total = sum(ob.piece_count(P.B, P.tasks[pc[0]], pc[1], pc[2], P.dirs[pc[0]]) for pc in P.pieces)
    assert total == oracle.count(*g)
