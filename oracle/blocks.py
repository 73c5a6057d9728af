"""TEST INFRASTRUCTURE ONLY -- plain numpy definitions of the block method's steps.

Each function is the step's definition written out, for graphs small enough
that per-edge Python loops finish in seconds.  Step names follow SURVEY.md
§8(a) (S1..S8); readings R1..R19 are listed in DESIGN.md §3.

No code here is shared with, or imported by, the CUDA path.
"""
from __future__ import annotations

import numpy as np


# S1 -- canonicalise (§5.1: "transformed all graphs to
# undirected, and removed duplicate edges"; readings R1 self-loops, R2 dups).
def canonical_edges(n: int, src, dst) -> np.ndarray:
    """Sorted unique undirected non-loop edges as rows (a, b), a < b."""
    s = np.asarray(src, dtype=np.int64)
    d = np.asarray(dst, dtype=np.int64)
    if s.size and (s.max() >= n or d.max() >= n):
        raise ValueError("vertex id >= n")
    keep = s != d
    a = np.minimum(s, d)[keep]
    b = np.maximum(s, d)[keep]
    key = np.unique(a * int(n) + b)
    return np.stack([key // int(n), key % int(n)], 1) if key.size else np.zeros((0, 2), np.int64)


# S2 -- degree and degree order (§5.4; reading R3: ties by id).
def degrees(n: int, E: np.ndarray) -> np.ndarray:
    return np.bincount(E.ravel(), minlength=n).astype(np.int64)


def degree_rank(n: int, deg: np.ndarray, reverse: bool = False) -> np.ndarray:
    """rank[v] = position of v when vertices are sorted by (deg, id) ascending;
    reverse (reading R24): n - 1 - that position."""
    order = np.lexsort((np.arange(n), deg))
    rank = np.empty(n, np.int64)
    rank[order] = np.arange(n)
    return (n - 1 - rank) if reverse else rank


# S3 -- orient + relabel ("only requires half of the edges";
# reading R4: low rank -> high rank).
def dag(E: np.ndarray, rank: np.ndarray) -> np.ndarray:
    """DAG edges (r_lo, r_hi) in rank space, sorted by (row, col)."""
    if E.shape[0] == 0:
        return np.zeros((0, 2), np.int64)
    r = rank[E]
    lo, hi = r.min(1), r.max(1)
    o = np.lexsort((hi, lo))
    return np.stack([lo[o], hi[o]], 1)


# S4 -- conformal cuts (§4.3; reading R7).
def effective_p(n: int, p: int) -> int:
    if p <= 0:
        p = 8
    return max(1, min(p, n)) if n > 0 else 1


def cut_weights(n: int, D: np.ndarray, rule: int) -> np.ndarray:
    dplus = np.bincount(D[:, 0], minlength=n).astype(object) if D.size else np.zeros(n, object)
    dminus = np.bincount(D[:, 1], minlength=n).astype(object) if D.size else np.zeros(n, object)
    if rule == 0:        # estimated staged work: d+ (edges) + d- * d+ (list streams)
        return dplus + dminus * dplus
    if rule == 1:        # DAG out-degree
        return dplus
    if rule == 2:        # degree
        return dplus + dminus
    if rule == 3:        # estimated MID work (R25): d+ + C(d+, 2), the ids streamed for u's list
        return np.array([int(x) + int(x) * (int(x) - 1) // 2 for x in dplus], dtype=object)
    raise ValueError("cut rule")


def cuts(n: int, D: np.ndarray, p: int, rule: int = 0) -> np.ndarray:
    """cut_0 = 0, cut_p = n, cut_j = min{c : p * P[c] >= j * P[n]} (P = prefix of w)."""
    p = effective_p(n, p)
    w = cut_weights(n, D, rule)
    P = [0]
    for x in w:
        P.append(P[-1] + int(x))
    Wt = P[-1]
    out = [0]
    for j in range(1, p):
        c = 0
        while p * P[c] < j * Wt:
            c += 1
        out.append(c)
    out.append(n)
    return np.array(out, np.int64)


def part_of(cuts_: np.ndarray, r) -> np.ndarray:
    """part(r) = the j with cut_j <= r < cut_{j+1}."""
    return np.searchsorted(cuts_, r, side="right") - 1


# S5 -- block CSR (§4.3.2: "rearranges vertex ids within a block
# and uses Compressed Sparse Row"; §3.1 blocks are edge-disjoint).
def blocks(D: np.ndarray, cuts_: np.ndarray):
    """{(i, j): (rowptr, col)} for i <= j; rows local to part i, cols local to part j."""
    p = len(cuts_) - 1
    pr = part_of(cuts_, D[:, 0]) if D.size else np.zeros(0, np.int64)
    pc = part_of(cuts_, D[:, 1]) if D.size else np.zeros(0, np.int64)
    B = {}
    for i in range(p):
        wi = int(cuts_[i + 1] - cuts_[i])
        for j in range(i, p):
            sel = (pr == i) & (pc == j)
            rows = D[sel, 0] - cuts_[i]
            col = D[sel, 1] - cuts_[j]
            rowptr = np.zeros(wi + 1, np.int64)
            np.add.at(rowptr, rows + 1, 1)
            B[(i, j)] = (np.cumsum(rowptr), col.astype(np.int64))
    return B


def row(B, i, j, r):
    rp, col = B[(i, j)]
    return col[rp[r]:rp[r + 1]]


# S6 -- block triples (Listing 5 PAPER.md:682-701 code reading, reading R5;
# pruning reading R6).
def tasks(B, p: int):
    out = []
    for i in range(p):
        for j in range(i, p):
            if B[(i, j)][1].size == 0:
                continue
            for x in range(j, p):
                if B[(i, x)][1].size and B[(j, x)][1].size:
                    out.append((i, j, x))
    return out


def _edges(B, i, j):
    rp, col = B[(i, j)]
    u = np.repeat(np.arange(rp.size - 1), np.diff(rp))
    return u, col


# S10 -- the task's count: sum over (u,v) in A_ij of |A_ix[u] ∩ A_jx[v]|
# (Listing 5 lines "N_u = Edges(E_l, u); N_v = Edges(E_m, v); n_t += Intersect").
def task_count(B, t) -> int:
    i, j, x = t
    c = 0
    for u, v in zip(*_edges(B, i, j)):
        c += np.intersect1d(row(B, i, x, u), row(B, j, x, v), assume_unique=True).size
    return int(c)


# S7 -- cost (§4.4, the E functor; reading R17).
def row_costs(B, t) -> np.ndarray:
    """rowcost(r) = sum_{v in A_ij[r]} (|A_ix[r]| + |A_jx[v]|), local rows of part i."""
    i, j, x = t
    rp_ij, col = B[(i, j)]
    rp_ix = B[(i, x)][0]
    rp_jx = B[(j, x)][0]
    nrows = rp_ij.size - 1
    out = np.zeros(nrows, np.int64)
    for r in range(nrows):
        lu = rp_ix[r + 1] - rp_ix[r]
        for v in col[rp_ij[r]:rp_ij[r + 1]]:
            out[r] += lu + (rp_jx[v + 1] - rp_jx[v])
    return out


def task_cost(B, t) -> int:
    return int(row_costs(B, t).sum())


def task_alg_bytes(B, t) -> int:
    """Staged model (reading R19): over the rows u of part i with
    A_ij[u] and A_ix[u] both non-empty (a row with an empty A_ix[u] has nothing to
    intersect), 4*(|A_ix[u]| + sum over v in A_ij[u] of |A_jx[v]|) + 12*|A_ij[u]|."""
    i, j, x = t
    rp_ij, col = B[(i, j)]
    rp_ix = B[(i, x)][0]
    rp_jx = B[(j, x)][0]
    total = 0
    for r in range(rp_ij.size - 1):
        la = int(rp_ix[r + 1] - rp_ix[r])
        vs = col[rp_ij[r]:rp_ij[r + 1]]
        if la == 0 or vs.size == 0:
            continue
        el = la + sum(int(rp_jx[v + 1] - rp_jx[v]) for v in vs)
        total += 4 * el + 12 * vs.size
    return int(total)


# Reading R25 -- the orientation of a task's intersections.  Listing 5
# fixes WHAT a task sums, |A_ix[u] ∩ A_jx[v]| over (u,v) in
# A_ij, not which list is held and which is streamed.  LOW (the listing's own
# loop order): per row u of part i hold A_ix[u], stream A_jx[v] for every v in
# A_ij[u].  MID: per row v of part j hold A_jx[v], and for every u with (u,v) in
# A_ij stream only the part of A_ix[u] that can close a triangle, the ids w > v:
# A_jx[v] holds only ids > v (the DAG runs low -> high, R4), so no other w can
# be common.  When x > j every id of part x is > v; when x == j (A_ix = A_ij)
# it is the suffix of A_ij[u] after v.  Both sum the same intersections.
LOW, MID = 0, 1


def column(B, i, j, v):
    """(u, e): the rows u of part i with (u, v) in A_ij, ascending, and the
    block-local position e of (u, v) in A_ij's col array."""
    rp, col = B[(i, j)]
    e = np.nonzero(col == v)[0]
    u = np.searchsorted(rp, e, side="right") - 1
    return u, e


def streamed_mid(B, t, u, v, e) -> int:
    """|{w in A_ix[u] : w > v}| (only the ids that can be in A_jx[v])."""
    i, j, x = t
    if x > j:
        return int(row(B, i, x, u).size)
    rp = B[(i, j)][0]
    return int(rp[u + 1] - (e + 1))


def task_streams(B, t):
    """(S_low, S_mid): the ids each orientation streams, summed over (u,v) in A_ij:
    S_low = sum |A_jx[v]|, S_mid = sum |{w in A_ix[u] : w > v}|."""
    i, j, x = t
    rp_jx = B[(j, x)][0]
    s_low = s_mid = 0
    rp_ij, col = B[(i, j)]
    for u in range(rp_ij.size - 1):
        for e in range(rp_ij[u], rp_ij[u + 1]):
            v = col[e]
            s_low += int(rp_jx[v + 1] - rp_jx[v])
            s_mid += streamed_mid(B, t, u, v, e)
    return s_low, s_mid


MID_SAVING = 2


def orientation(B, t, orient=0) -> int:
    """orient 1 = LOW, 2 = MID, 0 = auto: MID iff it streams (a) more than
    MID_SAVING fewer ids per visit (per edge of A_ij), S_mid + 2 nnz(A_ij) < S_low,
    and (b) at most 3/4 of LOW's ids, 4 S_mid < 3 S_low.  A MID visit first reads
    the transpose's u (and suffix position), which short lists do not repay, and
    LOW streams hub lists as bitmap words, which a small saving does not beat
    (DESIGN R25: ER, grid and R-MAT hub tasks measured faster in LOW)."""
    if orient == 1:
        return LOW
    if orient == 2:
        return MID
    s_low, s_mid = task_streams(B, t)
    visits = int(B[(t[0], t[1])][1].size)
    return MID if s_mid + MID_SAVING * visits < s_low and 4 * s_mid < 3 * s_low else LOW


def row_costs_mid(B, t) -> np.ndarray:
    """rowcost(v), local rows v of part j: |A_jx[v]| (held once) if some u has
    (u,v) in A_ij, plus sum over those u of |{w in A_ix[u] : w > v}|."""
    i, j, x = t
    rp_jx = B[(j, x)][0]
    nrows = rp_jx.size - 1
    out = np.zeros(nrows, np.int64)
    for v in range(nrows):
        us, es = column(B, i, j, v)
        if us.size == 0:
            continue
        out[v] = int(rp_jx[v + 1] - rp_jx[v]) + sum(streamed_mid(B, t, u, v, e) for u, e in zip(us, es))
    return out


def task_cost_mid(B, t) -> int:
    return int(row_costs_mid(B, t).sum())


def task_alg_bytes_mid(B, t) -> int:
    """Staged model of a MID task (R25, the R19 model with the roles swapped): over
    the rows v of part j with A_jx[v] and column v of A_ij both non-empty,
    4*(|A_jx[v]| + sum over those u of |{w in A_ix[u] : w > v}|) + 12 per u."""
    i, j, x = t
    rp_jx = B[(j, x)][0]
    total = 0
    for v in range(rp_jx.size - 1):
        lv = int(rp_jx[v + 1] - rp_jx[v])
        us, es = column(B, i, j, v)
        if lv == 0 or us.size == 0:
            continue
        total += 4 * (lv + sum(streamed_mid(B, t, u, v, e) for u, e in zip(us, es))) + 12 * us.size
    return int(total)


def out_out_wedges(n: int, D: np.ndarray) -> int:
    """sum_u C(d+(u), 2): the pairs v < w of out-neighbours of a vertex (in rank
    space), i.e. what MID streams over all tasks at p = 1."""
    if D.size == 0:
        return 0
    dp = np.bincount(D[:, 0], minlength=n).astype(np.int64)
    return int((dp * (dp - 1) // 2).sum())


# S8 -- pieces and LPT (§4.1/§4.4 "sorts them in
# decreasing order"; reading R18).
def pieces(B, tasks_, costs, G: int, weights=None, dirs=None):
    """[(task_idx, row_begin, row_end, weight)] in (task, row) order; zero-cost dropped.

    weights (reading R22): the scheduler's task estimates E(t) (PAPER.md:843-846,
    "E functor if defined"); None means E(t) = the S7 cost.  cap = ceil(total E /
    (4G)); a task with E(t) > cap is cut into k = ceil(E(t)/cap) row ranges at
    row-cost quantiles, and a range's weight is floor(E(t) * its row cost / cost).
    dirs[ti] (reading R25): the task's orientation -- its rows are those of part i
    (LOW, row costs R17) or of part j (MID, row costs R25); None = all LOW."""
    E = [int(c) for c in costs] if weights is None else [int(w) for w in weights]
    total = sum(E[ti] for ti in range(len(tasks_)) if int(costs[ti]) > 0)
    cap = None if G <= 1 else max(1, -(-total // (4 * G)))
    out = []
    for ti, t in enumerate(tasks_):
        d = LOW if dirs is None else dirs[ti]
        nrows = B[(t[0], t[1])][0].size - 1 if d == LOW else B[(t[1], t[1])][0].size - 1
        cost = int(costs[ti])
        if cost == 0:
            continue
        w = E[ti]
        if cap is None or w <= cap:
            out.append((ti, 0, nrows, w))
            continue
        k = -(-w // cap)
        R = np.concatenate([[0], np.cumsum(row_costs(B, t) if d == LOW else row_costs_mid(B, t))])
        bnd = [0]
        for q in range(1, k):
            bnd.append(int(np.searchsorted(k * R, q * cost, side="left")))
        bnd.append(nrows)
        for q in range(k):
            c = int(R[bnd[q + 1]] - R[bnd[q]])
            if c > 0:
                out.append((ti, bnd[q], bnd[q + 1], w * c // cost))
    return out


def lpt(pieces_, G: int):
    """owner[k] for each piece: heaviest first (ties: task, row), least-loaded rank
    (ties: lowest rank)."""
    order = sorted(range(len(pieces_)), key=lambda k: (-pieces_[k][3], pieces_[k][0], pieces_[k][1]))
    loads = [0] * max(G, 1)
    owner = [0] * len(pieces_)
    for k in order:
        r = min(range(len(loads)), key=lambda g: (loads[g], g))
        owner[k] = r
        loads[r] += pieces_[k][3]
    return owner, loads


def piece_count(B, t, r0: int, r1: int, orient: int = LOW) -> int:
    """Count of the piece's rows: rows u of part i (LOW) or rows v of part j (MID)."""
    i, j, x = t
    c = 0
    u_all, v_all = _edges(B, i, j)
    r_all = u_all if orient == LOW else v_all
    sel = (r_all >= r0) & (r_all < r1)
    for u, v in zip(u_all[sel], v_all[sel]):
        c += np.intersect1d(row(B, i, x, u), row(B, j, x, v), assume_unique=True).size
    return int(c)


class Plan:
    """All intermediate objects of the block method for one (graph, p, rule, G)."""

    def __init__(self, n, src, dst, p, rule=0, G=1, weights=None, reverse=False, orient=1):
        self.n = int(n)
        self.E = canonical_edges(n, src, dst)
        self.deg = degrees(n, self.E)
        self.rank = degree_rank(n, self.deg, reverse)
        self.D = dag(self.E, self.rank)
        self.p = effective_p(n, p)
        self.cuts = cuts(n, self.D, self.p, rule)
        self.B = blocks(self.D, self.cuts)
        self.tasks = tasks(self.B, self.p)
        # reading R25: each task's orientation, then its cost and bytes in it
        self.dirs = [orientation(self.B, t, orient) for t in self.tasks]
        self.costs = [task_cost(self.B, t) if d == LOW else task_cost_mid(self.B, t)
                      for t, d in zip(self.tasks, self.dirs)]
        self.alg_bytes = [task_alg_bytes(self.B, t) if d == LOW else task_alg_bytes_mid(self.B, t)
                          for t, d in zip(self.tasks, self.dirs)]
        self.G = G
        self.pieces = pieces(self.B, self.tasks, self.costs, G, weights, self.dirs)
        self.owner, self.loads = lpt(self.pieces, G)

    def task_counts(self):
        return [task_count(self.B, t) for t in self.tasks]


def wedges_dag(n: int, D: np.ndarray) -> int:
    """W = sum_v d-(v) d+(v)."""
    if D.size == 0:
        return 0
    dp = np.bincount(D[:, 0], minlength=n).astype(np.int64)
    dm = np.bincount(D[:, 1], minlength=n).astype(np.int64)
    return int((dp * dm).sum())

