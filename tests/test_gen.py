"""The seeded generators: determinism, shapes and structure."""
import numpy as np

import gen


def test_rmat_deterministic_and_in_range():
    n, s, d = gen.rmat(12, 16, seed=1)
    n2, s2, d2 = gen.rmat(12, 16, seed=1)
    assert n == 4096 and s.size == 16 * 4096
    assert (s == s2).all() and (d == d2).all()
    assert s.max() < n and d.max() < n
    n3, s3, _ = gen.rmat(12, 16, seed=2)
    assert not (s3 == s).all()


def test_rmat_skew_matches_graph500_initiator():
    # quadrant a=.57 dominates: the unpermuted top bit of u is 0 with prob a+b = .76
    n, s, d = gen.rmat(14, 16, seed=3, permute=False)
    frac_u0 = np.mean((s >> 13) == 0)
    frac_v0 = np.mean((d >> 13) == 0)
    assert abs(frac_u0 - 0.76) < 0.01 and abs(frac_v0 - 0.76) < 0.01


def test_permutation_is_bijection():
    for bits in (1, 5, 10, 13):
        img = {gen.permute_id(x, bits, 7) for x in range(1 << bits)}
        assert img == set(range(1 << bits))


def test_er_uniform():
    n, s, d = gen.er(1 << 16, 32, seed=1)
    assert s.size == 16 * (1 << 16)
    assert s.max() < n and d.max() < n
    h = np.bincount(s >> 12, minlength=16)
    assert h.min() > 0.9 * h.mean()


def test_grid_shape_and_diagonals():
    side, f = 64, 0.25
    n, s, d = gen.grid(side, f, seed=5)
    k = gen.grid_ndiag(side, f, seed=5)
    assert n == side * side
    assert s.size == 2 * side * (side - 1) + k
    diag = (d.astype(np.int64) - s.astype(np.int64)) == side + 1
    assert int(diag.sum()) == k
    assert abs(k / (side - 1) ** 2 - f) < 0.05
    assert gen.grid_ndiag(side, 0.0) == 0
    assert gen.grid_ndiag(side, 1.0) == (side - 1) ** 2


def test_messy_keeps_simple_graph():
    g = gen.complete(6)
    n, s, d = gen.messy(g, seed=3)
    pairs = {frozenset((int(a), int(b))) for a, b in zip(s, d) if a != b}
    ref = {frozenset((int(a), int(b))) for a, b in zip(g[1], g[2])}
    assert pairs == ref
    assert (s == d).sum() >= 1
