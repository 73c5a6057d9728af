"""Seeded synthetic graph generators shared by oracle/, tests/ and bench.py.

This module holds none of the triangle-counting method's arithmetic: every
function returns ``(n, src, dst)`` -- the vertex count and two uint32 numpy
arrays of edge tuples, which may contain duplicates, both directions and
self-loops (the method canonicalises them; §5.1).

Large families (R-MAT, ER, grid) are counter-based C generators in ``gen.c``
(bit-identical for any thread count).  Small closed-form families are plain
numpy.  The recipe of every family is stated in DESIGN.md "Input recipe".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libpgabb_gen.so")
_SRC = os.path.join(_HERE, "gen.c")
_lib = None


def build(force: bool = False) -> str:
    """Compile gen.c into libpgabb_gen.so (gcc, OpenMP)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", _SRC, "-o", tmp])
        os.replace(tmp, _SO)
    return _SO


def _L():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        u64, u32p = ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint32)
        lib.pgabb_gen_rmat.argtypes = [ctypes.c_int, u64, ctypes.c_int, u64, u64, u32p, u32p]
        lib.pgabb_gen_rmat.restype = None
        lib.pgabb_gen_er.argtypes = [u64, u64, u64, u64, u32p, u32p]
        lib.pgabb_gen_er.restype = None
        lib.pgabb_gen_grid_ndiag.argtypes = [u64, ctypes.c_double, u64]
        lib.pgabb_gen_grid_ndiag.restype = u64
        lib.pgabb_gen_grid.argtypes = [u64, ctypes.c_double, u64, u32p, u32p]
        lib.pgabb_gen_grid.restype = None
        lib.pgabb_gen_permute.argtypes = [u64, ctypes.c_int, u64]
        lib.pgabb_gen_permute.restype = u64
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def rmat(scale: int, edge_factor: int, seed: int = 1, permute: bool = True):
    """Graph500 R-MAT (a,b,c,d = .57,.19,.19,.05), edge_factor * 2^scale tuples."""
    n = 1 << scale
    m = edge_factor * n
    src = np.empty(m, np.uint32)
    dst = np.empty(m, np.uint32)
    _L().pgabb_gen_rmat(scale, seed, int(permute), 0, m, _p(src), _p(dst))
    return n, src, dst


def er(n: int, avg_degree: float, seed: int = 1):
    """Erdos-Renyi G(n, m) with replacement, m = n * avg_degree / 2 tuples."""
    m = int(n * avg_degree // 2)
    src = np.empty(m, np.uint32)
    dst = np.empty(m, np.uint32)
    _L().pgabb_gen_er(n, seed, 0, m, _p(src), _p(dst))
    return n, src, dst


def grid_ndiag(side: int, f: float, seed: int = 1) -> int:
    """Number of diagonal cells the grid generator emits for (side, f, seed)."""
    return int(_L().pgabb_gen_grid_ndiag(side, float(f), seed))


def grid(side: int, f: float = 0.0, seed: int = 1):
    """side x side 4-neighbour lattice + diagonals in a seeded fraction f of cells."""
    k = grid_ndiag(side, f, seed)
    m = 2 * side * (side - 1) + k
    src = np.empty(m, np.uint32)
    dst = np.empty(m, np.uint32)
    _L().pgabb_gen_grid(side, float(f), seed, _p(src), _p(dst))
    return side * side, src, dst


def permute_id(x: int, bits: int, seed: int) -> int:
    return int(_L().pgabb_gen_permute(x, bits, seed))


# ---------------------------------------------------------------------------
# Small closed-form families (numpy).  Closed-form triangle counts live in the
# tests, next to the citation of each formula; nothing here computes them.
# ---------------------------------------------------------------------------

def _pack(n, pairs):
    a = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    return n, a[:, 0].astype(np.uint32), a[:, 1].astype(np.uint32)


def complete(n: int):
    iu, ju = np.triu_indices(n, 1)
    return _pack(n, np.stack([iu, ju], 1))


def cycle(n: int):
    i = np.arange(n)
    return _pack(n, np.stack([i, (i + 1) % n], 1))


def path(n: int):
    i = np.arange(n - 1)
    return _pack(n, np.stack([i, i + 1], 1))


def star(n: int):
    """Hub 0 plus n-1 leaves (n vertices)."""
    i = np.arange(1, n)
    return _pack(n, np.stack([np.zeros_like(i), i], 1))


def wheel(n: int):
    """W_n: hub 0 + (n-1)-cycle on 1..n-1 (n vertices; networkx wheel_graph(n))."""
    r = np.arange(1, n)
    rim = np.stack([r, np.where(r == n - 1, 1, r + 1)], 1)
    spokes = np.stack([np.zeros_like(r), r], 1)
    return _pack(n, np.concatenate([spokes, rim]))


def windmill(k: int, m: int):
    """k copies of K_m sharing vertex 0."""
    pairs = []
    for c in range(k):
        verts = [0] + [1 + c * (m - 1) + t for t in range(m - 1)]
        for a in range(m):
            for b in range(a + 1, m):
                pairs.append((verts[a], verts[b]))
    return _pack(1 + k * (m - 1), pairs)


def clique_union(sizes):
    """Disjoint union of cliques K_{s_0}, K_{s_1}, ... (contiguous ids)."""
    pairs, off = [], 0
    for s in sizes:
        iu, ju = np.triu_indices(s, 1)
        pairs.append(np.stack([iu + off, ju + off], 1))
        off += s
    allp = np.concatenate(pairs) if pairs else np.zeros((0, 2), np.int64)
    return _pack(off, allp)


def rook(a: int, b: int):
    """Rook graph K_a x K_b (Cartesian product): vertex (r, c) -> r*b + c."""
    pairs = []
    for r in range(a):
        for c1 in range(b):
            for c2 in range(c1 + 1, b):
                pairs.append((r * b + c1, r * b + c2))
    for c in range(b):
        for r1 in range(a):
            for r2 in range(r1 + 1, a):
                pairs.append((r1 * b + c, r2 * b + c))
    return _pack(a * b, pairs)


def king(r: int, c: int):
    """King graph on an r x c board: both diagonals in every cell."""
    pairs = []
    vid = lambda i, j: i * c + j
    for i in range(r):
        for j in range(c):
            if j + 1 < c:
                pairs.append((vid(i, j), vid(i, j + 1)))
            if i + 1 < r:
                pairs.append((vid(i, j), vid(i + 1, j)))
            if i + 1 < r and j + 1 < c:
                pairs.append((vid(i, j), vid(i + 1, j + 1)))
                pairs.append((vid(i, j + 1), vid(i + 1, j)))
    return _pack(r * c, pairs)


def complete_bipartite(a: int, b: int):
    i, j = np.meshgrid(np.arange(a), np.arange(a, a + b), indexing="ij")
    return _pack(a + b, np.stack([i.ravel(), j.ravel()], 1))


def random_tree(n: int, seed: int = 1):
    """Uniform random recursive tree: vertex i>0 attaches to a parent < i."""
    rng = np.random.default_rng(seed)
    i = np.arange(1, n)
    par = (rng.random(n - 1) * i).astype(np.int64)
    return _pack(n, np.stack([par, i], 1))


def er_small(n: int, p: float, seed: int = 1):
    """G(n, p) on n vertices (numpy), for brute-force-sized tests."""
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, 1)
    keep = rng.random(iu.size) < p
    return _pack(n, np.stack([iu[keep], ju[keep]], 1))


def disjoint_union(*graphs):
    """Disjoint union of (n, src, dst) graphs, ids offset in order."""
    off, ss, dd = 0, [], []
    for n, s, d in graphs:
        ss.append(s.astype(np.int64) + off)
        dd.append(d.astype(np.int64) + off)
        off += n
    return off, np.concatenate(ss).astype(np.uint32), np.concatenate(dd).astype(np.uint32)


def messy(graph, seed: int = 1, dup: float = 0.3, loops: int = 3):
    """Same simple graph, noisier tuples: shuffled, random reversals, duplicates
    and self-loops (the method canonicalises them away; SURVEY §8(c) readings 1-2)."""
    n, s, d = graph
    rng = np.random.default_rng(seed)
    s = s.astype(np.int64)
    d = d.astype(np.int64)
    flip = rng.random(s.size) < 0.5
    s2, d2 = np.where(flip, d, s), np.where(flip, s, d)
    nd = int(dup * s.size)
    pick = rng.integers(0, max(s.size, 1), nd) if s.size else np.zeros(0, np.int64)
    s3 = np.concatenate([s2, d[pick], rng.integers(0, max(n, 1), loops if n else 0)])
    d3 = np.concatenate([d2, s[pick], np.zeros(0, np.int64)])
    d3 = np.concatenate([d3, s3[s3.size - (loops if n else 0):]])
    perm = rng.permutation(s3.size)
    return n, s3[perm].astype(np.uint32), d3[perm].astype(np.uint32)


def relabel(graph, seed: int = 1):
    """Apply a random vertex permutation (T is invariant under it)."""
    n, s, d = graph
    perm = np.random.default_rng(seed).permutation(n).astype(np.uint32)
    return n, perm[s], perm[d]
