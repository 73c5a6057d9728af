"""TEST INFRASTRUCTURE ONLY -- the plain CPU oracle for block-based triangle counting.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA path in ``paper_2209_04541_b200/`` and neither imports the other.

* ``tc_oracle.c`` (via :class:`Graph`, :func:`brute`): the node iterator with
  marks over the degree order and the O(n^3) brute-force definition
  (§3.6; §5.4).
* ``blocks.py``: the block method's intermediate objects, each written out as
  its plain definition (degree order, DAG, conformal cuts, block CSR, block
  triples, per-task counts and costs, LPT assignment) for small graphs.

Every function is pinned by ``tests/test_oracle*.py`` against brute force,
closed forms, library routines (scipy, networkx) or invariants.  Functions
without such a pin are marked "parity unpinned" in their docstring and in
DESIGN.md (currently: none).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "tc_oracle.c")
_lib = None


def build(force: bool = False) -> str:
    """Compile tc_oracle.c (gcc -O2 -fopenmp).  Building the checker is not using it."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", _SRC, "-o", tmp])
        os.replace(tmp, _SO)
    return _SO


def _L():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        vp, u32, u64 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64
        u32p = ctypes.POINTER(ctypes.c_uint32)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        lib.oracle_build.argtypes = [u32, u64, u32p, u32p]
        lib.oracle_build.restype = vp
        lib.oracle_free.argtypes = [vp]
        lib.oracle_free.restype = None
        lib.oracle_num_edges.argtypes = [vp]
        lib.oracle_num_edges.restype = u64
        lib.oracle_degrees.argtypes = [vp, u32p]
        lib.oracle_degrees.restype = None
        lib.oracle_count_range.argtypes = [vp, u32, u32, u32, u64p, u64p]
        lib.oracle_count_range.restype = u64
        lib.oracle_wedges.argtypes = [vp]
        lib.oracle_wedges.restype = u64
        lib.oracle_brute.argtypes = [u32, u64, u32p, u32p]
        lib.oracle_brute.restype = u64
        lib.oracle_threads.argtypes = []
        lib.oracle_threads.restype = ctypes.c_int
        lib.oracle_count_roles.argtypes = [vp, u64p, u64p, u64p]
        lib.oracle_count_roles.restype = u64
        lib.oracle_components.argtypes = [vp, u32p]
        lib.oracle_components.restype = u64
        lib.oracle_set_threads.argtypes = [ctypes.c_int]
        lib.oracle_set_threads.restype = None
        _lib = lib
    return _lib


def _u32(a):
    a = np.ascontiguousarray(a, dtype=np.uint32)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def threads() -> int:
    return int(_L().oracle_threads())


def set_threads(k: int) -> None:
    """OpenMP threads of the oracle's parallel loops (all host cores by default)."""
    _L().oracle_set_threads(int(k))


class Graph:
    """G_s built from tuples by the oracle's own canonicalisation (tc_oracle.c)."""

    def __init__(self, n: int, src, dst):
        s, sp = _u32(src)
        d, dp = _u32(dst)
        if s.size != d.size:
            raise ValueError("src/dst length mismatch")
        self.n = int(n)
        self._h = _L().oracle_build(self.n, s.size, sp, dp)
        if not self._h:
            raise ValueError("oracle_build failed (vertex id >= n or out of memory)")

    def close(self):
        if getattr(self, "_h", None):
            _L().oracle_free(self._h)
            self._h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def m_edges(self) -> int:
        """|E| of G_s: unique undirected non-loop edges (SURVEY §8(c) reading 15)."""
        return int(_L().oracle_num_edges(self._h))

    def degrees(self) -> np.ndarray:
        out = np.empty(self.n, np.uint32)
        _L().oracle_degrees(self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)))
        return out

    def count(self, per_vertex: bool = False):
        """T (and t(v) if per_vertex) by the node iterator."""
        tv = np.zeros(self.n, np.uint64) if per_vertex else None
        tvp = tv.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)) if per_vertex else None
        T = int(_L().oracle_count_range(self._h, 0, self.n, 1, tvp, None))
        if T == (1 << 64) - 1:
            raise MemoryError("oracle mark arrays")
        return (T, tv) if per_vertex else T

    def count_range(self, v0: int, v1: int, stride: int = 1):
        """(triangles whose lowest vertex is in range(v0, v1, stride), DAG edges owned)."""
        e = ctypes.c_uint64(0)
        T = int(_L().oracle_count_range(self._h, v0, v1, stride, None, ctypes.byref(e)))
        return T, int(e.value)

    def count_roles(self):
        """(T, tlow, tmid, thigh): per-vertex counts of the triangles in which the
        vertex is the lowest / middle / highest in the (deg, id) order (R24)."""
        arrs = [np.zeros(max(self.n, 1), np.uint64) for _ in range(3)]
        ptr = [a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)) for a in arrs]
        T = int(_L().oracle_count_roles(self._h, *ptr))
        if T == (1 << 64) - 1:
            raise MemoryError("oracle mark array")
        return (T, *[a[:self.n] for a in arrs])

    def components(self):
        """(labels, ncomponents): labels[v] = smallest id of v's component in G_s."""
        lab = np.zeros(max(self.n, 1), np.uint32)
        nc = int(_L().oracle_components(self._h, lab.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))))
        if nc == (1 << 64) - 1:
            raise MemoryError("oracle union-find array")
        return lab[:self.n], nc

    def wedges(self) -> int:
        """W = sum_v d-(v) d+(v) over the degree-ordered DAG."""
        return int(_L().oracle_wedges(self._h))


def count(n, src, dst, per_vertex: bool = False):
    with Graph(n, src, dst) as g:
        return g.count(per_vertex)


def count_roles(n, src, dst):
    """(T, tlow, tmid, thigh) by role in the degree order (DESIGN R24)."""
    with Graph(n, src, dst) as g:
        return g.count_roles()


def components(n, src, dst):
    """Connected components (NEXT-4): (labels, ncomponents), labels[v] = smallest id
    in v's component (union-find, tc_oracle.c)."""
    with Graph(n, src, dst) as g:
        return g.components()


def clustering(n, src, dst):
    """Local clustering coefficient of every vertex of G_s (the measure the paper
    motivates triangle counting with, §1), by its definition:
    cc(v) = t(v) / C(deg(v), 2) = 2 t(v) / (deg(v) (deg(v) - 1)), and 0 when
    deg(v) < 2.  t(v) from the node iterator, deg from the oracle's own
    canonicalisation; one fp64 division of exact integers per vertex.
    Pinned by tests/test_oracle.py against networkx.clustering and closed forms."""
    with Graph(n, src, dst) as g:
        _, tv = g.count(per_vertex=True)
        deg = g.degrees().astype(np.uint64)
    cc = np.zeros(int(n), np.float64)
    m = deg >= 2
    cc[m] = (2.0 * tv[m].astype(np.float64)) / (deg[m] * (deg[m] - np.uint64(1))).astype(np.float64)
    return tv, cc


def brute(n, src, dst) -> int:
    """O(n^3) brute force over a dense adjacency (n <= 4096)."""
    s, sp = _u32(src)
    d, dp = _u32(dst)
    if n > 4096:
        raise ValueError("brute force is for n <= 4096")
    T = int(_L().oracle_brute(int(n), s.size, sp, dp))
    if T == (1 << 64) - 1:
        raise ValueError("bad input")
    return T
