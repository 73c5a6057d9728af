"""B200-native block-based triangle counting (PGAbB, arXiv 2209.04541, §3.6 / §5.4).

Thin Python binding over the C ABI in ``include/pgabb.h`` (``libpgabb.so``):
argument marshalling only -- every step of the path (S1..S11)
runs in the CUDA library.  There is no CPU fallback: importing this package
without the built library raises ImportError, and calls without a CUDA device
raise :class:`PgabbError` (ECUDA).

    import paper_2209_04541_b200 as pg
    with pg.build_blocks(n, src, dst, p=8) as b:     # S1..S8
        T = b.triangle_count()                          # S9..S11
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _abi

_lib = _abi.load()

RESIDENT_DEVICE = _abi.RESIDENT_DEVICE
RESIDENT_HOST = _abi.RESIDENT_HOST


class PgabbError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = _lib.pgabb_last_error().decode(errors="replace")
        super().__init__(f"{where}: {_abi.STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = _abi.STATUS.get(status, str(status))


def _ck(st: int, where: str):
    if st != 0:
        raise PgabbError(st, where)


def version() -> str:
    return _lib.pgabb_version().decode()


_CUDA_STREAM_LEGACY = 1   # cudaStreamLegacy: the ABI reads NULL as "the handle's own stream"


def _stream_arg(stream):
    """cudaStream_t for CountOpts.cuda_stream from a torch stream or a raw handle.
    torch's default stream reports cuda_stream == 0 (the legacy default stream);
    passed through as NULL the library would use its private non-blocking stream,
    unordered with torch's work, so 0 becomes cudaStreamLegacy."""
    raw = int(getattr(stream, "cuda_stream", stream) or 0)
    return raw if raw else _CUDA_STREAM_LEGACY


def _pointer(x):
    """(pointer, length, on_device, keepalive) for a numpy array or torch tensor of uint32/int32."""
    if hasattr(x, "data_ptr") and hasattr(x, "is_cuda"):
        import torch
        if x.dtype not in (torch.int32, torch.uint32):
            raise TypeError("tuples must be 32-bit integers")
        x = x.contiguous()
        if x.is_cuda:
            return x.data_ptr(), x.numel(), True, x
        x = x.numpy()
    a = np.ascontiguousarray(x)
    if a.dtype not in (np.uint32, np.int32):
        if a.dtype.kind not in "iu":
            raise TypeError(f"tuples must be integers, got {a.dtype}")
        # a wider integer array is narrowed only when every id fits in uint32 (ids of
        # 2^32 or more would otherwise wrap to small ids and count another graph)
        if a.size and (int(a.min()) < 0 or int(a.max()) >= (1 << 32)):
            raise ValueError("vertex ids must lie in [0, 2^32)")
        a = a.astype(np.uint32)
    return a.ctypes.data, a.size, False, a


class Blocks:
    """A built block grid (handle).  Use as a context manager or call free()."""

    def __init__(self, handle, ntasks: int, p: int, n: int):
        self._h = handle
        self.ntasks = ntasks
        self.p = p
        self.n = n

    # --- lifetime ---
    def free(self):
        if self._h:
            _lib.pgabb_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.free()

    # --- S9..S11 ---
    def triangle_count(self, stream=None, d_count=None, task_counts: bool = False, sync: bool = True,
                       trace: bool = False):
        """This rank's triangle count (host int).  stream: a cudaStream_t int or torch
        stream; d_count: device pointer (int) receiving the count; task_counts: also
        return the per-task counts; trace: record the streaming waves' timeline
        (read with wave_trace())."""
        o = _abi.CountOpts()
        if stream is not None:
            o.cuda_stream = _stream_arg(stream)
        if d_count is not None:
            o.d_count = d_count
        tc = np.zeros(max(self.ntasks, 1), np.uint64) if task_counts else None
        if tc is not None:
            o.task_counts = tc.ctypes.data_as(_abi.u64p)
        if not sync:
            o.flags = _abi.COUNT_ASYNC
        if trace:
            o.flags |= _abi.COUNT_TRACE
        out = ctypes.c_uint64(0)
        _ck(_lib.pgabb_triangle_count(self._h, ctypes.byref(o), ctypes.byref(out)), "pgabb_triangle_count")
        if not sync:
            return None
        return (int(out.value), tc[:self.ntasks]) if task_counts else int(out.value)

    def wave_trace(self):
        """Per-wave timeline of the last traced streaming count: float64[waves, 4] =
        (copy start, copy end, compute start, compute end), ms from the call start."""
        nw = ctypes.c_uint64(0)
        _ck(_lib.pgabb_get_wave_trace(self._h, None, ctypes.byref(nw)), "pgabb_get_wave_trace")
        out = np.zeros(max(4 * nw.value, 1), np.float64)
        _ck(_lib.pgabb_get_wave_trace(self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                      ctypes.byref(nw)), "pgabb_get_wave_trace")
        return out[:4 * nw.value].reshape(-1, 4)

    # --- per-vertex counts ---
    def vertex_triangles(self, stream=None, out=None, sync: bool = True, roles: str = "all",
                         accumulate: bool = False):
        """This rank's t(v) for every original id v (numpy uint64[n]), or, with
        ``out`` a CUDA int64/uint64 tensor of n entries, written into it on the
        device (stream-ordered; ready for an NCCL allreduce).  Returns (tv, T_rank).
        roles: "all", "low" or "low+mid" -- which vertices of each triangle
        {u<v<w} (rank order) are credited (DESIGN R24)."""
        o = _abi.CountOpts()
        o.flags = {"all": 0, "low": _abi.ROLE_LOW, "low+mid": _abi.ROLE_LOW | _abi.ROLE_MID}[roles]
        if stream is not None:
            o.cuda_stream = _stream_arg(stream)
        cnt = ctypes.c_uint64(0)
        if out is not None:
            if not getattr(out, "is_cuda", False) or out.numel() < self.n or out.element_size() != 8:
                raise ValueError("out must be a CUDA 8-byte tensor with >= n entries")
            o.flags |= _abi.OUT_DEVICE | (0 if sync else _abi.COUNT_ASYNC) | (_abi.OUT_ACCUMULATE if accumulate else 0)
            _ck(_lib.pgabb_vertex_triangles(self._h, ctypes.byref(o), out.data_ptr(), ctypes.byref(cnt)),
                "pgabb_vertex_triangles")
            return out, (int(cnt.value) if sync else None)
        tv = np.zeros(max(self.n, 1), np.uint64)
        _ck(_lib.pgabb_vertex_triangles(self._h, ctypes.byref(o), tv.ctypes.data, ctypes.byref(cnt)),
            "pgabb_vertex_triangles")
        return tv[:self.n], int(cnt.value)

    def local_clustering(self, tv, stream=None):
        """cc(v) = 2 t(v) / (deg(v)(deg(v)-1)) from the COMPLETE t(v): numpy in ->
        numpy float64 out, or a CUDA 8-byte tensor in -> CUDA float64 tensor out."""
        o = _abi.CountOpts()
        if stream is not None:
            o.cuda_stream = _stream_arg(stream)
        if getattr(tv, "is_cuda", False):
            import torch
            if tv.numel() < self.n or tv.element_size() != 8:
                raise ValueError("tv must hold n 8-byte counts")
            tv = tv.contiguous()
            cc = torch.empty(max(self.n, 1), dtype=torch.float64, device=tv.device)
            o.flags = _abi.OUT_DEVICE
            _ck(_lib.pgabb_local_clustering(self._h, ctypes.byref(o), tv.data_ptr(), cc.data_ptr()),
                "pgabb_local_clustering")
            return cc[:self.n]
        t = np.ascontiguousarray(tv, dtype=np.uint64)
        if t.size < self.n:
            raise ValueError("tv must hold n counts")
        cc = np.zeros(max(self.n, 1), np.float64)
        _ck(_lib.pgabb_local_clustering(self._h, ctypes.byref(o), t.ctypes.data, cc.ctypes.data),
            "pgabb_local_clustering")
        return cc[:self.n]

    def connected_components(self, stream=None, out=None):
        """Shiloach-Vishkin components (NEXT-4): (labels, ncomponents, iterations);
        labels[v] = smallest original id of v's component (numpy uint32[n], or
        written into ``out``, a CUDA 4-byte tensor of n entries)."""
        o = _abi.CountOpts()
        if stream is not None:
            o.cuda_stream = _stream_arg(stream)
        nc, it = ctypes.c_uint64(0), ctypes.c_uint32(0)
        if out is not None:
            if not getattr(out, "is_cuda", False) or out.numel() < self.n or out.element_size() != 4:
                raise ValueError("out must be a CUDA 4-byte tensor with >= n entries")
            o.flags = _abi.OUT_DEVICE
            _ck(_lib.pgabb_connected_components(self._h, ctypes.byref(o), out.data_ptr(), ctypes.byref(nc),
                                                ctypes.byref(it)), "pgabb_connected_components")
            return out[:self.n], int(nc.value), int(it.value)
        lab = np.zeros(max(self.n, 1), np.uint32)
        _ck(_lib.pgabb_connected_components(self._h, ctypes.byref(o), lab.ctypes.data, ctypes.byref(nc),
                                            ctypes.byref(it)), "pgabb_connected_components")
        return lab[:self.n], int(nc.value), int(it.value)

    def task_times(self) -> np.ndarray:
        """Measured device time per task (ns, uint64[ntasks]) of this handle's pieces:
        the scheduler's E(t) for a balanced multi-GPU plan (pgabb_task_times)."""
        out = np.zeros(max(self.ntasks, 1), np.uint64)
        _ck(_lib.pgabb_task_times(self._h, out.ctypes.data_as(_abi.u64p)), "pgabb_task_times")
        return out[:self.ntasks]

    # --- introspection ---
    def stats(self) -> dict:
        s = _abi.Stats()
        _ck(_lib.pgabb_get_stats(self._h, ctypes.byref(s)), "pgabb_get_stats")
        return s.as_dict()

    def rank(self) -> np.ndarray:
        out = np.empty(max(self.n, 1), np.uint32)
        _ck(_lib.pgabb_get_rank(self._h, out.ctypes.data_as(_abi.u32p)), "pgabb_get_rank")
        return out[:self.n]

    def cuts(self) -> np.ndarray:
        out = np.empty(self.p + 1, np.uint32)
        _ck(_lib.pgabb_get_cuts(self._h, out.ctypes.data_as(_abi.u32p)), "pgabb_get_cuts")
        return out

    def block(self, i: int, j: int):
        """(rowptr, col) of A_ij, local ids."""
        nnz = ctypes.c_uint64(0)
        _ck(_lib.pgabb_get_block(self._h, i, j, None, None, ctypes.byref(nnz)), "pgabb_get_block")
        c = self.cuts()
        rp = np.empty(int(c[i + 1] - c[i]) + 1, np.uint32)
        col = np.empty(max(int(nnz.value), 1), np.uint32)
        _ck(_lib.pgabb_get_block(self._h, i, j, rp.ctypes.data_as(_abi.u32p), col.ctypes.data_as(_abi.u32p),
                                 ctypes.byref(nnz)), "pgabb_get_block")
        return rp, col[:int(nnz.value)]

    def tasks(self):
        """(ijx[ntasks,3], cost[ntasks], alg_bytes[ntasks])."""
        nt = max(self.ntasks, 1)
        ijx = np.empty(3 * nt, np.uint32)
        cost = np.empty(nt, np.uint64)
        alg = np.empty(nt, np.uint64)
        _ck(_lib.pgabb_get_tasks(self._h, ijx.ctypes.data_as(_abi.u32p), cost.ctypes.data_as(_abi.u64p),
                                 alg.ctypes.data_as(_abi.u64p)), "pgabb_get_tasks")
        k = self.ntasks
        return ijx[:3 * k].reshape(k, 3), cost[:k], alg[:k]

    def task_orient(self):
        """(dir[ntasks] 0 LOW / 1 MID, s_low[ntasks], s_mid[ntasks]) -- DESIGN R25."""
        nt = max(self.ntasks, 1)
        d = np.empty(nt, np.uint32)
        sl = np.empty(nt, np.uint64)
        sm = np.empty(nt, np.uint64)
        _ck(_lib.pgabb_get_task_orient(self._h, d.ctypes.data_as(_abi.u32p), sl.ctypes.data_as(_abi.u64p),
                                       sm.ctypes.data_as(_abi.u64p)), "pgabb_get_task_orient")
        k = self.ntasks
        return d[:k], sl[:k], sm[:k]

    def pieces(self):
        """list of (task, row_begin, row_end, cost) and owner list (rows of part i for
        a LOW task, of part j for a MID task)."""
        npc = int(self.stats()["npieces"])
        m = max(npc, 1)
        t, r0, r1 = (np.empty(m, np.uint32) for _ in range(3))
        c = np.empty(m, np.uint64)
        o = np.empty(m, np.int32)
        _ck(_lib.pgabb_get_pieces(self._h, t.ctypes.data_as(_abi.u32p), r0.ctypes.data_as(_abi.u32p),
                                  r1.ctypes.data_as(_abi.u32p), c.ctypes.data_as(_abi.u64p),
                                  o.ctypes.data_as(_abi.i32p)), "pgabb_get_pieces")
        pcs = [(int(t[k]), int(r0[k]), int(r1[k]), int(c[k])) for k in range(npc)]
        return pcs, [int(o[k]) for k in range(npc)]


ORIENTS = {"auto": 0, "low": 1, "mid": 2}


def build_blocks(n: int, src, dst, p: int = 0, cut_rule: int = 0, device: int = -1, rank: int = 0,
                 world_size: int = 1, residency: int = RESIDENT_DEVICE, device_budget_bytes: int = 0,
                 task_weights=None, reverse_order: bool = False, orient="auto", host_permille: int = 0,
                 host_threads: int = 0, light_held: int = 0) -> Blocks:
    """S1..S8: canonicalise, degree-order, orient, cut, block, enumerate, cost, assign.

    orient: task orientation (DESIGN R25) -- "auto" (per task, fewer streamed ids),
    "low" (hold A_ix[u], stream A_jx[v]; no transposes) or "mid" (hold A_jx[v],
    stream the ids w > v of A_ix[u]); also 0 / 1 / 2.
    host_permille / host_threads: collaborative CPU + GPU (NEXT-3) on a host-resident
    handle -- the sparsest pieces up to this share of the cost are counted by host
    threads while the GPU counts the rest.
    light_held: largest held list of a thread-per-row item -- 8, 15 (rows with 9..15
    held ids get the second thread-per-row kernel) or 0 = auto (DESIGN R29).

    src/dst: uint32 tuples as numpy arrays (host) or torch CUDA tensors (device).
    task_weights: optional per-task estimates E(t) (e.g. Blocks.task_times() of a
    1-rank handle, identical on every rank) used by S8 instead of the S7 cost."""
    sp, sn, sdev, keep_s = _pointer(src)
    dp, dn, ddev, keep_d = _pointer(dst)
    if sn != dn:
        raise ValueError("src and dst differ in length")
    if sdev != ddev:
        raise ValueError("src and dst must both be host or both be device arrays")
    o = _abi.BuildOpts()
    _lib.pgabb_default_build_opts(ctypes.byref(o))
    o.p, o.cut_rule, o.device = p, cut_rule, device
    o.inputs_on_device = int(sdev)
    o.rank, o.world_size, o.residency = rank, world_size, residency
    o.reverse_order = int(bool(reverse_order))
    o.orient = ORIENTS[orient] if isinstance(orient, str) else int(orient)
    o.host_permille, o.host_threads = int(host_permille), int(host_threads)
    o.light_held = int(light_held)
    o.device_budget_bytes = device_budget_bytes
    tw = None
    if task_weights is not None:
        tw = np.ascontiguousarray(task_weights, dtype=np.uint64)
        o.task_weights = tw.ctypes.data_as(_abi.u64p)
        o.n_task_weights = tw.size
    h = ctypes.c_void_p(0)
    st = _lib.pgabb_build_blocks(int(n), int(sn), ctypes.c_void_p(sp) if sn else None,
                                 ctypes.c_void_p(dp) if dn else None, ctypes.byref(o), ctypes.byref(h))
    del keep_s, keep_d, tw
    _ck(st, "pgabb_build_blocks")
    s = _abi.Stats()
    _ck(_lib.pgabb_get_stats(h, ctypes.byref(s)), "pgabb_get_stats")
    return Blocks(h, int(s.ntasks), int(s.p), int(n))


def vertex_triangles_two_pass(n: int, src, dst, p: int = 0, **kw):
    """t(v) for every original id by two cheap passes (DESIGN R24): the lowest and
    middle vertex of every triangle from the forward handle (row totals and pair
    counts: no per-hit atomics), the highest vertex as the LOWEST of the handle
    built on the reversed degree order.  Returns (tv, T)."""
    import torch
    dev = kw.get("device", -1)
    out = torch.zeros(max(n, 1), dtype=torch.int64,
                      device=torch.device("cuda", dev) if dev is not None and dev >= 0 else "cuda")
    with build_blocks(n, src, dst, p=p, **kw) as f:
        _, T = f.vertex_triangles(out=out, roles="low+mid")
    with build_blocks(n, src, dst, p=p, reverse_order=True, **kw) as r:
        # the second pass adds into the first on the device (PGABB_OUT_ACCUMULATE)
        _, T2 = r.vertex_triangles(out=out, roles="low", accumulate=True)
    if T2 != T:
        raise RuntimeError(f"forward and reversed counts differ: {T} != {T2}")
    return out[:n].cpu().numpy().astype(np.uint64), T


def triangle_count(n: int, src, dst, **kw) -> int:
    """One-shot convenience: build, count, free."""
    with build_blocks(n, src, dst, **kw) as b:
        return b.triangle_count()
