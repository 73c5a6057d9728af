"""Multi-GPU driver: one process per GPU (torchrun), tasks split by LPT (S8) and
the per-rank uint64 counts combined with ONE NCCL allreduce of 8 bytes (S11).

torch.distributed is plumbing here: it provides the process group and the
NCCL allreduce of the per-rank count, which the library writes straight into
a device int64 tensor on the same stream (no host round trip before the
collective).  Counts are < 2^63, so int64 is exact.
"""
from __future__ import annotations

from . import Blocks, build_blocks


def build_blocks_for_rank(n, src, dst, p=0, cut_rule=0, residency=0, device_budget_bytes=0, group=None,
                          orient="auto"):
    """This rank's handle: every rank builds the same grid from the same tuples
    (S1-S8 are deterministic) and keeps the LPT share of pieces it owns."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    ws = dist.get_world_size(group) if dist.is_initialized() else 1
    dev = torch.cuda.current_device() if torch.cuda.is_available() else -1
    return build_blocks(n, src, dst, p=p, cut_rule=cut_rule, device=dev, rank=rank, world_size=ws,
                        residency=residency, device_budget_bytes=device_budget_bytes, orient=orient)


def triangle_count_allreduce(b: Blocks, out=None, group=None) -> int:
    """This rank's count -> device int64 -> NCCL allreduce(sum) -> host int."""
    import torch
    import torch.distributed as dist
    stream = torch.cuda.current_stream()
    if out is None:
        out = torch.zeros(1, dtype=torch.int64, device="cuda")
    b.triangle_count(stream=stream.cuda_stream, d_count=out.data_ptr(), sync=False)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return int(out.item())


def combine_counts_host(local: int, group=None) -> int:
    """Allreduce of host-side partial counts (CPU/gloo path used by the tests)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([local], dtype=torch.int64)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item())


def vertex_triangles_allreduce(b: Blocks, out=None, group=None):
    """t(v) for every original id: this rank's share written on the device, then
    ONE NCCL allreduce(sum) of the n-entry int64 vector (the exchange step of the
    per-vertex path; t(v) < 2^63).  Returns the device tensor."""
    import torch
    import torch.distributed as dist
    if out is None:
        out = torch.empty(max(b.n, 1), dtype=torch.int64, device="cuda")
    b.vertex_triangles(stream=torch.cuda.current_stream(), out=out, sync=False)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return out[:b.n]


def combine_vertex_counts_host(local, group=None):
    """Allreduce of host-side per-vertex partials (CPU/gloo path used by the tests)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(np.ascontiguousarray(local, dtype=np.int64))
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.numpy().astype(np.uint64)


def build_blocks_balanced(n, src, dst, p=0, cut_rule=0, group=None, **kw):
    """S8 with measured task estimates (DESIGN R22): rank 0 alone builds a 1-rank
    handle and times every task on it (pgabb_task_times), broadcasts the per-task
    nanoseconds, and every rank plans its LPT share with them -- the same plan
    everywhere, balanced by device time instead of the S7 merge cost.  Untimed
    pre-processing.  The returned handle carries the weights as
    ``task_weights_used`` (another handle of the same plan, e.g. host-resident,
    is built with them)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    ws = dist.get_world_size(group) if dist.is_initialized() else 1
    dev = torch.cuda.current_device() if torch.cuda.is_available() else -1
    if ws <= 1:
        return build_blocks(n, src, dst, p=p, cut_rule=cut_rule, device=dev, **kw)
    ns = None
    if rank == 0:
        with build_blocks(n, src, dst, p=p, cut_rule=cut_rule, device=dev, orient=kw.get("orient", "auto")) as b1:
            ns = b1.task_times()
    w = broadcast_weights(ns, group)
    b = build_blocks(n, src, dst, p=p, cut_rule=cut_rule, device=dev, rank=rank, world_size=ws,
                     task_weights=w, **kw)
    b.task_weights_used = w
    return b


def broadcast_weights(ns, group=None):
    """Rank 0's per-task estimates to every rank (int64 over the group's backend).
    Only rank 0 needs ``ns``: the length is broadcast first."""
    import numpy as np
    import torch
    import torch.distributed as dist
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return np.ascontiguousarray(ns, dtype=np.uint64)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    rank = dist.get_rank(group)
    k = torch.tensor([len(ns) if rank == 0 else 0], dtype=torch.int64, device=dev)
    dist.broadcast(k, src=0, group=group)
    if rank == 0:
        t = torch.from_numpy(np.ascontiguousarray(ns, dtype=np.uint64).astype(np.int64)).to(dev)
    else:
        t = torch.zeros(int(k.item()), dtype=torch.int64, device=dev)
    dist.broadcast(t, src=0, group=group)
    return t.cpu().numpy().astype(np.uint64)
