"""N>1 host logic on CPU: world_size-2 gloo process groups.

Each rank takes its LPT share of the row pieces (S8, computed identically and
independently on every rank -- no scheduling messages), counts it, and the
partial counts are combined with ONE allreduce (S11).  On CPU the per-piece
counts come from the oracle's definitions (there is no GPU here); the GPU
version of the same flow is tests/test_gpu_parity.py::test_pieces_lpt_and_rank_sum
and bench.py under torchrun.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import gen
import oracle
import oracle.blocks as ob


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, graph, p, out):
    import torch.distributed as dist

    from paper_2209_04541_b200.dist import combine_counts_host
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        P = ob.Plan(*graph, p=p, G=ws)
        mine = [pc for pc, o in zip(P.pieces, P.owner) if o == rank]
        local = sum(ob.piece_count(P.B, P.tasks[pc[0]], pc[1], pc[2]) for pc in mine)
        total = combine_counts_host(local)
        # every rank derived the same plan without exchanging it
        import torch
        sig = torch.tensor([hash(tuple(P.owner)) & 0x7fffffff], dtype=torch.int64)
        sigs = [torch.zeros_like(sig) for _ in range(ws)]
        dist.all_gather(sigs, sig)
        out[rank] = (local, total, len(set(int(s) for s in sigs)) == 1, sum(pc[3] for pc in mine))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2])
def test_gloo_lpt_shares_sum_to_T(ws):
    graph = gen.rmat(9, 16, seed=31)
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(ws, port, graph, 3, out), nprocs=ws, join=True)
    T = oracle.count(*graph)
    locals_ = [out[r][0] for r in range(ws)]
    assert sum(locals_) == T
    assert all(out[r][1] == T for r in range(ws))
    assert all(out[r][2] for r in range(ws))
    loads = [out[r][3] for r in range(ws)]
    assert max(loads) <= 1.5 * (sum(loads) / ws)   # LPT keeps the shares balanced


def _worker_weights(rank, ws, port, graph, p, out):
    import numpy as np
    import torch.distributed as dist

    from paper_2209_04541_b200.dist import broadcast_weights, combine_counts_host, combine_vertex_counts_host
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        P0 = ob.Plan(*graph, p=p)
        # rank 0's "measurement" (here: seeded numbers standing in for pgabb_task_times);
        # the other ranks start from zeros and must receive rank 0's values
        ns = (np.random.default_rng(7).integers(1, 10 ** 9, len(P0.tasks)).astype(np.uint64)
              if rank == 0 else np.zeros(len(P0.tasks), np.uint64))
        w = broadcast_weights(ns)
        P = ob.Plan(*graph, p=p, G=ws, weights=[int(x) for x in w])
        mine = [pc for pc, o in zip(P.pieces, P.owner) if o == rank]
        local = sum(ob.piece_count(P.B, P.tasks[pc[0]], pc[1], pc[2]) for pc in mine)
        total = combine_counts_host(local)
        # per-vertex partials: t(v) restricted to this rank's pieces, summed by one allreduce
        tv = np.zeros(graph[0], np.uint64)
        for pc in mine:
            i, j, x = P.tasks[pc[0]]
            rp_ij, col_ij = P.B[(i, j)]
            for r in range(pc[1], pc[2]):
                for v in col_ij[rp_ij[r]:rp_ij[r + 1]]:
                    common = np.intersect1d(ob.row(P.B, i, x, r), ob.row(P.B, j, x, int(v)))
                    for gid in ([P.cuts[i] + r] * len(common) + [P.cuts[j] + int(v)] * len(common)
                                + [P.cuts[x] + int(c) for c in common]):
                        tv[gid] += 1
        tv_all = combine_vertex_counts_host(tv)
        out[rank] = (total, [int(a) for a in w], [int(a) for a in tv_all])
    finally:
        dist.destroy_process_group()


def test_gloo_measured_weights_plan_and_vertex_allreduce():
    ws = 2
    graph = gen.rmat(8, 16, seed=32)
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_weights, args=(ws, port, graph, 3, out), nprocs=ws, join=True)
    T, tv = oracle.count(*graph, per_vertex=True)
    assert out[0][1] == out[1][1]                         # every rank planned with rank 0's E(t)
    assert all(out[r][0] == T for r in range(ws))
    # rank-space t(v) summed over ranks: its multiset equals the oracle's t(v) (ids permuted by rank)
    P0 = ob.Plan(*graph, p=3)
    got = np.asarray(out[0][2], np.uint64)
    want = np.zeros(graph[0], np.uint64)
    want[P0.rank] = tv                                     # t in rank space
    assert np.array_equal(got, want)
