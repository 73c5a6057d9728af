"""The library's N > 1 flow on real devices: one process per rank,
each builds its rank's handle through the C ABI (dist.build_blocks_for_rank),
counts its LPT share on the GPU and the shares are combined by one allreduce.

* two ranks on ONE GPU over gloo (runs on any GPU box): the library path of every
  rank, with the host-side allreduce;
* two ranks on TWO GPUs over NCCL (skipped with fewer than 2 visible GPUs): the
  count and the n-vector t(v) allreduced on the device (triangle_count_allreduce,
  vertex_triangles_allreduce).
Both are checked against the oracle.
"""
import os
import socket

import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


GRAPH = (14, 16, 91)


def _worker(rank, ws, port, backend, orient, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import paper_2209_04541_b200 as pg  # noqa: F401
    from paper_2209_04541_b200 import dist as pgd
    dev = rank if backend == "nccl" else 0
    torch.cuda.set_device(dev)
    dist.init_process_group(backend, rank=rank, world_size=ws)
    g = gen.rmat(*GRAPH)
    with pgd.build_blocks_for_rank(*g, p=6, orient=orient) as b:
        if backend == "nccl":
            T = pgd.triangle_count_allreduce(b)
            tv = pgd.vertex_triangles_allreduce(b).cpu().numpy().astype(np.uint64)
            local = b.stats()["items_heavy"] + b.stats()["items_light"]
        else:
            T = pgd.combine_counts_host(b.triangle_count())
            tv_l, _ = b.vertex_triangles()
            tv = pgd.combine_vertex_counts_host(tv_l)
            local = b.stats()["items_heavy"] + b.stats()["items_light"]
    out[rank] = (int(T), tv.tobytes(), int(local))
    dist.barrier()
    dist.destroy_process_group()


def _run(backend, orient):
    ws = 2
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(ws, _port(), backend, orient, out), nprocs=ws, join=True)
        res = dict(out)
    T0, tv0 = oracle.count(*gen.rmat(*GRAPH), per_vertex=True)
    for r in range(ws):
        T, tvb, local = res[r]
        assert T == T0
        assert np.array_equal(np.frombuffer(tvb, np.uint64), tv0)
        assert local > 0                     # every rank owns work
    return res


@pytest.mark.parametrize("orient", ["auto", "low"])
def test_two_ranks_one_gpu_gloo(orient):
    _run("gloo", orient)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_two_ranks_two_gpus_nccl():
    _run("nccl", "auto")
