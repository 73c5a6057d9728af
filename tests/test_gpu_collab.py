"""Collaborative CPU + GPU counting:
a host-resident handle whose sparsest pieces are counted by host threads from the
pinned host blocks while the GPU counts the rest.  Counts, per-task counts and
multi-rank sums must equal the oracle's for every share, in both orientations."""
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


@pytest.mark.parametrize("orient", ["auto", "low", "mid"])
@pytest.mark.parametrize("permille", [0, 1, 250, 700, 1000])
def test_host_share_counts(orient, permille):
    for g, p in ((gen.rmat(13, 16, seed=101), 5), (gen.er(1 << 13, 24, seed=102), 4),
                 (gen.grid(150, 0.4, seed=103), 1)):
        P = ob.Plan(*g, p=p, orient={"auto": 0, "low": 1, "mid": 2}[orient])
        with pg.build_blocks(*g, p=p, orient=orient, residency=pg.RESIDENT_HOST, host_permille=permille,
                             host_threads=4) as b:
            T, tc = b.triangle_count(task_counts=True)
            assert T == oracle.count(*g)
            assert list(map(int, tc)) == P.task_counts()
            st = b.stats()
            if permille == 1000:
                assert st["ms_host_last"] > 0 and st["h2d_bytes_last"] == 0   # nothing copied
            if permille == 0:
                assert st["ms_host_last"] == 0


def test_host_share_ranks_and_errors():
    g = gen.rmat(12, 16, seed=104)
    T0 = oracle.count(*g)
    total = 0
    for r in range(3):
        with pg.build_blocks(*g, p=4, rank=r, world_size=3, residency=pg.RESIDENT_HOST, host_permille=400) as b:
            total += b.triangle_count()
    assert total == T0
    for kw in ({"host_permille": 300}, {"host_permille": 1001, "residency": pg.RESIDENT_HOST},
               {"host_permille": 300, "residency": pg.RESIDENT_HOST, "device_budget_bytes": 1 << 30}):
        with pytest.raises(pg.PgabbError) as e:
            pg.build_blocks(*g, p=4, **kw)
        assert e.value.name == "EINVAL"
    with pg.build_blocks(*g, p=4, residency=pg.RESIDENT_HOST, host_permille=300) as b:
        with pytest.raises(pg.PgabbError):
            b.vertex_triangles()
