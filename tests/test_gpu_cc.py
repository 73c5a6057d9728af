"""GPU parity of connected components: Shiloach-Vishkin
HOOK/LINK on the 2D blocks through pgabb_connected_components,
against the oracle's union-find.  Labels are canonical (smallest original id of
the component), so the comparison is element-by-element and bit-exact.
"""
import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2209_04541_b200 as pg  # noqa: E402


def check(g, **kw):
    want, nc = oracle.components(*g)
    with pg.build_blocks(*g, **kw) as b:
        lab, k, it = b.connected_components()
        assert lab.dtype == np.uint32 and lab.shape == (g[0],)
        assert np.array_equal(lab, want), kw
        assert k == nc and it >= 1
        assert b.triangle_count() == oracle.count(*g)   # the blocks are shared with S10
    return lab, it


@pytest.mark.parametrize("p", [1, 2, 5, 8])
def test_cc_families(p):
    check(gen.path(2000), p=p)                          # a long chain: many SV rounds
    check(gen.clique_union([3, 9, 1, 64, 200]), p=p)
    check(gen.disjoint_union(gen.star(50), gen.cycle(33), gen.king(9, 7), gen.random_tree(300, 4)), p=p)
    check(gen.grid(120, 0.2, seed=5), p=p)


@pytest.mark.parametrize("scale,ef,p", [(10, 1, 2), (14, 2, 4), (16, 16, 8)])
def test_cc_rmat(scale, ef, p):
    check(gen.rmat(scale, ef, seed=scale), p=p)        # low edge factor: many components


def test_cc_er_sparse_many_components():
    check(gen.er(1 << 16, 1.2, seed=7), p=6)            # below/around the giant-component threshold


def test_cc_degenerate_and_messy():
    e = np.zeros(0, np.uint32)
    with pg.build_blocks(9, e, e, p=3) as b:
        lab, k, _ = b.connected_components()
        assert lab.tolist() == list(range(9)) and k == 9
    check((4, np.arange(4, dtype=np.uint32), np.arange(4, dtype=np.uint32)), p=2)   # self-loops only
    check(gen.messy(gen.rmat(11, 4, seed=3), seed=4), p=3)
    check(gen.relabel(gen.path(500), seed=9), p=4)


def test_cc_host_residency_and_device_output():
    g = gen.rmat(13, 4, seed=12)
    want, nc = oracle.components(*g)
    with pg.build_blocks(*g, p=4, residency=pg.RESIDENT_HOST) as b:
        lab, k, _ = b.connected_components()
        assert np.array_equal(lab, want) and k == nc
    with pg.build_blocks(*g, p=4) as b:
        out = torch.empty(g[0], dtype=torch.int32, device="cuda")
        lab_d, k, _ = b.connected_components(out=out)
        assert np.array_equal(lab_d.cpu().numpy().astype(np.uint32), want) and k == nc
        assert b.stats()["ms_cc_last"] > 0


def test_cc_rejects_multirank_and_streaming():
    g = gen.rmat(10, 8, seed=1)
    with pg.build_blocks(*g, p=2, rank=0, world_size=2) as b:
        with pytest.raises(pg.PgabbError) as e:
            b.connected_components()
        assert e.value.name == "EINVAL"
    with pg.build_blocks(*g, p=2) as ref:
        mt = ref.stats()["max_task_bytes"]
    with pg.build_blocks(*g, p=2, residency=pg.RESIDENT_HOST, device_budget_bytes=8 * mt) as b:
        with pytest.raises(pg.PgabbError) as e:
            b.connected_components()
        assert e.value.name == "EINVAL"
