"""Full-size parity at BASELINE.json's configs, in the launch configuration bench.py
times (same p, same cut rule, device-resident blocks).

Expected values come from tests/golden/triangles.json, written by
tests/golden/make_golden.py, which calls only gen/ and oracle/ (never the CUDA
path); c4 is additionally pinned by its closed form T = 2 * (#diagonal cells).
c2 is also re-counted by the oracle in the test itself.
"""
import json
import os

import numpy as np
import pytest

import gen
import oracle
from gen.configs import CONFIGS

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2209_04541_b200 as pg  # noqa: E402

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "triangles.json")))


def run(name, **kw):
    cfg = CONFIGS[name]
    n, s, d = cfg.generate()
    kw.setdefault("p", cfg.p)
    with pg.build_blocks(n, s, d, **kw) as b:
        st = b.stats()
        T = b.triangle_count()
    return (n, s, d), T, st


def test_c2_vs_oracle_in_job_and_golden():
    g, T, st = run("c2")
    assert T == GOLDEN["c2"]["triangles"]
    assert st["m_edges"] == GOLDEN["c2"]["m_edges"]
    assert st["wedges"] == GOLDEN["c2"]["wedges"]
    assert T == oracle.count(*g)


@pytest.mark.parametrize("p,rule", [(4, 0), (16, 0), (8, 1), (1, 0)])
def test_c2_p_invariance(p, rule):
    _, T, _ = run("c2", p=p, cut_rule=rule)
    assert T == GOLDEN["c2"]["triangles"]


def test_c3_er_full():
    _, T, st = run("c3")
    assert T == GOLDEN["c3"]["triangles"]
    assert st["m_edges"] == GOLDEN["c3"]["m_edges"]


def test_c4_grid_full_closed_form():
    _, T, _ = run("c4")
    side, f, seed = CONFIGS["c4"].args
    assert T == 2 * gen.grid_ndiag(side, f, seed) == GOLDEN["c4"]["triangles"]


def test_c5_graph500_s26_full():
    _, T, st = run("c5")
    assert st["m_edges"] == GOLDEN["c5"]["m_edges"]
    assert st["wedges"] == GOLDEN["c5"]["wedges"]
    assert T == GOLDEN["c5"]["triangles"]


def test_c5_streamed_out_of_core():
    # S9 streaming: blocks in pinned host memory, a device budget
    # of 14 GiB (about half the block CSR with the MID transposes, R25), double-buffered
    # waves -- same exact count
    _, T, st = run("c5", residency=pg.RESIDENT_HOST, device_budget_bytes=14 << 30)
    assert st["waves"] > 1
    assert T == GOLDEN["c5"]["triangles"]


def test_two_c5_copies_streamed_beyond_c5():
    # NEXT-2 at twice C5's size: the disjoint union of C5 and
    # a relabelled copy -- n = 2^27, |E| = 2 x 2,078,644,777 = 4.16e9 edges -- built
    # from host tuples (chunked upload, 64-bit edge offsets), kept in pinned host DRAM
    # and counted through a 32 GiB device budget, about half the ~60 GB of blocks.
    # Exact pin without the oracle: disjoint-union additivity, T = 2 T(C5) (golden).
    cfg = CONFIGS["c5"]
    n, s, d = cfg.generate()
    s2 = np.concatenate([s, s + np.uint32(n)])
    del s
    d2 = np.concatenate([d, d + np.uint32(n)])
    del d
    with pg.build_blocks(2 * n, s2, d2, p=cfg.p, residency=pg.RESIDENT_HOST,
                         device_budget_bytes=32 << 30) as b:
        del s2, d2
        st = b.stats()
        assert st["m_edges"] == 2 * GOLDEN["c5"]["m_edges"]
        assert st["block_bytes"] > 32 << 30
        assert st["waves"] > 1
        T = b.triangle_count(trace=True)
        assert T == 2 * GOLDEN["c5"]["triangles"]
        tr = b.wave_trace()
        assert tr.shape == (st["waves"], 4)
        assert (tr[:, 1] <= tr[:, 2] + 1e-3).all()        # a wave computes after its copy


def test_c2_per_vertex_and_clustering_full():
    # NEXT-1 at the bench's c2 size: every t(v) and cc(v) against the oracle
    cfg = CONFIGS["c2"]
    n, s, d = cfg.generate()
    want_tv, want_cc = oracle.clustering(n, s, d)
    with pg.build_blocks(n, s, d, p=cfg.p) as b:
        tv, T = b.vertex_triangles()
        cc = b.local_clustering(tv)
    assert T == GOLDEN["c2"]["triangles"]
    assert np.array_equal(tv, want_tv)
    assert np.array_equal(cc, want_cc)


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_components_full(name):
    # NEXT-4 at full size: every label against the oracle's union-find
    cfg = CONFIGS[name]
    n, s, d = cfg.generate()
    want, k = oracle.components(n, s, d)
    with pg.build_blocks(n, s, d, p=cfg.p) as b:
        lab, kk, _ = b.connected_components()
    assert kk == k and np.array_equal(lab, want)
