"""Small runs of every kernel path for compute-sanitizer (memcheck / racecheck):
    compute-sanitizer --tool memcheck python tools/sanitize_run.py
Each call is checked against the oracle, so a silent corruption fails too."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import gen  # noqa: E402
import oracle  # noqa: E402
import paper_2209_04541_b200 as pg  # noqa: E402

cases = [
    ("rmat12 p4", gen.rmat(12, 16, seed=3), dict(p=4)),
    ("rmat14 p8", gen.rmat(14, 16, seed=4), dict(p=8)),
    ("wide p1", gen.disjoint_union(gen.rmat(16, 8, seed=7), gen.complete(700)), dict(p=1)),   # hash + mode 2
    ("er p6", gen.er(1 << 14, 24, seed=5), dict(p=6)),
    ("grid p3", gen.grid(200, 0.3, seed=6), dict(p=3)),
    ("cliques p5", gen.clique_union([3, 40, 200, 1, 90]), dict(p=5)),
]
for name, g, kw in cases:
    T, tv = oracle.count(*g, per_vertex=True)
    lab, k = oracle.components(*g)
    with pg.build_blocks(*g, **kw) as b:
        assert b.triangle_count() == T, name
        t2, _ = b.vertex_triangles()
        assert np.array_equal(t2, tv), name
        l2, k2, _ = b.connected_components()
        assert k2 == k and np.array_equal(l2, lab), name
        ns = b.task_times()
        mt = b.stats()["max_task_bytes"]
    with pg.build_blocks(*g, residency=pg.RESIDENT_HOST, device_budget_bytes=3 * mt, **kw) as b:
        assert b.triangle_count() == T, name
        t3, _ = b.vertex_triangles()
        assert np.array_equal(t3, tv), name
    with pg.build_blocks(*g, rank=1, world_size=3, task_weights=ns, **kw) as b:
        b.triangle_count()
    print("ok", name, flush=True)
