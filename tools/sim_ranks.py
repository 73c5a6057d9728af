"""Projected multi-GPU balance on ONE GPU: every logical rank r of G builds its own
handle (rank=r, world_size=G: the S8 LPT share it would own on an 8-GPU box) and
times its count phase alone; the projected G-GPU count time is the max over ranks
(plus the 8-byte allreduce, a few microseconds over NVLink, not included).
Counts are summed and checked against the 1-rank total.

    python tools/sim_ranks.py c5 1 2 4 8 [--measured] > gpurun_out/sim_c5.json
(--measured: plan with rank 0's measured task times, DESIGN R22)

This is evidence for load balance (the only thing that separates the ranks: no
data-path collective), not a substitute for a real multi-GPU run.
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2209_04541_b200 as pg  # noqa: E402
from gen.configs import CONFIGS  # noqa: E402


def time_rank(n, s, d, p, r, G, steps=3, warmup=2, weights=None):
    with pg.build_blocks(n, s, d, p=p, rank=r, world_size=G, device=0, task_weights=weights) as b:
        for _ in range(warmup):
            T = b.triangle_count()
        ms = []
        for _ in range(steps):
            T = b.triangle_count()
            ms.append(b.stats()["ms_count_last"])
        st = b.stats()
        return T, statistics.median(ms), int(st["cost_local"]), int(st["items_heavy"]), int(st["items_light"])


def main(name, Gs, balance):
    cfg = CONFIGS[name]
    n, s, d = cfg.generate()
    out = {"config": name, "workload": cfg.desc, "p": cfg.p, "balance": balance, "by_G": {}}
    weights = None
    if balance == "measured":   # rank 0's pgabb_task_times on a 1-rank handle (dist.build_blocks_balanced)
        with pg.build_blocks(n, s, d, p=cfg.p, device=0) as b1:
            b1.triangle_count()
            weights = b1.task_times()
    t1 = None
    for G in Gs:
        ranks = []
        for r in range(G):
            T, ms, cost, ih, il = time_rank(n, s, d, cfg.p, r, G, weights=weights if G > 1 else None)
            ranks.append({"rank": r, "triangles": T, "ms": ms, "cost": cost, "items_heavy": ih, "items_light": il})
            print(f"{name} G={G} r={r} ms={ms:.3f} T={T}", file=sys.stderr, flush=True)
        tmax = max(x["ms"] for x in ranks)
        total = sum(x["triangles"] for x in ranks)
        if t1 is None and G == 1:
            t1 = tmax
        out["by_G"][G] = {"ranks": ranks, "projected_ms": tmax, "triangles": total,
                          "cost_balance": min(x["cost"] for x in ranks) / max(1, max(x["cost"] for x in ranks)),
                          "projected_efficiency": (t1 / (G * tmax)) if t1 else None}
    Ts = {v["triangles"] for v in out["by_G"].values()}
    out["counts_agree"] = len(Ts) == 1
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    torch.cuda.init()
    args = sys.argv[1:]
    bal = "cost"
    if "--measured" in args:
        args.remove("--measured")
        bal = "measured"
    main(args[0], [int(x) for x in args[1:]] or [1, 2, 4, 8], bal)
