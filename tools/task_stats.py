"""Per-task structure of a built block grid (for kernel tuning): widths, block
densities, nnz, S7 costs and staged-model bytes.  Runs on a GPU box:
    python tools/task_stats.py c5s [p] [orient] > gpurun_out/tasks_c5s.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2209_04541_b200 as pg  # noqa: E402
from gen.configs import CONFIGS  # noqa: E402


def main(name, p=None, orient="auto"):
    cfg = CONFIGS[name]
    n, s, d = cfg.generate()
    with pg.build_blocks(n, s, d, p=int(p) if p else cfg.p, orient=orient) as b:
        st = b.stats()
        cuts = [int(c) for c in b.cuts()]
        p = len(cuts) - 1
        nnz = {}
        import ctypes
        for i in range(p):
            for j in range(i, p):
                z = ctypes.c_uint64(0)
                pg._lib.pgabb_get_block(b._h, i, j, None, None, ctypes.byref(z))
                nnz[(i, j)] = int(z.value)
        ijx, cost, alg = b.tasks()
        dirs, s_low, s_mid = b.task_orient()
        ns = b.task_times()
        tasks = []
        for t in range(len(cost)):
            i, j, x = (int(v) for v in ijx[t])
            wj, wx = cuts[j + 1] - cuts[j], cuts[x + 1] - cuts[x]
            tasks.append({"t": [i, j, x], "wi": cuts[i + 1] - cuts[i], "wj": wj, "wx": wx,
                          "nnz_ij": nnz[(i, j)], "nnz_ix": nnz[(i, x)], "nnz_jx": nnz[(j, x)],
                          "dens_jx": nnz[(j, x)] / max(1, wj * wx), "cost": int(cost[t]), "alg_bytes": int(alg[t]),
                          "dir": int(dirs[t]), "s_low": int(s_low[t]), "s_mid": int(s_mid[t]), "ns": int(ns[t])})
        json.dump({"config": name, "stats": st, "cuts": cuts, "tasks": tasks}, sys.stdout)


if __name__ == "__main__":
    main(*sys.argv[1:])
