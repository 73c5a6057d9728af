"""Write tests/golden/triangles.json: the oracle's triangle counts for the full-size
BASELINE configs.  Calls only gen/ (inputs) and oracle/ (counts) -- never the
CUDA path.  Usage:  python tests/golden/make_golden.py c2 c3 c4 c5
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import gen  # noqa: E402
import oracle  # noqa: E402
from gen.configs import CONFIGS  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "triangles.json")


def main(names):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for name in names:
        cfg = CONFIGS[name]
        t0 = time.time()
        n, s, d = cfg.generate()
        t_gen = time.time() - t0
        t0 = time.time()
        g = oracle.Graph(n, s, d)
        del s, d
        t_build = time.time() - t0
        t0 = time.time()
        T = g.count()
        t_count = time.time() - t0
        rec = {"config": cfg.desc, "n": n, "m_edges": g.m_edges, "wedges": g.wedges(), "triangles": T,
               "oracle": "oracle/tc_oracle.c node iterator", "cores": oracle.threads(),
               "seconds": {"generate": round(t_gen, 1), "oracle_build": round(t_build, 1),
                           "oracle_count": round(t_count, 1)}}
        if cfg.kind == "grid":
            rec["closed_form"] = 2 * gen.grid_ndiag(*cfg.args)
        g.close()
        data[name] = rec
        json.dump(data, open(OUT, "w"), indent=1, sort_keys=True)
        print(name, rec, flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c3", "c4"])
