"""Streaming-residency timeline (S9 / NEXT-2): one traced count of a host-resident
handle through a device budget, written as a Chrome trace (chrome://tracing,
Perfetto) plus an overlap summary.  nsys is not in this image; the timeline comes
from the library's own CUDA events (PGABB_COUNT_TRACE, pgabb_get_wave_trace).

    python tools/wave_trace.py c5 16 > gpurun_out/wave_trace_c5.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2209_04541_b200 as pg  # noqa: E402
from gen.configs import CONFIGS  # noqa: E402


def main(name, budget_gb="16", orient="auto"):
    cfg = CONFIGS[name]
    n, s, d = cfg.generate()
    with pg.build_blocks(n, s, d, p=cfg.p, orient=orient, residency=pg.RESIDENT_HOST,
                         device_budget_bytes=int(float(budget_gb) * (1 << 30))) as b:
        b.triangle_count()                       # warm-up
        T = b.triangle_count(trace=True)
        tr = b.wave_trace()
        st = b.stats()
    events = []
    for k, (c0, c1, k0, k1) in enumerate(tr):
        events.append({"name": f"H2D wave {k}", "ph": "X", "pid": 0, "tid": "copy stream", "ts": c0 * 1e3,
                       "dur": max(0.0, c1 - c0) * 1e3})
        events.append({"name": f"intersect wave {k}", "ph": "X", "pid": 0, "tid": "count stream",
                       "ts": k0 * 1e3, "dur": max(0.0, k1 - k0) * 1e3})
    copy = sum(max(0.0, c1 - c0) for c0, c1, _, _ in tr)
    comp = sum(max(0.0, k1 - k0) for _, _, k0, k1 in tr)
    # copy time hidden under compute: overlap of wave k+1's copy with wave k's compute
    hidden = sum(max(0.0, min(tr[k + 1][1], tr[k][3]) - max(tr[k + 1][0], tr[k][2])) for k in range(len(tr) - 1))
    summary = {"config": name, "budget_gb": float(budget_gb), "orient": orient, "triangles": T,
               "waves": len(tr), "ms_count": st["ms_count_last"], "ms_copy_sum": copy, "ms_compute_sum": comp,
               "ms_copy_hidden": hidden, "h2d_bytes": st["h2d_bytes_last"], "d2d_bytes": st["d2d_bytes_last"],
               "block_bytes": st["block_bytes"]}
    json.dump({"traceEvents": events, "displayTimeUnit": "ms", "summary": summary}, sys.stdout)
    print(json.dumps(summary), file=sys.stderr)


if __name__ == "__main__":
    main(*sys.argv[1:])
