"""Compact summary of an ncu launch list (--metrics gpu__time_duration.sum --csv):
per kernel name, launch count and total / mean device time, and each kernel's
share of the count-phase launches (k_tc_rows + k_tc_light + k_sum_tasks)."""
import csv
import collections
import json
import sys


def summarize(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.DictReader(lines)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("pgabb::<unnamed>::", "")
        if name.startswith("void "):
            name = name[5:]
        name = name.split("<")[0] if name.startswith("k_") else name   # k_tc_rows<0, 0> -> k_tc_rows
        unit = r["Metric Unit"]
        v = float(r["Metric Value"].replace(",", ""))
        ns = v * {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "s": 1e9}.get(unit, 1)
        rows.append((name, ns))
    agg = collections.OrderedDict()
    for name, ns in rows:
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ns
    count_phase = {k: v for k, v in agg.items() if k in ("k_tc_rows", "k_tc_light", "k_sum_tasks")}
    tot = sum(v[1] for v in count_phase.values()) or 1.0
    out = {k: {"launches": v[0], "total_ms": v[1] / 1e6, "mean_ms": v[1] / v[0] / 1e6,
               "share_of_count_phase": (v[1] / tot) if k in count_phase else None} for k, v in agg.items()}
    return out


if __name__ == "__main__":
    print(json.dumps(summarize(sys.argv[1]), indent=1))
