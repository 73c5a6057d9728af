"""Collect one GPU call's evidence into profiles/: the bench line, the ncu launch
list summary and the ncu --set full summary of k_tc_rows.

    python tools/make_profile.py <tag> <config> [round]
reads gpurun_out/{bench,launches,prof}_<tag>.* and writes profiles/r<round>_<tag>.json;
also records the kernel's DRAM bytes per launch in profiles/ncu_summary.json
(bench.py reports it as roofline.traffic for that config).
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)

from launch_summary import summarize  # noqa: E402
from ncu_summary import summary  # noqa: E402


def to_bytes(s):
    v, u = s.split()
    return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[u]


def aggregate(ks):
    """One summary over launches of several instantiations (sums and time-weighted ratios)."""
    def num(d, q):
        return float(str(d.get(q, "0 x")).split()[0] or 0)
    def unit(d, q):
        parts = str(d.get(q, "")).split()
        return parts[1] if len(parts) > 1 else ""
    t = [num(d, "gpu__time_duration.sum") * {"ms": 1.0, "s": 1e3, "us": 1e-3}.get(unit(d, "gpu__time_duration.sum"), 1.0)
         for d in ks]
    T = sum(t) or 1.0
    out = dict(ks[0])
    out["kernel"] = " + ".join(d["kernel"] for d in ks)
    out["gpu__time_duration.sum"] = f"{sum(t)} ms"
    for q in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        out[q] = f"{sum(to_bytes(d[q]) for d in ks)} byte"
    out["smsp__inst_executed.sum"] = f"{sum(num(d, 'smsp__inst_executed.sum') for d in ks)} inst"
    for q in list(out):
        if q.endswith(".pct") or q.endswith("pct_of_peak_sustained_active") or q.startswith("smsp__pcsamp"):
            try:
                out[q] = f"{sum(num(d, q) * ti for d, ti in zip(ks, t)) / T} {unit(ks[0], q)}"
            except Exception:
                pass
    return out


def main(tag, config, rnd="01", src_hash=None):
    """src_hash: bench.kernel_src_hash() of the sources the capture ran (default: now)."""
    if src_hash is None:
        sys.path.insert(0, ROOT)
        from bench import kernel_src_hash
        src_hash = kernel_src_hash()
    g = os.path.join(ROOT, "gpurun_out")
    out = {"tag": tag, "config": config}
    bj = os.path.join(g, f"bench_{tag}.json")
    if os.path.exists(bj):
        lines = [ln for ln in open(bj) if ln.strip().startswith("{")]
        out["bench"] = json.loads(lines[0]) if lines else None
    lc = os.path.join(g, f"launches_{tag}.csv")
    if os.path.exists(lc):
        s = summarize(lc)
        cp = ("k_tc_rows", "k_tc_light", "k_sum_tasks")
        out["launches"] = {k: v for k, v in s.items() if k in cp}
        out["launches_build_total_ms"] = sum(v["total_ms"] for k, v in s.items() if k not in cp)
        out["launches_note"] = ("ncu launch list (--metrics gpu__time_duration.sum --clock-control none): "
                                "cold-cache, serialised; compare shares, not absolutes")
    rep = os.path.join(g, f"prof_{tag}.ncu-rep")
    if os.path.exists(rep):
        ns = os.path.join(ROOT, "profiles", "ncu_summary.json")
        js = json.load(open(ns)) if os.path.exists(ns) else {}
        entry = js.get(config, {})
        entry = {k: v for k, v in entry.items() if k.startswith("k_")}   # per-kernel entries only
        for kname in ("k_tc_rows", "k_tc_light"):
            ks = [d for d in summary(rep) if kname in d["kernel"]]
            if not ks:
                continue
            k = ks[0]
            # several instantiations of one kernel in one count (k_tc_light<.., 8> and the
            # medium <.., 15>, R29): the capture must hold one launch of each; their DRAM
            # bytes, times and instructions add, ratios are time-weighted
            inst = {}
            for d in ks:
                inst.setdefault(d["kernel"], d)
            if len(inst) > 1:
                k = aggregate(list(inst.values()))
            out[f"ncu_{kname}"] = k
            traffic = to_bytes(k["dram__bytes_read.sum"]) + to_bytes(k["dram__bytes_write.sum"])
            out[f"dram_bytes_per_launch_{kname}"] = traffic
            stalls = {q.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v.split()[0] or 0)
                      for q, v in k.items() if q.startswith("smsp__pcsamp_warps_issue_stalled_")
                      and not q.endswith("_not_issued")}
            top = max(stalls, key=stalls.get) if stalls else None
            entry[kname] = {"dram_bytes_per_launch": traffic, "source": f"profiles/r{rnd}_{tag}.json",
                            "l2_hit_pct": k.get("lts__t_sector_hit_rate.pct"),
                            "kernel_ms_under_ncu": k.get("gpu__time_duration.sum"),
                            "issue_active_pct": k.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                            "warp_inst_per_launch": float(k["smsp__inst_executed.sum"].split()[0]),
                            "top_stall": top, "src_hash": src_hash}
        js[config] = entry
        json.dump(js, open(ns, "w"), indent=1, sort_keys=True)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    path = os.path.join(ROOT, "profiles", f"r{rnd}_{tag}.json")
    json.dump(out, open(path, "w"), indent=1)
    print(path)


if __name__ == "__main__":
    main(*sys.argv[1:])
