"""Summarise an ncu --set full report: key throughput / stall metrics (reads with ncu -i)."""
import csv
import io
import json
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
        "sm__maximum_warps_per_active_cycle_pct", "launch__grid_size", "launch__block_size",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum", "smsp__average_warp_latency_per_inst_issued.ratio"]


def summary(rep):
    raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    out = []
    for v in vals:
        d = {"kernel": v[hdr.index("Kernel Name")][:60]}
        for i, k in enumerate(hdr):
            if k in WANT or k.startswith("smsp__average_warp_latency_issue_stalled") or \
                    k.startswith("smsp__pcsamp_warps_issue_stalled"):
                d[k] = f"{v[i]} {units[i]}".strip()
        out.append(d)
    return out


if __name__ == "__main__":
    for d in summary(sys.argv[1]):
        stalls = {k: v for k, v in d.items() if "stalled" in k}
        top = sorted(stalls.items(), key=lambda kv: -float(kv[1].split()[0].replace(",", "") or 0))[:8]
        base = {k: v for k, v in d.items() if "stalled" not in k}
        print(json.dumps(base, indent=1))
        print("top stalls:", json.dumps(dict(top), indent=1))
