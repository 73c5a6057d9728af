"""Attribute an ncu SASS source page (instructions executed, stall samples) to CUDA
source lines, using nvdisasm's line info for the kernel in the cubin.

    python tools/sass_lines.py <ncu-rep> <cubin> <kernel-substring (mangled, for the cubin)> [<ncu kernel regex>]
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict


def line_map(cubin, kname):
    out = subprocess.check_output(["nvdisasm", "-g", "-c", cubin], text=True, stderr=subprocess.DEVNULL)
    cur_fn, cur_line, mapping = None, None, {}
    for ln in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            cur_fn = m.group(1)
            continue
        m = re.search(r"//## File \"([^\"]+)\", line (\d+)", ln)
        if m:
            cur_line = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur_fn and kname in cur_fn:
            mapping[int(m.group(1), 16)] = cur_line
    return mapping


def main(rep, cubin, kname, ncu_kname=None):
    mp = line_map(cubin, kname)
    raw = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                                   "-k", f"regex:{ncu_kname or kname}"], text=True)
    rows = list(csv.reader(io.StringIO(raw)))
    hi = next(k for k, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hi]
    data = []
    for r in rows[hi + 1:]:
        if not r or r[0] in ("Kernel Name", "Address"):
            break   # next kernel's section
        data.append(r)
    iE, iW = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    ins, stl = defaultdict(int), defaultdict(int)
    for k, r in enumerate(data):
        key = mp.get(16 * k, "?")
        ins[key] += int(r[iE] or 0)
        stl[key] += int(r[iW] or 0)
    ti, ts = sum(ins.values()) or 1, sum(stl.values()) or 1
    for key in sorted(ins, key=lambda q: -ins[q])[:30]:
        print(f"{key:22s} inst {100 * ins[key] / ti:5.1f}%  stall {100 * stl[key] / ts:5.1f}%")


if __name__ == "__main__":
    main(*sys.argv[1:])
