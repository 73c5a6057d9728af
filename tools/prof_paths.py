"""Per-path SM-cycle breakdown of k_tc_rows (instrumented build, -DPGABB_PROF).

    python tools/prof_paths.py build            # here: nvcc -> libpgabb_prof.so
    python tools/prof_paths.py run c2 [c5 ...]  # on a GPU box: one count per config

Each warp accumulates clock64() deltas per code path in registers (count.cu
PROF_MARK) and adds them to a device array at exit; shares are of the summed
warp-cycles, so they say where warps spend their time, not wall time.
"""
import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CATS = {0: "item setup", 1: "probe_dense_row", 2: "stage set", 3: "dense AND", 4: "skew search",
        5: "long lists", 6: "short flattened", 7: "reduce+atomic", 8: "mode2 fallback",
        9: "batch header", 10: "batched small rows", 16: "#items dense-row", 17: "#items bitmap", 18: "#items hash",
        19: "#items mode2"}


def build():
    import __graft_entry__ as g
    srcs = [os.path.join(g.CSRC, f) for f in sorted(os.listdir(g.CSRC)) if f.endswith(".cu")]
    out = os.path.join(g.PKG, "libpgabb_prof.so")
    subprocess.check_call([g.NVCC, *g.NVCC_FLAGS, "-DPGABB_PROF", "-I", os.path.join(ROOT, "include"),
                           *srcs, "-o", out])
    print(out)


def run(names):
    os.environ["PGABB_LIB_VARIANT"] = "prof"
    import paper_2209_04541_b200 as pg
    from gen.configs import CONFIGS
    lib = pg._lib
    lib.pgabb_prof_read.argtypes = [ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
    buf = (ctypes.c_uint64 * 32)()
    for spec in names:
        name, _, path = spec.partition(":")   # "c2" (count) or "c2:vertex" (per-vertex t(v), VM=3)
        cfg = CONFIGS[name]
        n, s, d = cfg.generate()
        with pg.build_blocks(n, s, d, p=cfg.p) as b:
            run1 = (lambda: int(b.vertex_triangles()[0].sum()) // 3) if path == "vertex" else b.triangle_count
            run1()
            lib.pgabb_prof_read(buf, 1)
            T = run1()
            ms = b.stats()["ms_main_kernel_last"]
            lib.pgabb_prof_read(buf, 1)
        tot = sum(buf[c] for c in range(11))
        res = {"config": spec, "triangles": T, "kernel_ms": ms,
               "share": {CATS[c]: round(buf[c] / max(tot, 1), 4) for c in range(11)},
               "counts": {CATS[c]: int(buf[c]) for c in range(16, 20)}}
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    else:
        run(sys.argv[2:])
