"""A/B kernel variants: in-tree builds of the same sources with extra -D switches,
selected at run time by PGABB_LIB_VARIANT=<name> (paper_2209_04541_b200/_abi.py).

    python tools/variants.py build <name> -DFOO=1 [-DBAR=2 ...]   # here (nvcc)
    PGABB_LIB_VARIANT=<name> python bench.py ...                  # on the GPU box
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build(name, defs):
    import __graft_entry__ as g
    srcs = [os.path.join(g.CSRC, f) for f in sorted(os.listdir(g.CSRC)) if f.endswith(".cu")]
    out = os.path.join(g.PKG, f"libpgabb_{name}.so")
    subprocess.check_call([g.NVCC, *g.NVCC_FLAGS, *defs, "-I", os.path.join(ROOT, "include"), *srcs, "-o", out])
    print(out)


if __name__ == "__main__":
    if len(sys.argv) >= 3 and sys.argv[1] == "build":
        build(sys.argv[2], sys.argv[3:])
    else:
        print(__doc__)
        sys.exit(2)
