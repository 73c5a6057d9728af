"""CPU-side checks of the C ABI: the library loads, exports every symbol that
include/pgabb.h declares, and -- without a GPU -- fails loudly (ECUDA), never
falling back to a CPU path."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pgabb.h")


@pytest.fixture(scope="module")
def lib_path():
    import __graft_entry__ as g
    return g.build_lib()


def declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"PGABB_API\s+[\w\s\*]*?\b(pgabb_\w+)\s*\(", txt)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("pgabb_build_blocks", "pgabb_triangle_count", "pgabb_free", "pgabb_last_error"):
        assert must in names
    assert len(names) >= 10


def test_every_declared_symbol_exported(lib_path):
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib_path]).decode()
    exported = set(re.findall(r"\b(pgabb_\w+)\b", out))
    missing = [s for s in declared() if s not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(lib_path)
    for s in declared():
        assert getattr(lib, s) is not None


def test_binding_matches_header():
    from paper_2209_04541_b200 import _abi
    assert sorted(n for n, _, _ in _abi.SIGNATURES) == declared()


def test_struct_layouts(tmp_path):
    # the ctypes mirrors against the C compiler's layout of include/pgabb.h
    from paper_2209_04541_b200 import _abi
    structs = {"BuildOpts": "pgabb_build_opts_t", "CountOpts": "pgabb_count_opts_t", "Stats": "pgabb_stats_t"}
    lines = []
    for py, c in structs.items():
        cls = getattr(_abi, py)
        lines.append(f'printf("{py} size %zu\\n", sizeof({c}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{py} {f} %zu\\n", offsetof({c}, {f}));')
    src = tmp_path / "layout.c"
    src.write_text("#include <stdio.h>\n#include <stddef.h>\n#include \"pgabb.h\"\nint main(void){"
                   + "".join(lines) + "return 0;}\n")
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = {}
    for ln in subprocess.check_output([str(exe)]).decode().splitlines():
        py, f, v = ln.split()
        got[(py, f)] = int(v)
    for py in structs:
        cls = getattr(_abi, py)
        assert got[(py, "size")] == ctypes.sizeof(cls), py
        for f, _ in cls._fields_:
            assert got[(py, f)] == getattr(cls, f).offset, (py, f)


def test_sm100a_cubin(lib_path):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path]).decode()
    assert "sm_100a" in out


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2209_04541_b200 as pg
    n, s, d = 3, np.array([0, 1, 2], np.uint32), np.array([1, 2, 0], np.uint32)
    with pytest.raises(pg.PgabbError) as e:
        pg.build_blocks(n, s, d, p=1)
    assert e.value.name in ("ECUDA", "EINVAL")


def test_null_arguments_rejected():
    import paper_2209_04541_b200 as pg
    lib = pg._lib
    assert lib.pgabb_build_blocks(3, 0, None, None, None, None) == 1   # out NULL -> EINVAL
    assert b"NULL" in lib.pgabb_last_error()
    assert lib.pgabb_triangle_count(None, None, None) == 1
    assert lib.pgabb_vertex_triangles(None, None, None, None) == 1
    assert lib.pgabb_local_clustering(None, None, None, None) == 1
    assert lib.pgabb_connected_components(None, None, None, None, None) == 1
    lib.pgabb_free(None)   # no-op
    assert pg.version().startswith("pgabb")
