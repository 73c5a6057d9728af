"""ctypes declarations of include/pgabb.h (argument marshalling only).

Loads the in-tree ``libpgabb.so`` built by ``__graft_entry__.build()``; there is
no fallback of any kind -- a missing library raises ImportError.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpgabb.so")
# tooling only (tools/prof_paths.py, tools/variants.py): an in-tree build of the same
# sources with other compile-time switches (instrumentation, kernel-variant A/B runs)
if os.environ.get("PGABB_LIB_VARIANT"):
    LIB_PATH = os.path.join(_HERE, "libpgabb_%s.so" % os.environ["PGABB_LIB_VARIANT"])

u32, u64, i32 = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32
u32p = ctypes.POINTER(ctypes.c_uint32)
u64p = ctypes.POINTER(ctypes.c_uint64)
i32p = ctypes.POINTER(ctypes.c_int32)
vp = ctypes.c_void_p

STATUS = {0: "OK", 1: "EINVAL", 2: "ENOMEM", 3: "ECUDA", 4: "ERANGE", 5: "EBUDGET"}
RESIDENT_DEVICE, RESIDENT_HOST = 0, 1
COUNT_ASYNC = 1
OUT_DEVICE = 2
ROLE_LOW, ROLE_MID, ROLE_HIGH = 4, 8, 16
OUT_ACCUMULATE = 32
COUNT_TRACE = 64


class BuildOpts(ctypes.Structure):
    _fields_ = [("p", u32), ("cut_rule", u32), ("device", i32), ("inputs_on_device", u32),
                ("rank", i32), ("world_size", i32), ("residency", u32), ("reverse_order", u32),
                ("device_budget_bytes", u64), ("task_weights", u64p), ("n_task_weights", u64),
                ("orient", u32), ("host_permille", u32), ("host_threads", u32), ("light_held", u32)]


class CountOpts(ctypes.Structure):
    _fields_ = [("cuda_stream", vp), ("d_count", vp), ("task_counts", u64p), ("flags", u32),
                ("reserved0", u32)]


class Stats(ctypes.Structure):
    _fields_ = [("n", u64), ("m_tuples", u64), ("m_edges", u64), ("p", u64), ("ntasks", u64),
                ("npieces", u64), ("npieces_local", u64), ("wedges", u64), ("cost_total", u64),
                ("cost_local", u64), ("alg_bytes_total", u64), ("alg_bytes_local", u64),
                ("block_bytes", u64), ("h2d_bytes_last", u64), ("launches_last", u64),
                ("waves", u64), ("max_task_bytes", u64), ("items_heavy", u64), ("items_light", u64),
                ("alg_bytes_light", u64), ("d2d_bytes_last", u64), ("ms_build", ctypes.c_double),
                ("ms_count_last", ctypes.c_double), ("ms_main_kernel_last", ctypes.c_double),
                ("ms_light_kernel_last", ctypes.c_double), ("ms_cc_last", ctypes.c_double),
                ("ms_host_last", ctypes.c_double), ("items_medium", u64), ("light_held", u64), ("ell_bytes", u64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if not k.startswith("reserved")}


# (name, restype, argtypes) for every entry point declared in include/pgabb.h
SIGNATURES = [
    ("pgabb_default_build_opts", None, [ctypes.POINTER(BuildOpts)]),
    ("pgabb_build_blocks", ctypes.c_int, [u32, u64, vp, vp, ctypes.POINTER(BuildOpts), ctypes.POINTER(vp)]),
    ("pgabb_triangle_count", ctypes.c_int, [vp, ctypes.POINTER(CountOpts), u64p]),
    ("pgabb_vertex_triangles", ctypes.c_int, [vp, ctypes.POINTER(CountOpts), vp, u64p]),
    ("pgabb_local_clustering", ctypes.c_int, [vp, ctypes.POINTER(CountOpts), vp, vp]),
    ("pgabb_get_stats", ctypes.c_int, [vp, ctypes.POINTER(Stats)]),
    ("pgabb_task_times", ctypes.c_int, [vp, u64p]),
    ("pgabb_connected_components", ctypes.c_int, [vp, ctypes.POINTER(CountOpts), vp, u64p, u32p]),
    ("pgabb_get_rank", ctypes.c_int, [vp, u32p]),
    ("pgabb_get_cuts", ctypes.c_int, [vp, u32p]),
    ("pgabb_get_block", ctypes.c_int, [vp, u32, u32, u32p, u32p, u64p]),
    ("pgabb_get_tasks", ctypes.c_int, [vp, u32p, u64p, u64p]),
    ("pgabb_get_task_orient", ctypes.c_int, [vp, u32p, u64p, u64p]),
    ("pgabb_get_pieces", ctypes.c_int, [vp, u32p, u32p, u32p, u64p, i32p]),
    ("pgabb_get_wave_trace", ctypes.c_int, [vp, ctypes.POINTER(ctypes.c_double), u64p]),
    ("pgabb_free", None, [vp]),
    ("pgabb_last_error", ctypes.c_char_p, []),
    ("pgabb_version", ctypes.c_char_p, []),
]


def load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        if os.environ.get("PGABB_LIB_VARIANT") and not hasattr(lib, name):
            continue   # A/B runs against an older build of the library (tools/variants.py)
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib
