"""ctypes binding of libpsg.so (the C ABI declared in include/psg.h).

The shared library is built in-tree by paper_2605_03561_b200/build.py.  There
is no fallback: if the library or a CUDA device is missing, loading fails
loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# PSG_LIB overrides the library path (A/B runs of tools/variants.sh builds)
LIB_PATH = os.environ.get("PSG_LIB") or os.path.join(HERE, "libpsg.so")

# ps_status (reference proj/include/perfslice.h:24-40)
PS_OK = 0
STATUS_NAMES = [
    "ok", "io_error", "format_error", "invalid_image", "not_found", "invalid_config",
    "no_summary", "degenerate_summary", "parse_error", "no_such_metric", "no_periodicity",
    "no_outliers", "insufficient_data", "invalid_argument", "internal",
]

Q_WINDOW, Q_CUBE, Q_STATS, Q_OUTLIERS = 1, 2, 4, 8
Q_NO_CUBE_STORE = 1 << 8
Q_CLAMP_TEND = 1 << 9
Q_CUBE64 = 1 << 10
Q_EXACT_BOUNDS = 1 << 11
Q_SPARSE = 1 << 12
Q_ALL = Q_WINDOW | Q_CUBE | Q_STATS | Q_OUTLIERS
ANCHOR_AUTO = 0xFFFFFFFF


class PsgError(RuntimeError):
    def __init__(self, status: int, message: str):
        name = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)
        super().__init__(f"{name}: {message}")
        self.status = status
        self.name = name


class IterScenario(C.Structure):
    _fields_ = [
        ("n_ranks", C.c_uint32), ("n_iterations", C.c_uint32), ("n_kernels", C.c_uint32),
        ("mean_time_s", C.POINTER(C.c_double)), ("jitter_frac", C.POINTER(C.c_double)),
        ("spread", C.POINTER(C.c_double)), ("spread_kernel_stride", C.c_uint64),
        ("copy_segment_s", C.c_double), ("seed", C.c_uint64),
    ]


class ShardInfo(C.Structure):
    _fields_ = [("n_traces", C.c_uint32), ("n_ctx", C.c_uint32), ("n_events", C.c_uint64),
                ("t_min", C.c_uint64), ("t_max", C.c_uint64)]


class QuerySpec(C.Structure):
    _fields_ = [
        ("flags", C.c_uint32), ("t0_ns", C.c_uint64), ("t1_ns", C.c_uint64),
        ("anchor_ctx", C.c_uint32), ("site_ctx", C.POINTER(C.c_uint32)), ("n_sites", C.c_uint32),
        ("top_k", C.c_uint32), ("z_min", C.c_double),
    ]


class PsgCol(C.Structure):
    _fields_ = [("dtype", C.c_uint32), ("data", C.c_void_p)]


class QueryInfo(C.Structure):
    _fields_ = [
        ("n_window_groups", C.c_uint64), ("n_window_rows", C.c_uint64),
        ("n_nodes", C.c_uint32), ("n_kept", C.c_uint32), ("n_skipped", C.c_uint32),
        ("min_iterations", C.c_uint32), ("n_kept_global", C.c_uint32), ("n_cells", C.c_uint64),
        ("n_leaves", C.c_uint32), ("n_internal", C.c_uint32), ("anchor", C.c_uint32),
        ("worst_site", C.c_uint32), ("worst_ratio", C.c_double),
        ("n_outliers", C.c_uint32), ("n_racks", C.c_uint32),
        ("ms_total", C.c_float), ("ms_main", C.c_float), ("ms_bounds", C.c_float),
        ("cube_cell_bytes", C.c_uint32), ("cube_store_bytes", C.c_uint64),
        ("host_syncs", C.c_uint32), ("window_sparse", C.c_uint32), ("n_remat_rows", C.c_uint64),
    ]


_lib = None

# int (*)(void* buf, uint64_t count, int dtype, int op, void* user)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.c_int, C.c_int, C.c_void_p)

P = C.c_void_p
U8P, U32P, U64P = C.POINTER(C.c_uint8), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)
U16P = C.POINTER(C.c_uint16)
I32P, I64P, F64P = C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_double)

_SIGS = {
    "psg_version": (C.c_char_p, []),
    "psg_last_error": (C.c_char_p, []),
    "psg_status_name": (C.c_char_p, [C.c_int]),
    "psg_open": (C.c_int, [C.c_int, P, C.POINTER(P)]),
    "psg_close": (None, [P]),
    "psg_stream": (P, [P]),
    "psg_device_bytes": (C.c_uint64, [P]),
    "psg_comm_unique_id": (C.c_int, [U8P]),
    "psg_comm_init": (C.c_int, [P, C.c_int, C.c_int, U8P]),
    "psg_comm_init_host": (C.c_int, [P, C.c_int, C.c_int, ALLREDUCE_FN, P]),
    "psg_set_cct": (C.c_int, [P, U32P, C.c_uint32]),
    "psg_load_traces_aos": (C.c_int, [P, P, C.c_uint64, U64P, U32P, U64P, C.c_uint32]),
    "psg_prefetch_aos": (C.c_int, [P, P, C.c_uint64]),
    "psg_load_trace_db": (C.c_int, [P, C.c_char_p, U32P, C.c_uint32]),
    "psg_generate_iterative": (C.c_int, [P, C.POINTER(IterScenario), C.c_uint32, C.c_uint32]),
    "psg_set_nodes": (C.c_int, [P, U32P, C.c_uint32, U32P, U32P]),
    "psg_shard": (C.c_int, [P, C.POINTER(ShardInfo)]),
    "psg_get_traces": (C.c_int, [P, U64P, U32P, U64P, U64P, U32P]),
    "psg_query": (C.c_int, [P, C.POINTER(QuerySpec), C.POINTER(QueryInfo)]),
    "psg_get_window": (C.c_int, [P, U64P, I64P, I64P, I64P, F64P, I64P, I64P]),
    "psg_get_carry": (C.c_int, [P, U8P, U64P, U32P]),
    "psg_get_window_groups": (C.c_int, [P, U64P, U32P, U32P, U64P, I64P, I64P, I64P, F64P]),
    "psg_get_remat_rows": (C.c_int, [P, U64P, U32P, U32P, I64P, I64P]),
    "psg_get_cube": (C.c_int, [P, U32P, U32P, U64P, I64P, I64P, I64P, I64P]),
    "psg_get_stats": (C.c_int, [P, C.c_double, U32P, F64P, F64P, F64P, I32P]),
    "psg_get_outliers": (C.c_int, [P, F64P, F64P, F64P, U32P, U32P, U64P, U64P]),
    "psg_get_topology": (C.c_int, [P, U32P, U32P]),
    "psg_get_boundaries": (C.c_int, [P, C.c_uint32, U32P, U64P]),
    "psg_node_name": (C.c_int, [C.c_char_p, U32P, U32P]),
    "psg_dev_alloc": (C.c_int, [P, C.c_uint64, C.POINTER(C.c_void_p)]),
    "psg_dev_free": (None, [P, C.c_void_p]),
    "psg_copy": (C.c_int, [P, C.c_void_p, C.c_void_p, C.c_uint64]),
    "psg_vector_stats": (C.c_int, [P, F64P, C.c_uint64, C.c_uint32, F64P]),
    "psg_node_means": (C.c_int, [P, F64P, U32P, C.c_uint64, C.c_uint32, F64P, U32P]),
    "psg_localize": (C.c_int, [P, U32P, U32P, C.c_uint32, C.c_uint32, U32P, C.c_uint32, U32P, U32P]),
    "psg_get_cube_stored": (C.c_int, [P, U32P, U32P, U64P, C.c_void_p, U64P, U64P, I64P]),
    "psg_get_cube_stored_async": (C.c_int, [P, C.c_void_p, U64P, I64P]),
    "psg_wait_copies": (C.c_int, [P]),
    "psg_get_cube_range": (C.c_int, [P, C.c_uint32, C.c_uint32, U64P, U32P, I64P, I64P, I64P, I64P]),
    "psg_export_aos_range": (C.c_int, [P, C.c_uint32, C.c_uint32, C.c_void_p]),
    "psg_window_rows": (C.c_int, [P, C.c_uint64, C.c_uint64, U64P, U32P, U64P, U32P]),
    "psg_export_aos": (C.c_int, [P, P]),
    "psg_kernel_launches": (C.c_uint64, []),
    "psg_load_profiles": (C.c_int, [P, P, U64P, U32P, I32P, U32P, C.c_uint32]),
    "psg_load_profile_db": (C.c_int, [P, C.c_char_p]),
    "psg_slice": (C.c_int, [P, U32P, C.c_uint32, U32P, C.c_uint32, U16P, C.c_uint32, U64P, U32P, U32P,
                            U16P, F64P]),
    "psg_profile_outliers": (C.c_int, [P, C.c_uint16, U32P, C.c_uint32, C.c_uint32, C.c_double,
                                       C.POINTER(QueryInfo)]),
    "psg_frame_argsort": (C.c_int, [P, C.POINTER(PsgCol), C.c_uint32, U8P, C.c_uint64, P]),
    "psg_frame_group": (C.c_int, [P, C.POINTER(PsgCol), C.c_uint32, C.c_uint64, P, P, U64P]),
    "psg_frame_group_agg": (C.c_int, [P, PsgCol, P, P, C.c_uint64, C.c_uint64, C.c_uint32, P]),
    "psg_frame_gather": (C.c_int, [P, PsgCol, P, C.c_uint64, P]),
    "psg_frame_filter": (C.c_int, [P, PsgCol, C.c_uint32, P, C.c_uint64, P, U64P]),
    "psg_frame_merge": (C.c_int, [P, C.POINTER(PsgCol), C.POINTER(PsgCol), C.c_uint32, C.c_uint64,
                                  C.c_uint64, C.c_uint64, P, P, U64P]),
    "psg_frame_vector_add": (C.c_int, [P, P, P, C.c_uint64, P]),
    "psg_frame_multiply": (C.c_int, [P, P, C.c_double, C.c_uint64, P]),
    "psg_frame_scalar_compare": (C.c_int, [P, P, C.c_uint32, C.c_double, C.c_uint64, P]),
    "psg_frame_reduce_sum": (C.c_int, [P, P, C.c_uint64, C.POINTER(C.c_double)]),
    "psg_frame_cumsum": (C.c_int, [P, P, C.c_uint64, P]),
}

EXPORTED = sorted(_SIGS)


def load(path: str = LIB_PATH):
    """Loads libpsg.so and declares every entry point of include/psg.h."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -m paper_2605_03561_b200.build` "
            "(no CPU fallback exists for the psg kernels)")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int):
    if status != PS_OK:
        raise PsgError(status, load().psg_last_error().decode())
