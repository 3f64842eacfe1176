"""ctypes binding of libsssp_cuda.so (include/sssp_cuda.h, include/sssp_graph_gen.h).

The shared library is the product: it is built in-tree by
``__graft_entry__.build()`` (``make -C paper_2504_03667_b200/csrc``).  There is
no fallback -- importing this module raises if the library is missing.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SSSP_LIB") or os.path.join(_HERE, "libsssp_cuda.so")  # SSSP_LIB: dev A/B builds

SSSP_OK = 0
SSSP_ERR_BAD_SOURCE = 1
SSSP_ERR_BAD_ARG = 2
SSSP_ERR_WEIGHT_RANGE = 3
SSSP_ERR_OOM = 4
SSSP_ERR_CUDA = 5
SSSP_ERR_NO_PEER = 6
SSSP_ERR_TIMEOUT = 7
SSSP_ERR_UNSUPPORTED = 8
SSSP_IPC_HANDLE_BYTES = 64
SSSP_FLAGS_DEFAULT = 3

# every symbol include/*.h declares (checked by tests/test_abi.py)
EXPORTED = (
    "sssp_status_string", "sssp_last_error", "sssp_abi_version", "sssp_device_count",
    "sssp_graph_create", "sssp_graph_create_from_edges", "sssp_shard_create", "sssp_shard_export", "sssp_shard_connect",
    "sssp_shard_range", "sssp_graph_destroy", "sssp_graph_info", "sssp_solve",
    "sssp_solve_batch", "sssp_enqueue", "sssp_finish", "sssp_stream",
    "sssp_probe_sync", "sssp_probe_skeleton", "sssp_nccl_begin", "sssp_nccl_local_min",
    "sssp_nccl_relax", "sssp_nccl_end", "sssp_validate", "sssp_solve_dataparallel", "sssp_round_times", "sssp_block_weight_range", "sssp_gen_dense", "sssp_gen_sparse", "sssp_gen_bernoulli", "sssp_graph_from_edges", "sssp_parse_edge_list",
)


class Options(ctypes.Structure):
    _fields_ = [
        ("engine", ctypes.c_int),
        ("ctas_per_shard", ctypes.c_uint32),
        ("flags", ctypes.c_uint32),
        ("max_batch", ctypes.c_uint32),
        ("timeout_ms", ctypes.c_uint64),
        ("record_visit_order", ctypes.c_int),
        ("replicas", ctypes.c_uint32),
        ("warps_per_cta", ctypes.c_uint32),
        ("global_min_weight", ctypes.c_int64),
        ("record_round_times", ctypes.c_int),
    ]


class Stats(ctypes.Structure):
    _fields_ = [
        ("transfer_in_s", ctypes.c_double),
        ("rounds_s", ctypes.c_double),
        ("transfer_out_s", ctypes.c_double),
        ("iterations", ctypes.c_uint64),
        ("relax_checks", ctypes.c_uint64),
        ("mispredicts", ctypes.c_uint64),
        ("matrix_bytes", ctypes.c_uint64),
        ("weight_bytes", ctypes.c_uint32),
        ("ctas", ctypes.c_uint32),
        ("shards", ctypes.c_uint32),
        ("packed_key", ctypes.c_uint32),
        ("engine", ctypes.c_uint32),
        ("classes", ctypes.c_uint32),
        ("rows_read", ctypes.c_uint64),
        # ABI 3: the reference's OpCounters / CollectiveStats, device exchange counts
        ("extract_min_scans", ctypes.c_uint64),
        ("ref_relax_checks", ctypes.c_uint64),
        ("allreduce_count", ctypes.c_uint64),
        ("scatter_bytes", ctypes.c_uint64),
        ("gather_bytes", ctypes.c_uint64),
        ("exchanges", ctypes.c_uint64),
        ("barriers", ctypes.c_uint64),
        ("upload_bytes", ctypes.c_uint64),
        ("download_bytes", ctypes.c_uint64),
        ("bytes_read", ctypes.c_uint64),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_u64p = ctypes.POINTER(ctypes.c_uint64)
_vp = ctypes.c_void_p


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    sig = {
        "sssp_status_string": (ctypes.c_char_p, [ctypes.c_int]),
        "sssp_last_error": (ctypes.c_char_p, []),
        "sssp_abi_version": (ctypes.c_int, []),
        "sssp_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
        "sssp_graph_create": (ctypes.c_int, [_u64p, ctypes.c_uint64, ctypes.c_int,
                                             ctypes.POINTER(ctypes.c_int), ctypes.c_int,
                                             ctypes.POINTER(Options), ctypes.POINTER(_vp)]),
        "sssp_graph_create_from_edges": (ctypes.c_int, [ctypes.c_uint64, _u64p, ctypes.c_uint64,
                                                        ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                                        ctypes.c_int, ctypes.POINTER(Options),
                                                        ctypes.POINTER(_vp)]),
        "sssp_shard_create": (ctypes.c_int, [_u64p, ctypes.c_uint64, ctypes.c_uint64,
                                             ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                                             ctypes.c_int, ctypes.POINTER(Options),
                                             ctypes.POINTER(_vp)]),
        "sssp_shard_export": (ctypes.c_int, [_vp, ctypes.c_void_p]),
        "sssp_shard_connect": (ctypes.c_int, [_vp, ctypes.c_void_p]),
        "sssp_shard_range": (ctypes.c_int, [_vp, _u64p, _u64p]),
        "sssp_graph_destroy": (ctypes.c_int, [_vp]),
        "sssp_graph_info": (ctypes.c_int, [_vp, ctypes.POINTER(Stats)]),
        "sssp_solve": (ctypes.c_int, [_vp, ctypes.c_uint64, _u64p, _u64p, _u64p,
                                      ctypes.POINTER(Stats)]),
        "sssp_solve_batch": (ctypes.c_int, [_vp, _u64p, ctypes.c_uint32, _u64p, _u64p,
                                            ctypes.POINTER(Stats)]),
        "sssp_enqueue": (ctypes.c_int, [_vp, _u64p, ctypes.c_uint32]),
        "sssp_finish": (ctypes.c_int, [_vp, ctypes.POINTER(Stats)]),
        "sssp_stream": (ctypes.c_void_p, [_vp, ctypes.c_int]),
        "sssp_probe_sync": (ctypes.c_int, [_vp, ctypes.c_uint32, ctypes.POINTER(ctypes.c_double)]),
        "sssp_probe_skeleton": (ctypes.c_int, [_vp, ctypes.c_uint32, ctypes.c_uint32,
                                               ctypes.POINTER(ctypes.c_double)]),
        "sssp_nccl_begin": (ctypes.c_int, [_vp, ctypes.c_uint64]),
        "sssp_nccl_local_min": (ctypes.c_int, [_vp, _vp]),
        "sssp_nccl_relax": (ctypes.c_int, [_vp, _vp]),
        "sssp_nccl_end": (ctypes.c_int, [_vp, _u64p, _u64p]),
        "sssp_validate": (ctypes.c_int, [_vp, ctypes.c_uint64, _u64p, _u64p, _u64p]),
        "sssp_solve_dataparallel": (ctypes.c_int, [_vp, ctypes.c_uint64, _u64p, _u64p, _u64p,
                                                   ctypes.POINTER(Stats)]),
        "sssp_round_times": (ctypes.c_int, [_vp, _u64p, ctypes.c_uint64, _u64p]),
        "sssp_block_weight_range": (ctypes.c_int, [_u64p, ctypes.c_uint64, ctypes.c_uint64,
                                                   ctypes.c_uint64, ctypes.c_uint64, _u64p, _u64p]),
        "sssp_parse_edge_list": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_uint64, _u64p, _u64p, _u64p,
                                                 ctypes.c_uint64, _u64p, ctypes.c_char_p,
                                                 ctypes.c_uint64]),
        "sssp_gen_dense": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                          ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                          _u64p]),
        "sssp_gen_sparse": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                           ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                           _u64p]),
        "sssp_gen_bernoulli": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint64,
                                              ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64,
                                              ctypes.c_uint64, ctypes.c_uint64, _u64p]),
        "sssp_graph_from_edges": (ctypes.c_int, [ctypes.c_uint64, _u64p, ctypes.c_uint64,
                                                 ctypes.c_int, ctypes.c_uint64,
                                                 ctypes.c_uint64, ctypes.c_uint64, _u64p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class SsspError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        detail = lib.sssp_last_error().decode(errors="replace")
        super().__init__(f"{where}: {lib.sssp_status_string(status).decode()} ({detail})")


def check(status: int, where: str) -> None:
    if status == SSSP_ERR_BAD_SOURCE:
        # serial.hpp:30 throws std::invalid_argument
        raise ValueError(f"{where}: source out of range")
    if status != SSSP_OK:
        raise SsspError(status, where)
