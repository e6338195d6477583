"""ctypes binding of the in-tree C ABI (include/mpb200.h, libmpb200.so).

There is no Python fallback: if the library is missing the import fails with
a message telling how to build it (the one exception is the build command
itself, `python -m paper_2604_22228_b200.build`, which must import the
package before the library exists: then `lib` is None and the package
exports nothing).  Every call returns a status; `check`
re-raises failures as the reference's exception classes with the message
text produced by the C++ side (which reproduces the reference wording).
"""

from __future__ import annotations

import ctypes as C
import os
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmpb200.so")

MP_OK = 0
MP_ERR_TOPOLOGY = -1
MP_ERR_PLAN = -2
MP_ERR_CHUNK = -3
MP_ERR_VALUE = -4
MP_ERR_CAPACITY = -5
MP_ERR_CUDA = -6
MP_ERR_STATE = -7

MP_HOST = -1
MP_NO_STAGE = -2

MP_PATH_DIRECT, MP_PATH_GPU, MP_PATH_HOST = 0, 1, 2
MP_ROLE_DIRECT, MP_ROLE_HOP1, MP_ROLE_HOP2 = 0, 1, 2
MP_SHARE_BANDWIDTH, MP_SHARE_EQUAL = 0, 1
MP_DUPLEX_FULL, MP_DUPLEX_HALF = 0, 1
MP_ENGINE_SM, MP_ENGINE_CE, MP_ENGINE_AUTO = 0, 1, 2
MP_COPY_VEC, MP_COPY_TMA = 0, 1
MP_SCHED_AUTO, MP_SCHED_DYNAMIC = 0, 1


class mp_config(C.Structure):
    _fields_ = [("num_gpu_paths", C.c_int32), ("host_path_enabled", C.c_int32),
                ("max_chunks", C.c_int32), ("graph_mode", C.c_int32),
                ("cache_capacity", C.c_int32), ("share_policy", C.c_int32)]


class mp_link(C.Structure):
    _fields_ = [("a", C.c_int32), ("b", C.c_int32), ("bandwidth", C.c_double),
                ("latency", C.c_double), ("duplex", C.c_int32), ("sublinks", C.c_int32)]


class mp_channel(C.Structure):
    _fields_ = [("id", C.c_char * 32), ("bandwidth", C.c_double), ("latency", C.c_double),
                ("a", C.c_int32), ("b", C.c_int32)]


class mp_hop(C.Structure):
    _fields_ = [("channel", C.c_int32), ("src", C.c_int32), ("dst", C.c_int32)]


class mp_path(C.Structure):
    _fields_ = [("kind", C.c_int32), ("stage", C.c_int32), ("share", C.c_double),
                ("nhops", C.c_int32), ("hops", mp_hop * 2)]


class mp_chunk(C.Structure):
    _fields_ = [("offset", C.c_uint64), ("length", C.c_uint64),
                ("path_index", C.c_int32), ("seq", C.c_int32)]


class mp_lane(C.Structure):
    _fields_ = [("lane_id", C.c_int32), ("path_index", C.c_int32), ("hop", C.c_int32),
                ("first", C.c_int32), ("count", C.c_int32)]


class mp_lane_dep(C.Structure):
    _fields_ = [("lane1", C.c_int32), ("pos1", C.c_int32), ("lane2", C.c_int32),
                ("pos2", C.c_int32)]


class mp_node(C.Structure):
    _fields_ = [("id", C.c_int32), ("src_dev", C.c_int32), ("dst_dev", C.c_int32),
                ("channel", C.c_int32), ("offset", C.c_uint64), ("length", C.c_uint64),
                ("lane", C.c_int32), ("role", C.c_int32), ("chunk_index", C.c_int32),
                ("path_index", C.c_int32)]


class mp_edge(C.Structure):
    _fields_ = [("from_", C.c_int32), ("to", C.c_int32)]


class mp_send_stats(C.Structure):
    _fields_ = [("hit", C.c_int32), ("graph_mode", C.c_int32), ("nodes_logical", C.c_int32),
                ("nodes_physical", C.c_int32), ("kernels", C.c_int32), ("ce_copies", C.c_int32),
                ("creation_us", C.c_double), ("construction_us", C.c_double),
                ("instantiation_us", C.c_double), ("launch_us", C.c_double),
                ("plan_us", C.c_double), ("cache_hits", C.c_uint64),
                ("cache_misses", C.c_uint64), ("cache_evictions", C.c_uint64),
                ("kernel", C.c_int32), ("pad", C.c_int32)]


class mp_trace_rec(C.Structure):
    _fields_ = [("node", C.c_int32), ("engine", C.c_int32), ("device", C.c_int32),
                ("pad", C.c_int32), ("start_us", C.c_double), ("end_us", C.c_double)]


class mp_xfer(C.Structure):
    _fields_ = [("src", C.c_void_p), ("dst", C.c_void_p), ("size", C.c_uint64),
                ("src_dev", C.c_int32), ("dst_dev", C.c_int32)]


class mp_engine_opts(C.Structure):
    _fields_ = [("direct_engine", C.c_int32), ("relay_engine", C.c_int32),
                ("copy_kind", C.c_int32), ("ctas_per_sm", C.c_int32), ("threads", C.c_int32),
                ("tile_bytes", C.c_int64), ("host_slots", C.c_int32), ("pull", C.c_int32),
                ("sm_min_bytes", C.c_int64), ("unroll", C.c_int32), ("tma_stages", C.c_int32),
                ("tma_block", C.c_int32), ("host_engine", C.c_int32), ("tma_peer", C.c_int32),
                ("sched", C.c_int32), ("small_max_bytes", C.c_int64),
                ("pdl", C.c_int32), ("wait_timeout_ms", C.c_int32),
                ("fault_inject", C.c_int32)]


P = C.POINTER
_vp = C.c_void_p
_i32 = C.c_int32
_u64 = C.c_uint64

# name -> (restype, argtypes); the list IS the exported surface of mpb200.h
SIGNATURES = {
    "mp_last_error": (C.c_char_p, []),
    "mp_abi_version": (C.c_int, []),
    "mp_topology_load": (C.c_int, [C.c_char_p, C.c_char_p, P(_vp)]),
    "mp_topology_create": (C.c_int, [C.c_char_p, _i32, P(mp_link), _i32, P(_vp)]),
    "mp_topology_destroy": (None, [_vp]),
    "mp_topology_info": (C.c_int, [_vp, P(_i32), P(_i32), P(_i32)]),
    "mp_topology_name": (C.c_int, [_vp, C.c_char_p, C.c_size_t]),
    "mp_topology_link": (C.c_int, [_vp, _i32, P(mp_link)]),
    "mp_topology_channel": (C.c_int, [_vp, _i32, P(mp_channel)]),
    "mp_topology_channel_for": (C.c_int, [_vp, _i32, _i32, P(_i32)]),
    "mp_config_validate": (C.c_int, [P(mp_config)]),
    "mp_plan_paths": (C.c_int, [_vp, _i32, _i32, P(mp_config), P(mp_path), _i32, P(_i32)]),
    "mp_plan_contention_free": (C.c_int, [_vp, P(_i32), P(_i32), _i32, P(mp_config),
                                          P(mp_path), _i32, P(_i32), P(_i32)]),
    "mp_pathset_validate": (C.c_int, [P(mp_path), _i32]),
    "mp_make_chunk_plan": (C.c_int, [P(mp_path), _i32, _u64, _i32, P(mp_chunk), _i32,
                                     P(_i32)]),
    "mp_lane_schedule": (C.c_int, [P(mp_path), _i32, P(mp_chunk), _i32, P(mp_lane), _i32,
                                   P(_i32), P(_i32), _i32, P(_i32), P(mp_lane_dep), _i32,
                                   P(_i32)]),
    "mp_build_graph": (C.c_int, [P(mp_path), _i32, P(mp_chunk), _i32, P(mp_node), _i32,
                                 P(_i32), P(mp_edge), _i32, P(_i32), P(_i32)]),
    "mp_graph_digest": (C.c_int, [P(mp_config), _i32, _i32, P(mp_path), _i32,
                                  P(C.c_char_p), _i32, C.c_char_p]),
    "mp_link_validate": (C.c_int, [P(mp_link)]),
    "mp_format_double": (C.c_int, [C.c_double, C.c_char_p, C.c_size_t]),
    "mp_cache_create": (C.c_int, [_i32, P(_vp)]),
    "mp_cache_destroy": (None, [_vp]),
    "mp_cache_access": (C.c_int, [_vp, C.c_char_p, C.c_size_t, P(_i32), P(_u64), P(_u64),
                                  _i32, P(_i32)]),
    "mp_cache_len": (C.c_int, [_vp, P(_i32)]),
    "mp_cache_contains": (C.c_int, [_vp, C.c_char_p, C.c_size_t, P(_i32)]),
    "mp_cache_values": (C.c_int, [_vp, P(_u64), _i32, P(_i32)]),
    "mp_ctx_create": (C.c_int, [_i32, P(_i32), P(_vp)]),
    "mp_ctx_destroy": (None, [_vp]),
    "mp_ctx_set_topology": (C.c_int, [_vp, _vp]),
    "mp_ctx_set_engine": (C.c_int, [_vp, P(mp_engine_opts)]),
    "mp_ctx_get_engine": (C.c_int, [_vp, P(mp_engine_opts)]),
    "mp_ctx_set_size_policy": (C.c_int, [_vp, P(C.c_uint64), P(_i32), P(_i32), _i32]),
    "mp_ctx_peer_matrix": (C.c_int, [_vp, P(_i32), _i32]),
    "mp_send": (C.c_int, [_vp, _vp, _vp, _u64, _i32, _i32, P(mp_config), _vp]),
    "mp_wait": (C.c_int, [_vp, _vp]),
    "mp_send_many": (C.c_int, [_vp, P(mp_xfer), _i32, P(mp_config), _i32, _vp]),
    "mp_send_trace": (C.c_int, [_vp, _vp, _vp, _u64, _i32, _i32, P(mp_config), P(mp_trace_rec),
                                _i32, P(_i32)]),
    "mp_send_stats_get": (C.c_int, [_vp, P(mp_send_stats)]),
    "mp_last_plan": (C.c_int, [_vp, P(mp_path), _i32, P(_i32), P(mp_chunk), _i32, P(_i32)]),
    "mp_cache_clear": (C.c_int, [_vp]),
    "mp_sync": (C.c_int, [_vp]),
    "mp_measure_paths": (C.c_int, [_vp, _i32, _i32, _u64, _i32, P(C.c_double), _i32]),
    "mp_kernel_time_ms": (C.c_int, [_vp, P(C.c_double)]),
    "mp_ctx_set_kernel_timing": (C.c_int, [_vp, _i32]),
    "mp_kernel_bench": (C.c_int, [_vp, _vp, _vp, _u64, _i32, _i32, P(mp_config), _i32,
                                  P(C.c_double)]),
    "mp_ipc_export": (C.c_int, [_vp, _i32, P(C.c_uint8), P(_u64)]),
    "mp_ipc_import": (C.c_int, [P(C.c_uint8), _i32, P(_vp)]),
    "mp_ipc_close": (C.c_int, [_vp, _i32]),
    "mp_group_create": (C.c_int, [_i32, _i32, _i32, _u64, _i32, P(_vp)]),
    "mp_group_export": (C.c_int, [_vp, P(C.c_uint8)]),
    "mp_group_host_arena": (C.c_int, [_vp, _u64]),
    "mp_group_import": (C.c_int, [_vp, _i32, P(C.c_uint8)]),
    "mp_group_open": (C.c_int, [_vp, P(C.c_uint8), _u64, P(_vp)]),
    "mp_group_send": (C.c_int, [_vp, _vp, C.c_uint32, _vp, _u64, _i32, _i32, P(mp_config), _vp]),
    "mp_group_role": (C.c_int, [_vp, P(_i32)]),
}

MP_GROUP_BLOB_BYTES = 256
MP_IPC_HANDLE_BYTES = 64


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the sm_100a engine first "
            "(python -m paper_2604_22228_b200.build, or python paper_2604_22228_b200/build.py). There is no Python fallback.")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def _building() -> bool:
    """True while `python -m paper_2604_22228_b200.build` imports the package."""
    a = getattr(sys, "orig_argv", [])
    return any(x == "-m" and y == f"{__package__}.build" for x, y in zip(a, a[1:]))


lib = None if _building() else _load()


class EngineError(RuntimeError):
    """A CUDA failure or misuse of the engine (no reference counterpart)."""


_ERROR_CLASSES: dict[int, type] = {}


def register_error(code: int, cls: type) -> None:
    _ERROR_CLASSES[code] = cls


def last_error() -> str:
    msg = lib.mp_last_error()
    return msg.decode() if msg else ""


def check(rc: int) -> None:
    if rc == MP_OK:
        return
    cls = _ERROR_CLASSES.get(rc, EngineError if rc in (MP_ERR_CUDA, MP_ERR_STATE) else ValueError)
    raise cls(last_error())


def format_double(x: float) -> str:
    buf = C.create_string_buffer(64)
    check(lib.mp_format_double(x, buf, 64))
    return buf.value.decode()
