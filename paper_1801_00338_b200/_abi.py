"""ctypes binding of libbfly_b200.so (include/bfly_b200.h) and libbfly_synth.so.

This is plumbing for the Python mirror of the reference API (api.py), for the tests and
for bench.py. The library is loaded from this package directory only; if it is missing
the import fails loudly -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbfly_b200.so")
SYNTH_PATH = os.path.join(HERE, "libbfly_synth.so")

U64P = C.POINTER(C.c_uint64)
U32P = C.POINTER(C.c_uint32)
U8P = C.POINTER(C.c_uint8)
F64P = C.POINTER(C.c_double)
VP = C.c_void_p


class PairCounts(C.Structure):
    _fields_ = [("bfly", C.c_uint64)] + [(f, C.c_uint64 * 2) for f in
                                         ("p_0v", "p_1v", "p_2v", "p_1e", "p_1w")]


class Stats(C.Structure):
    _fields_ = [("n", C.c_uint64), ("left", C.c_uint64), ("right", C.c_uint64),
                ("m", C.c_uint64), ("sum_deg_sq_left", C.c_double),
                ("sum_deg_sq_right", C.c_double), ("wedge_count", C.c_uint64),
                ("max_degree", C.c_uint32)]


# name -> (restype, argtypes); every symbol declared in include/bfly_b200.h
SIGNATURES = {
    "bfly_last_error": (C.c_char_p, []),
    "bfly_version": (C.c_char_p, []),
    "bfly_device_ok": (C.c_int, []),
    "bfly_graph_build_u32": (C.c_int, [U32P, U32P, C.c_uint64, C.POINTER(VP)]),
    "bfly_graph_build_u64": (C.c_int, [U64P, U64P, C.c_uint64, C.POINTER(VP)]),
    "bfly_graph_build_u32_device": (C.c_int, [VP, VP, C.c_uint64, C.POINTER(VP)]),
    "bfly_graph_load_text": (C.c_int, [C.c_char_p, C.c_uint64, C.POINTER(VP), U64P]),
    "bfly_graph_serialize": (C.c_int, [VP, C.c_char_p, C.c_uint64, U64P]),
    "bfly_graph_free": (None, [VP]),
    "bfly_graph_sizes": (C.c_int, [VP, U32P, U32P, U64P]),
    "bfly_graph_export": (C.c_int, [VP, U64P, U32P, U64P, U32P, U32P, U64P, U64P]),
    "bfly_has_edge_batch": (C.c_int, [VP, U32P, U32P, C.c_uint64, U8P]),
    "bfly_edge_at_batch": (C.c_int, [VP, U64P, C.c_uint64, U32P, U32P]),
    "bfly_graph_stats": (C.c_int, [VP, C.POINTER(Stats)]),
    "bfly_choose_side": (C.c_int, [VP, C.POINTER(C.c_int), F64P, F64P]),
    "bfly_exact_count": (C.c_int, [VP, C.c_int, U64P]),
    "bfly_local_vertex_all": (C.c_int, [VP, U64P]),
    "bfly_local_edge_all": (C.c_int, [VP, U64P]),
    "bfly_local_vertex_batch": (C.c_int, [VP, U64P, C.c_uint64, U64P]),
    "bfly_local_edge_batch": (C.c_int, [VP, U64P, C.c_uint64, U64P]),
    "bfly_local_edge_pairs": (C.c_int, [VP, U32P, U32P, C.c_uint64, U64P]),
    "bfly_wedge_batch": (C.c_int, [VP, U64P, U32P, U32P, C.c_uint64, U64P]),
    "bfly_wedge_index": (C.c_int, [VP, U64P, U64P]),
    "bfly_fast_edge_batch": (C.c_int, [VP, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, F64P,
                                       U64P, U64P]),
    "bfly_sample_batch": (C.c_int, [VP, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, U64P, U64P,
                                    U32P, U32P]),
    "bfly_common_neighbors_batch": (C.c_int, [VP, C.c_int, U32P, U32P, C.c_uint64, U64P]),
    "bfly_espar_count": (C.c_int, [VP, C.c_double, C.c_uint64, U64P, U64P]),
    "bfly_cspar_count": (C.c_int, [VP, C.c_uint64, C.c_uint64, U64P, U64P]),
    "bfly_keep_mask_count": (C.c_int, [VP, U8P, U64P, U64P]),
    "bfly_color_mask_count": (C.c_int, [VP, U32P, U64P, U64P]),
    "bfly_graph_stream": (VP, [VP]),
    "bfly_set_stream": (None, [VP]),
    "bfly_last_sample_path": (C.c_int, [VP]),
    "bfly_profile_enable": (None, [C.c_int]),
    "bfly_profile_reset": (None, []),
    "bfly_profile_count": (C.c_int, []),
    "bfly_profile_get": (C.c_int, [C.c_int, C.POINTER(C.c_char_p), F64P, U64P]),
    "bfly_launch_count": (C.c_uint64, []),
    "bfly_trim_pool": (C.c_int, [C.c_uint64]),
    "bfly_graph_build_pairs": (C.c_int, [U64P, C.c_uint64, C.POINTER(VP)]),
    "bfly_sparsify_stats": (C.c_int, [VP, C.c_int, U64P]),
    "bfly_last_exact_stats": (C.c_int, [VP, U64P, U64P, U64P, U64P, U64P]),
    "bfly_last_dense_stats": (C.c_int, [VP, U64P]),
    "bfly_pair_type_counts": (C.c_int, [VP, C.POINTER(PairCounts)]),
}

SYNTH_SIGNATURES = {
    "bfly_synth_uniform": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, U32P,
                                     U32P]),
    "bfly_synth_chung_lu": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint64, C.c_double,
                                      C.c_double, C.c_uint32, C.c_uint64, U32P, U32P]),
}

HOST_PATH = os.path.join(HERE, "libbfly_host.so")
HOST_SIGNATURES = {
    "bfly_host_last_error": (C.c_char_p, []),
    "bfly_host_run_estimator": (C.c_int, [VP, C.c_int, C.c_uint64, C.c_double, C.c_uint64,
                                          C.c_uint64, C.c_uint64, C.c_int, C.c_uint, F64P,
                                          U64P, F64P, F64P, U64P]),
    "bfly_host_run_estimator_ex": (C.c_int, [VP, C.c_int, C.c_uint64, C.c_double, C.c_uint64,
                                             C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                             C.c_uint, F64P, U64P, F64P, F64P, U64P]),
    "bfly_host_time_from_pairs": (C.c_int, [U32P, U32P, C.c_uint64, C.c_int, F64P, U64P]),
    "bfly_host_sample_ids": (C.c_int, [VP, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                                       C.c_uint, U64P, U32P, U32P]),
    "bfly_host_sparsify_run": (C.c_int, [VP, C.c_int, C.c_double, C.c_uint64, C.c_uint64,
                                         C.c_uint64, F64P, F64P]),
}

_lib = None
_synth = None
_host = None


def host():
    """The C++ facade library (estimator drivers); loads libbfly_b200.so first."""
    global _host
    if _host is None:
        lib()
        _host = _bind(HOST_PATH, HOST_SIGNATURES)
    return _host


def _bind(path, sigs):
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `make` (or "
                          f"`python -c 'import __graft_entry__ as g; g.build()'`)")
    lib = C.CDLL(path)
    for name, (res, args) in sigs.items():
        f = getattr(lib, name)  # AttributeError == header/library mismatch: fail loudly
        f.restype = res
        f.argtypes = args
    return lib


def lib():
    global _lib
    if _lib is None:
        _lib = _bind(LIB_PATH, SIGNATURES)
    return _lib


def synth():
    global _synth
    if _synth is None:
        _synth = _bind(SYNTH_PATH, SYNTH_SIGNATURES)
    return _synth


def last_error() -> str:
    msg = lib().bfly_last_error()
    return msg.decode() if msg else ""
