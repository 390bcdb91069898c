"""ctypes binding of libdndc.so (include/dndc.h).

The shared library is built in-tree by `paper_2007_13552_b200/csrc/Makefile`
(`__graft_entry__.build()`).  There is no fallback: if the library is missing
or cannot be loaded, importing the package's compute API raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
# DNDC_LIB_PATH: an alternative build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("DNDC_LIB_PATH") or os.path.join(HERE, "libdndc.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "dndc.h")

DNDC_OK, DNDC_EVALUE, DNDC_ETRANSPORT, DNDC_ECUDA, DNDC_EINTERNAL, DNDC_EDATA = 0, 1, 2, 3, 4, 5
DNDC_ETIMEOUT, DNDC_EORDERING = 6, 7
UNIQUE_ID_BYTES = 128


class TransportError(RuntimeError):
    """dnd::TransportError (errors.hpp:21-25)."""


class TimeoutError_(TransportError):
    """dnd::TimeoutError (errors.hpp:27-31): a rank did not arrive in time."""


class OrderingError(TransportError):
    """dnd::OrderingError (errors.hpp:33-37): ranks entered different collectives."""


class DataError(RuntimeError):
    """dnd::DataError (errors.hpp:40): file I/O and container format."""


class DeviceError(RuntimeError):
    """A CUDA failure inside libdndc."""


class Counters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in
                ("sends", "recvs", "sendrecvs", "allreduces", "allgathers", "alltoalls", "barriers")]


_P, _i64, _u64, _i32, _f64 = C.c_void_p, C.c_int64, C.c_uint64, C.c_int, C.c_double

# name -> argtypes; restype int unless listed in _RESTYPE
_SIGS = {
    "dndc_version": [],
    "dndc_last_error": [],
    "dndc_unique_id": [_P],
    "dndc_create": [_i32, _i32, _i32, _P, C.POINTER(_P)],
    "dndc_destroy": [_P],
    "dndc_set_stream": [_P, _P],
    "dndc_rank": [_P],
    "dndc_world": [_P],
    "dndc_transport_status": [_P],
    "dndc_synchronize": [_P],
    "dndc_get_counters": [_P, C.POINTER(Counters)],
    "dndc_launch_count": [_P],
    "dndc_chunk_map": [_i64, _i32, _P, _P],
    "dndc_device_count": [_P],
    "dndc_barrier": [_P],
    "dndc_alloc": [_P, C.c_size_t, _P],
    "dndc_free": [_P, _P],
    "dndc_memcpy": [_P, _P, _P, C.c_size_t, _i32],
    "dndc_allgather_rows": [_P, _P, _i64, _i64, _P, _P],
    "dndc_resplit": [_P, _P, _i32, _P, _i64, _i32, _i32, _P],
    "dndc_file_read_to_device": [_P, C.c_char_p, _u64, C.c_size_t, _P],
    "dndc_lasso_fit_f64": [_P, _P, _i64, _i64, _i64, _P, _f64, _i32, _f64, _P, _P, _P],
    "dndc_lasso_predict_f64": [_P, _P, _i64, _i64, _P, _P],
    "dndc_file_write_from_device": [_P, C.c_char_p, _u64, _P, C.c_size_t],
    "dndc_allreduce_f64": [_P, _P, _i64],
    "dndc_kmeans_step_f32": [_P, _P, _i64, _i64, _P, _i32, _P, _P],
    "dndc_kmeans_step_f64": [_P, _P, _i64, _i64, _P, _i32, _P, _P],
    "dndc_fill_uniform_f32": [_P, _u64, _i64, _i64, _i64, _P],
    "dndc_fill_uniform_f64": [_P, _u64, _i64, _i64, _i64, _P],
    "dndc_row_norms_f32": [_P, _P, _i64, _i64, _P],
    "dndc_row_norms_f64": [_P, _P, _i64, _i64, _P],
    "dndc_cdist_tile_f32": [_P, _P, _P, _i64, _P, _P, _i64, _i64, _P, _i64, _i64, _i64],
    "dndc_cdist_tile_f64": [_P, _P, _P, _i64, _P, _P, _i64, _i64, _P, _i64, _i64, _i64],
    "dndc_cdist_f32": [_P, _P, _i64, _i64, _i64, _P],
    "dndc_cdist_f64": [_P, _P, _i64, _i64, _i64, _P],
    "dndc_cdist_xy_f32": [_P, _P, _i64, _P, _i64, _i64, _P],
    "dndc_cdist_xy_f64": [_P, _P, _i64, _P, _i64, _i64, _P],
    "dndc_cdist_xy_ring_f32": [_P, _P, _i64, _P, _i64, _i64, _i64, _P],
    "dndc_cdist_xy_ring_f64": [_P, _P, _i64, _P, _i64, _i64, _i64, _P],
    "dndc_kmeans_init_indices": [_i64, _i32, _u64, _P],
    "dndc_kmeans_init_centroids_f32": [_P, _P, _i64, _i64, _i64, _i32, _u64, _P],
    "dndc_kmeans_fit_f32": [_P, _P, _i64, _i64, _i64, _i32, _i32, _f64, _u64, _P, _P, _P, _P],
    "dndc_kmeans_fit_f64": [_P, _P, _i64, _i64, _i64, _i32, _i32, _f64, _u64, _P, _P, _P, _P],
    "dndc_kmeans_predict_f32": [_P, _P, _i64, _i64, _P, _i32, _P],
    "dndc_kmeans_predict_f64": [_P, _P, _i64, _i64, _P, _i32, _P],
    "dndc_kmeans_last_refined": [_P, C.POINTER(_i64)],
    "dndc_kmeans_assign_timing": [_P, _i32],
    "dndc_kmeans_last_assign_ms": [_P, _P, _P],
    "dndc_kmeans_time_assign_f32": [_P, _P, _i64, _i64, _i32, _i32, _P, _P],
    "dndc_moments_axis0_f32": [_P, _P, _i64, _i64, _P, _P, _P],
    "dndc_moments_axis0_f64": [_P, _P, _i64, _i64, _P, _P, _P],
    "dndc_kmeanspp_indices_f32": [_P, _P, _i64, _i64, _i64, _i32, _u64, _P],
    "dndc_kmeanspp_indices_f64": [_P, _P, _i64, _i64, _i64, _i32, _u64, _P],
    "dndc_kmeans_last_kernel": [_P],
    "dndc_kmeans_persist_trace": [_P, _P, _i64, _P],
    "dndc_group_create": [_i32, _i64, C.POINTER(_P)],
    "dndc_group_destroy": [_P],
    "dndc_group_abort": [_P],
    "dndc_create_in_group": [_i32, _i32, _P, _i32, C.POINTER(_P)],
}
_RESTYPE = {"dndc_last_error": C.c_char_p, "dndc_launch_count": C.c_uint64, "dndc_transport_status": C.c_char_p,
            "dndc_kmeans_last_kernel": C.c_char_p, "dndc_kmeans_persist_trace": C.c_int64}


def header_symbols() -> list[str]:
    """Every function include/dndc.h declares (for the export check)."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(dndc_[a-z0-9_]+)\s*\(", text)))


_lib = None


def lib():
    """Load libdndc.so once; raise (never fall back) if it is unavailable."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (the CUDA path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = _RESTYPE.get(name, C.c_int)
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == DNDC_OK:
        return
    msg = lib().dndc_last_error().decode(errors="replace")
    if rc == DNDC_EVALUE:
        raise ValueError(msg)
    if rc == DNDC_ETRANSPORT:
        raise TransportError(msg)
    if rc == DNDC_EDATA:
        raise DataError(msg)
    if rc == DNDC_ETIMEOUT:
        raise TimeoutError_(msg)
    if rc == DNDC_EORDERING:
        raise OrderingError(msg)
    raise DeviceError(f"libdndc error {rc}: {msg}")
