"""ctypes binding of libswb.so (the C-ABI in include/swb.h).

The product path has no CPU fallback: if the shared library (built for sm_100a) is
missing this module raises at import, and on a machine without a B200 every entry point
that touches the device fails with ``CudaError``.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SWB_LIB") or os.path.join(_HERE, "_lib", "libswb.so")  # SWB_LIB: development A/B

SWB_OK, SWB_EINVAL, SWB_ECUDA, SWB_EUNSTABLE, SWB_ERANGE = 0, 1, 2, 3, 4
FORM_FACTORISED, FORM_PLAIN_F64, FORM_PLAIN_F32, FORM_FACTORISED_SIMPLE = 0, 1, 2, 3
FORM_FACTORISED_SIMPLE_F32C = 4


class SwbProblem(C.Structure):
    _fields_ = [
        ("shape", C.c_int32 * 3), ("spacing", C.c_float * 3), ("space_order", C.c_int32),
        ("dt", C.c_float), ("m", C.POINTER(C.c_float)), ("damp", C.POINTER(C.c_float)),
        ("weights", C.POINTER(C.c_float)), ("has_source", C.c_int32), ("source", C.c_int32 * 3),
        ("wavelet", C.POINTER(C.c_float)), ("wavelet_len", C.c_int32),
        ("n_receivers", C.c_int32), ("receivers", C.POINTER(C.c_int32)), ("form", C.c_int32),
        ("time_block", C.c_int32), ("device", C.c_int32), ("slab_lo", C.c_int32),
        ("slab_hi", C.c_int32), ("n_coord_receivers", C.c_int32),
        ("coord_receivers", C.POINTER(C.c_double)), ("check_bounds", C.c_int32),
        ("velocity", C.POINTER(C.c_float)), ("damp_max", C.c_float), ("damp_width", C.c_int32),
    ]


class SwbStats(C.Structure):
    _fields_ = [("device_ms", C.c_double), ("point_updates", C.c_uint64),
                ("kernel_launches", C.c_uint64), ("kernel_variant", C.c_int32),
                ("launch_steps", C.c_int32), ("peer_lo", C.c_int32), ("peer_hi", C.c_int32),
                ("fused_lo", C.c_int32), ("fused_hi", C.c_int32), ("grid", C.c_int32)]


class CudaError(RuntimeError):
    """Device/driver failure (SWB_ECUDA)."""


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a). There is no CPU fallback for the operator.")
    lib = C.CDLL(LIB_PATH)
    P = C.POINTER
    fp = P(C.c_float)
    h = C.c_void_p
    sig = {
        "swb_create": (C.c_int, [P(SwbProblem), P(h)]),
        "swb_set_level": (C.c_int, [h, C.c_int, fp]),
        "swb_get_level": (C.c_int, [h, C.c_int, fp]),
        "swb_get_level_padded": (C.c_int, [h, C.c_int, fp, C.c_int]),
        "swb_apply": (C.c_int, [h, C.c_int, C.c_int, fp, P(C.c_int32), fp]),
        "swb_apply_async": (C.c_int, [h, C.c_int, C.c_int]),
        "swb_apply_adjoint": (C.c_int, [h, C.c_int, fp, fp, fp, P(C.c_int32)]),
        "swb_apply_snapshots": (C.c_int, [h, C.c_int, C.c_int, C.c_int, P(fp), C.c_int, fp, P(C.c_int32), fp]),
        "swb_collect": (C.c_int, [h, fp, P(C.c_int32), fp]),
        "swb_stream": (C.c_void_p, [h]),
        "swb_get_stats": (C.c_int, [h, P(SwbStats)]),
        "swb_destroy": (C.c_int, [h]),
        "swb_last_error": (C.c_char_p, []),
        "swb_export_ghosts": (C.c_int, [h, C.c_void_p, P(C.c_size_t)]),
        "swb_link_neighbours": (C.c_int, [h, C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t]),
        "swb_link_local": (C.c_int, [h, h]),
        "swb_fd_weights": (C.c_int, [C.c_int, C.c_int, P(C.c_int64), P(C.c_int64)]),
        "swb_cfl_dt": (C.c_double, [C.c_int, P(C.c_double), C.c_double, C.c_int]),
        "swb_ricker_wavelet": (C.c_int, [C.c_double, C.c_double, C.c_int, fp]),
        "swb_m_data": (C.c_int, [fp, C.c_size_t, fp]),
        "swb_damp_data": (C.c_int, [P(C.c_int32), C.c_float, C.c_int, fp]),
        "swb_version": (C.c_char_p, []),
        "swb_debug_trace": (C.c_int, [h, P(C.c_uint64), C.c_int]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()

# C-ABI entry points declared in include/swb.h (checked by tests/test_capi.py::test_header_symbols_exported).
EXPORTED = ["swb_create", "swb_set_level", "swb_get_level", "swb_get_level_padded", "swb_apply", "swb_apply_async", "swb_apply_adjoint",
            "swb_apply_snapshots",
            "swb_collect", "swb_stream", "swb_get_stats", "swb_destroy", "swb_last_error",
            "swb_export_ghosts", "swb_link_neighbours", "swb_link_local", "swb_fd_weights",
            "swb_cfl_dt", "swb_ricker_wavelet", "swb_m_data", "swb_damp_data", "swb_version",
            "swb_debug_trace"]


def last_error() -> str:
    return lib.swb_last_error().decode()


def fptr(a):
    """float* of a C-contiguous float32 numpy array (None -> NULL)."""
    if a is None:
        return C.POINTER(C.c_float)()
    return a.ctypes.data_as(C.POINTER(C.c_float))
