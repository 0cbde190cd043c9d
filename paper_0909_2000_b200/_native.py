"""ctypes binding of the C ABI in include/alignplot_b200.h.

The shared library is built in-tree (``make`` or ``__graft_entry__.build()``)
as ``paper_0909_2000_b200/libalignplot_b200.so``.  There is no fallback: if the
library is missing, importing the engine raises; if no CUDA device is present,
every compute call returns AP_NODEV and the Python layer raises
``NoDeviceError``.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_float, c_int, c_int32, c_size_t, c_uint16, c_uint32, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
# AP_LIB_PATH: load another build of the same engine (tuning experiments, tools/exp/)
LIB_PATH = os.environ.get("AP_LIB_PATH") or os.path.join(_HERE, "libalignplot_b200.so")

AP_OK, AP_CONFIG, AP_EMPTY, AP_INVALID, AP_CUDA, AP_NODEV, AP_CAPACITY, AP_NOMEM = range(8)
AP_MAX_BLOWN_WINDOW = 65534   # sea16 bound (model.cpp:57-59)
AP_PACKED_WINDOW = 1024       # larger blown windows take the large-window kernels

# Every symbol declared in include/alignplot_b200.h (checked by tests/test_abi.py).
EXPORTS = (
    "ap_grid_dims", "ap_validate", "ap_plot_dense", "ap_plot_dense_u8", "ap_plot_threshold", "ap_plot_pgm",
    "ap_plot_threshold_cells", "ap_plot_threshold_into", "ap_plot_dense_i32", "ap_ctx_plot_dense_i32_device",
    "ap_last_error",
    "ap_device_count", "ap_ctx_create", "ap_ctx_destroy", "ap_ctx_plot_dense_device",
    "ap_ctx_plot_threshold_device", "ap_ctx_plot_pgm_device", "ap_ctx_plot_dense_u8_device",
    "ap_ctx_last_kernel_ms", "ap_ctx_last_launches", "ap_ctx_last_kernel",
)


class ApCell(ctypes.Structure):
    """ap_cell (include/alignplot_b200.h): one thresholded cell, PlotCell (scoring.hpp:33-42)."""
    _fields_ = [("row", c_uint32), ("col", c_uint32), ("half", c_int32)]


class ApConfig(ctypes.Structure):
    _fields_ = [
        ("window_w", c_uint64),
        ("step_h", c_uint64),
        ("blowup_r", c_uint32),
        ("has_threshold", c_int32),
        ("threshold_half", c_int32),
        ("n_devices", c_int32),
        ("row_begin", c_uint64),
        ("row_end", c_uint64),
    ]


# int (*ap_list_alloc_fn)(void* user, uint64_t count, uint32_t** rows, uint32_t** cols, int32_t** halves)
ListAllocFn = ctypes.CFUNCTYPE(c_int, c_void_p, c_uint64, POINTER(c_void_p), POINTER(c_void_p), POINTER(c_void_p))

_lib = None


def lib() -> ctypes.CDLL:
    """Load the engine library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA engine first (make, or __graft_entry__.build()); "
            "there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    u8p = POINTER(ctypes.c_uint8)
    L.ap_grid_dims.argtypes = [c_size_t, c_size_t, c_size_t, c_size_t, POINTER(c_size_t), POINTER(c_size_t)]
    L.ap_grid_dims.restype = c_int
    L.ap_validate.argtypes = [c_size_t, c_size_t, POINTER(ApConfig)]
    L.ap_validate.restype = c_int
    L.ap_plot_dense.argtypes = [c_void_p, c_size_t, c_void_p, c_size_t, POINTER(ApConfig), c_void_p]
    L.ap_plot_dense.restype = c_int
    L.ap_plot_threshold.argtypes = [c_void_p, c_size_t, c_void_p, c_size_t, POINTER(ApConfig),
                                    POINTER(c_uint64), c_void_p, c_void_p, c_void_p, c_size_t]
    L.ap_plot_threshold.restype = c_int
    L.ap_plot_threshold_cells.argtypes = [c_void_p, c_size_t, c_void_p, c_size_t, POINTER(ApConfig),
                                          POINTER(c_uint64), c_void_p, c_size_t]
    L.ap_plot_threshold_cells.restype = c_int
    L.ap_plot_threshold_into.argtypes = [c_void_p, c_size_t, c_void_p, c_size_t, POINTER(ApConfig), ListAllocFn,
                                         c_void_p, POINTER(c_uint64)]
    L.ap_plot_threshold_into.restype = c_int
    L.ap_plot_dense_i32.argtypes = [c_void_p, c_size_t, c_void_p, c_size_t, POINTER(ApConfig), c_void_p]
    L.ap_plot_dense_i32.restype = c_int
    L.ap_ctx_plot_dense_i32_device.argtypes = [c_void_p, c_void_p, c_size_t, c_void_p, c_size_t,
                                               POINTER(ApConfig), c_void_p, c_void_p]
    L.ap_ctx_plot_dense_i32_device.restype = c_int
    L.ap_plot_dense_u8.argtypes = [c_void_p, c_size_t, c_void_p, c_size_t, POINTER(ApConfig), c_void_p]
    L.ap_plot_dense_u8.restype = c_int
    L.ap_ctx_plot_dense_u8_device.argtypes = [c_void_p, c_void_p, c_size_t, c_void_p, c_size_t,
                                              POINTER(ApConfig), c_void_p, c_void_p]
    L.ap_ctx_plot_dense_u8_device.restype = c_int
    L.ap_plot_pgm.argtypes = [c_void_p, c_size_t, c_void_p, c_size_t, POINTER(ApConfig), c_void_p]
    L.ap_plot_pgm.restype = c_int
    L.ap_ctx_plot_pgm_device.argtypes = [c_void_p, c_void_p, c_size_t, c_void_p, c_size_t, POINTER(ApConfig),
                                         c_void_p, c_void_p]
    L.ap_ctx_plot_pgm_device.restype = c_int
    L.ap_last_error.argtypes = []
    L.ap_last_error.restype = c_char_p
    L.ap_device_count.argtypes = []
    L.ap_device_count.restype = c_int
    L.ap_ctx_create.argtypes = [c_int, POINTER(c_void_p)]
    L.ap_ctx_create.restype = c_int
    L.ap_ctx_destroy.argtypes = [c_void_p]
    L.ap_ctx_destroy.restype = c_int
    L.ap_ctx_plot_dense_device.argtypes = [c_void_p, c_void_p, c_size_t, c_void_p, c_size_t,
                                           POINTER(ApConfig), c_void_p, c_void_p]
    L.ap_ctx_plot_dense_device.restype = c_int
    L.ap_ctx_plot_threshold_device.argtypes = [c_void_p, c_void_p, c_size_t, c_void_p, c_size_t,
                                               POINTER(ApConfig), POINTER(c_uint64), c_void_p,
                                               c_void_p, c_void_p, c_size_t, c_void_p]
    L.ap_ctx_plot_threshold_device.restype = c_int
    L.ap_ctx_last_kernel_ms.argtypes = [c_void_p]
    L.ap_ctx_last_kernel_ms.restype = c_float
    L.ap_ctx_last_launches.argtypes = [c_void_p]
    L.ap_ctx_last_launches.restype = c_int
    L.ap_ctx_last_kernel.argtypes = [c_void_p]
    L.ap_ctx_last_kernel.restype = c_char_p
    _lib = L
    return L


def last_error() -> str:
    return lib().ap_last_error().decode("utf-8", "replace")
