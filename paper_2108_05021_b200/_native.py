"""ctypes binding of libosbf_gpu.so (the C ABI declared in include/osbf_gpu.h).

The shared library is the product: hand-written sm_100a CUDA.  There is no
Python or CPU fallback — if the library is missing or no B200 is visible,
every compute call raises.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "libosbf_gpu.so")

OSBF_OK = 0
OSBF_ERR_INVALID_ARGUMENT = 1
OSBF_ERR_DOMAIN = 2
OSBF_ERR_OUT_OF_RANGE = 3
OSBF_ERR_CUDA = 4
OSBF_ERR_NO_DEVICE = 5
OSBF_ERR_ALLOC = 6

DTYPES = {"u8": 0, "f32": 1, "f64": 2}
MODES = {"exact": 0, "fast": 1}

_c_void_p = ctypes.c_void_p
_c_int = ctypes.c_int
_c_size = ctypes.c_size_t

# (name, restype, argtypes) for every symbol of include/osbf_gpu.h.
SIGNATURES = [
    ("osbf_gpu_abi_version", _c_int, []),
    ("osbf_gpu_last_error", ctypes.c_char_p, []),
    ("osbf_gpu_last_kernel", ctypes.c_char_p, []),
    ("osbf_gpu_fast_max_radius", _c_int, []),
    ("osbf_gpu_set_fast_kernel", _c_int, [ctypes.c_char_p]),
    ("osbf_gpu_set_exact_kernel", _c_int, [ctypes.c_char_p]),
    ("osbf_gpu_device_available", _c_int, []),
    ("osbf_gpu_ctx_create", _c_int, [_c_int, ctypes.POINTER(_c_void_p)]),
    ("osbf_gpu_ctx_destroy", _c_int, [_c_void_p]),
    ("osbf_gpu_ctx_trim", _c_int, [_c_void_p]),
    ("osbf_gpu_ctx_launch_count", ctypes.c_uint64, [_c_void_p]),
    ("osbf_gpu_ctx_set_temporal_blocking", _c_int, [_c_void_p, _c_int]),
    ("osbf_gpu_iterate", _c_int,
     [_c_void_p, _c_int, _c_void_p, _c_size, _c_size, _c_void_p, _c_size, _c_size,
      _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _c_void_p]),
    ("osbf_gpu_fast_osbf", _c_int,
     [_c_void_p, _c_int, _c_void_p, _c_size, _c_size, _c_void_p, _c_size, _c_size,
      _c_int, _c_int, _c_int, _c_int, _c_int, _c_void_p]),
    ("osbf_gpu_box_filter", _c_int,
     [_c_void_p, _c_int, _c_void_p, _c_size, _c_size, _c_void_p, _c_size, _c_size,
      _c_int, _c_int, _c_int, _c_int, _c_int, _c_void_p]),
    ("osbf_gpu_osbf_3d", _c_int,
     [_c_void_p, _c_void_p, _c_void_p, _c_int, _c_int, _c_int, _c_int, _c_int, _c_void_p]),
    ("osbf_gpu_box_filter_3d", _c_int,
     [_c_void_p, _c_void_p, _c_void_p, _c_int, _c_int, _c_int, _c_int, _c_int, _c_void_p]),
    ("osbf_gpu_subwindow_means", _c_int,
     [_c_void_p, _c_int, _c_void_p, _c_size, _c_size, _c_int, _c_int, _c_int, _c_int,
      _c_void_p, _c_void_p, _c_int, _c_void_p]),
    ("osbf_gpu_sat", _c_int,
     [_c_void_p, _c_int, _c_void_p, _c_size, _c_size, _c_int, _c_int, _c_int, _c_void_p,
      _c_void_p]),
    ("osbf_gpu_step_band", _c_int,
     [_c_void_p, _c_int, _c_void_p, _c_size, _c_int, _c_int, _c_void_p, _c_size, _c_int, _c_int,
      _c_int, _c_int, _c_int, _c_int, _c_void_p]),
    ("osbf_gpu_step_band_push", _c_int,
     [_c_void_p, _c_int, _c_void_p, _c_size, _c_int, _c_int, _c_void_p, _c_size, _c_int, _c_int,
      _c_int, _c_int, _c_int, _c_int, _c_void_p, _c_void_p, _c_int, _c_size, _c_void_p]),
    ("osbf_gpu_osbf_host", _c_int,
     [_c_void_p, _c_int, _c_void_p, _c_void_p, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int]),
    ("osbf_gpu_osbf_step_host", _c_int,
     [_c_void_p, _c_void_p, _c_void_p, _c_int, _c_int, _c_int, _c_int]),
    ("osbf_gpu_filter_multichannel_host", _c_int,
     [_c_void_p, ctypes.POINTER(_c_void_p), ctypes.POINTER(_c_void_p), _c_int, _c_int, _c_int,
      _c_int, _c_int, _c_int]),
    ("osbf_gpu_fast_osbf_host", _c_int,
     [_c_void_p, _c_int, _c_void_p, _c_void_p, _c_int, _c_int, _c_int, _c_int, _c_int]),
    ("osbf_gpu_osbf_3d_host", _c_int,
     [_c_void_p, _c_void_p, _c_void_p, _c_int, _c_int, _c_int, _c_int, _c_int]),
    ("osbf_gpu_box_filter_3d_host", _c_int,
     [_c_void_p, _c_void_p, _c_void_p, _c_int, _c_int, _c_int, _c_int, _c_int]),
    ("osbf_gpu_svt_host", _c_int, [_c_void_p, _c_void_p, _c_int, _c_int, _c_int, _c_void_p]),
    ("osbf_gpu_smooth_raster_host", _c_int,
     [_c_void_p, _c_void_p, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int,
      _c_void_p, _c_int]),
    ("osbf_gpu_box_filter_host", _c_int,
     [_c_void_p, _c_int, _c_void_p, _c_void_p, _c_int, _c_int, _c_int, _c_int, _c_int]),
    ("osbf_gpu_filter_multichannel_box_host", _c_int,
     [_c_void_p, ctypes.POINTER(_c_void_p), ctypes.POINTER(_c_void_p), _c_int, _c_int, _c_int,
      _c_int, _c_int]),
    ("osbf_gpu_filter_multichannel_fast_host", _c_int,
     [_c_void_p, ctypes.POINTER(_c_void_p), ctypes.POINTER(_c_void_p), _c_int, _c_int, _c_int,
      _c_int, _c_int]),
    ("osbf_gpu_sat_host", _c_int, [_c_void_p, _c_void_p, _c_int, _c_int, _c_void_p]),
]

_lib = None


def build(verbose: bool = False) -> None:
    """Compile libosbf_gpu.so in-tree (nvcc, sm_100a)."""
    cmd = ["make", "-C", PKG_DIR, "-j4"]
    if not verbose:
        cmd.insert(1, "-s")
    subprocess.run(cmd, check=True)


def lib() -> ctypes.CDLL:
    """Load libosbf_gpu.so (once).  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the OSBF CUDA library must be built "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    handle = ctypes.CDLL(LIB_PATH)
    for name, restype, argtypes in SIGNATURES:
        fn = getattr(handle, name)
        fn.restype = restype
        fn.argtypes = argtypes
    _lib = handle
    return handle
