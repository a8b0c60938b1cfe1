"""B200-native One-Sided Box Filter (arXiv 2108.05021) — drop-in for the
reference's OSBF path (osbf::osbf / osbf_step / fast_osbf / filter_multichannel).

The compute lives in ``libosbf_gpu.so`` (hand-written sm_100a CUDA behind the
C ABI in ``include/osbf_gpu.h``); this package is the Python host side.
"""
from ._native import build, lib  # noqa: F401
from .api import (  # noqa: F401
    AllocError,
    Context,
    CudaError,
    DomainError,
    FilterConfig,
    FilterVariant,
    InvalidArgument,
    NoDevice,
    OsbfError,
    OutOfRange,
    SubWindowId,
    box_filter,
    box_filter_3d,
    smooth_raster,
    build_sat,
    default_context,
    fast_osbf,
    filter_multichannel,
    max_threads,
    osbf,
    osbf_3d,
    osbf_step,
    set_max_threads,
    sub_windows,
    subwindow_means,
)

__all__ = [
    "build", "lib", "Context", "default_context", "osbf", "osbf_step", "fast_osbf", "box_filter",
    "osbf_3d", "box_filter_3d", "smooth_raster",
    "filter_multichannel",
    "build_sat", "subwindow_means", "sub_windows", "SubWindowId", "FilterConfig", "FilterVariant",
    "set_max_threads", "max_threads", "OsbfError", "InvalidArgument", "DomainError", "OutOfRange",
    "CudaError", "NoDevice", "AllocError",
]
