"""Python mirror of the reference's exact-OSBF interface, over libosbf_gpu.so.

The reference API (namespace ``osbf``, /root/reference/proj/include/osbf/) is
C++; the drop-in C++ headers live in ``include/osbf/``.  This module exposes
the same operations to Python with the same names, argument meaning and
error behaviour, for tests, the benchmark and Python callers:

=====================================  =============================================
reference                              here
=====================================  =============================================
``sub_windows(r)`` core.hpp:212        :func:`sub_windows`
``FilterVariant`` / ``FilterConfig``   :class:`FilterVariant` / :class:`FilterConfig`
 core.hpp:227-254
``build_sat`` integral.hpp:77          :func:`build_sat` (GPU, bit-identical table)
``subwindow_means`` filters2d.hpp:26   :func:`subwindow_means` (all pixels at once)
``osbf_step`` filters2d.hpp:61         :func:`osbf_step`
``osbf`` filters2d.hpp:91              :func:`osbf`
``fast_osbf`` filters2d.hpp:105        :func:`fast_osbf` (paper Algorithm 3, bit-identical)
``box_filter`` filters2d.hpp:38        :func:`box_filter` (bit-identical)
``osbf_3d`` / ``box_filter_3d``        :func:`osbf_3d` / :func:`box_filter_3d` (bit-identical)
 filters3d.hpp:55-114
``filter_multichannel`` :371           :func:`filter_multichannel` (OsbfExact, OsbfFast, Box)
``set_max_threads`` parallel.hpp:20    :func:`set_max_threads` (no-op: the GPU
                                        result does not depend on any launch knob)
=====================================  =============================================

Inputs may be numpy arrays (host path: the C ABI copies in and out) or
CUDA torch tensors (device path: no host round trip, caller's stream).
Exceptions: ``InvalidArgument`` (std::invalid_argument), ``DomainError``
(std::domain_error), ``OutOfRange`` (std::out_of_range), ``CudaError``.
"""
from __future__ import annotations

import ctypes
import enum
import threading
from dataclasses import dataclass

import numpy as np

from . import _native as N


class OsbfError(RuntimeError):
    """Base class; ``status`` is the osbf_status code."""

    status = -1


class InvalidArgument(OsbfError, ValueError):
    status = N.OSBF_ERR_INVALID_ARGUMENT


class DomainError(OsbfError, ArithmeticError):
    status = N.OSBF_ERR_DOMAIN


class OutOfRange(OsbfError, IndexError):
    status = N.OSBF_ERR_OUT_OF_RANGE


class CudaError(OsbfError):
    status = N.OSBF_ERR_CUDA


class NoDevice(OsbfError):
    status = N.OSBF_ERR_NO_DEVICE


class AllocError(CudaError):
    status = N.OSBF_ERR_ALLOC


_ERRORS = {c.status: c for c in (InvalidArgument, DomainError, OutOfRange, CudaError, NoDevice,
                                 AllocError)}


def _check(st: int) -> None:
    if st != N.OSBF_OK:
        msg = N.lib().osbf_gpu_last_error().decode(errors="replace")
        raise _ERRORS.get(st, OsbfError)(msg)


def _mode_code(mode) -> int:
    if isinstance(mode, int):
        return mode
    try:
        return N.MODES[mode]
    except KeyError:
        raise InvalidArgument(f"unknown mode {mode!r}") from None


# ---------------------------------------------------------------------------
# reference value types (core.hpp)


@dataclass(frozen=True)
class SubWindowId:
    """One-sided sub-window, core.hpp:201-205: u = column offsets, v = row offsets."""

    id: int
    u0: int
    u1: int
    v0: int
    v1: int


def sub_windows(r: int) -> list[SubWindowId]:
    """The eight windows in selection (tie-break) order, core.hpp:212-225."""
    if r < 1:
        raise InvalidArgument("sub_windows: radius must be >= 1")
    return [SubWindowId(1, -r, 0, 0, r), SubWindowId(2, 0, r, 0, r), SubWindowId(3, 0, r, -r, 0),
            SubWindowId(4, -r, 0, -r, 0), SubWindowId(5, -r, 0, -r, r), SubWindowId(6, 0, r, -r, r),
            SubWindowId(7, -r, r, 0, r), SubWindowId(8, -r, r, -r, 0)]


class FilterVariant(enum.Enum):
    """core.hpp:227-233.  Only OsbfExact is on this library's path."""

    Box = 0
    OsbfExact = 1
    OsbfFast = 2
    OneSidedGeneric = 3
    Gaussian = 4


@dataclass
class FilterConfig:
    """core.hpp:238-254 (defaults r=2, iterations=10, OsbfExact, sigma=3)."""

    radius: int = 2
    iterations: int = 10
    variant: FilterVariant = FilterVariant.OsbfExact
    sigma: float = 3.0

    def validate(self) -> None:
        if self.radius < 1:
            raise InvalidArgument("FilterConfig: radius must be >= 1")
        if self.iterations < 0:
            raise InvalidArgument("FilterConfig: iterations must be >= 0")
        if self.variant in (FilterVariant.OneSidedGeneric, FilterVariant.Gaussian) and \
                not self.sigma > 0.0:
            raise InvalidArgument("FilterConfig: sigma must be > 0")


def set_max_threads(n: int) -> None:
    """parallel.hpp:20 — accepted for API compatibility; GPU results are
    identical for any launch configuration, so there is nothing to cap."""


def max_threads() -> int:
    return 1


# ---------------------------------------------------------------------------
# contexts


class Context:
    """Owns an ``osbf_ctx`` (device scratch + stream) on one GPU."""

    def __init__(self, device: int = 0):
        self._lib = N.lib()
        h = ctypes.c_void_p()
        _check(self._lib.osbf_gpu_ctx_create(device, ctypes.byref(h)))
        self.handle = h
        self.device = device

    def close(self) -> None:
        if getattr(self, "handle", None):
            self._lib.osbf_gpu_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(self._lib.osbf_gpu_ctx_launch_count(self.handle))

    @staticmethod
    def set_fast_kernel(name: str | None) -> None:
        """Diagnostics: force the fast-pass kernel family process-wide
        (osbf_gpu_set_fast_kernel): "walk", "tma", "stream", "strip", "tile", "sep",
        or None for the per-radius default."""
        _check(N.lib().osbf_gpu_set_fast_kernel((name or "").encode()))

    @staticmethod
    def set_exact_kernel(name: str | None) -> None:
        """Diagnostics: force the exact-pass kernel family process-wide
        (osbf_gpu_set_exact_kernel): "strip", "gwalk", "twalk", "stencil", or
        None for the default (table path + generic walk).  All bit-identical."""
        _check(N.lib().osbf_gpu_set_exact_kernel((name or "").encode()))

    @staticmethod
    def fast_max_radius() -> int:
        """Largest radius with a fast kernel (osbf_gpu_fast_max_radius):
        16 templated radii, then the generic vertical-first walk."""
        return int(N.lib().osbf_gpu_fast_max_radius())

    @property
    def last_kernel(self) -> str:
        """Kernel family of the last pass issued from this thread
        (osbf_gpu_last_kernel), e.g. ``fast_strip``."""
        return self._lib.osbf_gpu_last_kernel().decode()

    def set_temporal_blocking(self, passes_per_launch: int) -> None:
        """Fast mode temporal blocking: k = 2..4 passes per launch over tiles
        with a k*r halo (radius <= 4); 1 = one pass per launch (default)."""
        _check(self._lib.osbf_gpu_ctx_set_temporal_blocking(self.handle, passes_per_launch))

    # -- device tensors -----------------------------------------------------
    def iterate(self, src, radius: int, iterations: int, mode="exact", out=None, stream=None):
        """osbf over a CUDA tensor of shape (H, W) or (B, H, W), dtype uint8 /
        float32 / float64.  Returns (or fills) a float64 tensor of that shape."""
        import torch

        x, batch, h, w = _as_batch(src)
        if out is None:
            out = torch.empty((batch, h, w), dtype=torch.float64, device=x.device)
            ret = out.view(src.shape)
        else:
            ret = out
            out = _check_out(out, x, (batch, h, w))
        if stream is None:
            stream = torch.cuda.current_stream(x.device).cuda_stream
        _check(self._lib.osbf_gpu_iterate(
            self.handle, _dtype_code(x), ctypes.c_void_p(x.data_ptr()), x.stride(1), x.stride(0),
            ctypes.c_void_p(out.data_ptr()), out.stride(1), out.stride(0), w, h, batch, radius,
            iterations, _mode_code(mode), ctypes.c_void_p(stream)))
        return ret

    def fast_osbf(self, src, radius: int, iterations: int, out=None, stream=None):
        """Paper Algorithm 3 (filters2d.hpp:105-154) over a CUDA tensor of shape
        (H, W) or (B, H, W); bit-identical to the reference's fast_osbf."""
        return self._sat_filter("osbf_gpu_fast_osbf", src, radius, iterations, out, stream)

    def box_filter(self, src, radius: int, iterations: int, out=None, stream=None):
        """The classical box filter (filters2d.hpp:38-56) over a CUDA tensor;
        bit-identical to the reference's box_filter."""
        return self._sat_filter("osbf_gpu_box_filter", src, radius, iterations, out, stream)

    def osbf_3d(self, vol, radius: int, iterations: int, out=None, stream=None):
        """filters3d.hpp:78-114 on a CUDA float64 volume (D, H, W); bit-identical."""
        return self._filter3d("osbf_gpu_osbf_3d", vol, radius, iterations, out, stream)

    def box_filter_3d(self, vol, radius: int, iterations: int, out=None, stream=None):
        """filters3d.hpp:55-76 on a CUDA float64 volume (D, H, W); bit-identical."""
        return self._filter3d("osbf_gpu_box_filter_3d", vol, radius, iterations, out, stream)

    def _filter3d(self, fn, vol, radius, iterations, out, stream):
        import torch

        if vol.dim() != 3 or vol.dtype != torch.float64 or not vol.is_contiguous():
            raise InvalidArgument("expected a contiguous float64 (D, H, W) volume")
        d, h, w = vol.shape
        if out is None:
            out = torch.empty_like(vol)
        else:
            out = _check_out(out, vol, (d, h, w))
            if not out.is_contiguous():
                raise InvalidArgument("out volume must be contiguous")
        if stream is None:
            stream = torch.cuda.current_stream(vol.device).cuda_stream
        _check(getattr(self._lib, fn)(self.handle, ctypes.c_void_p(vol.data_ptr()),
                                      ctypes.c_void_p(out.data_ptr()), w, h, d, radius,
                                      iterations, ctypes.c_void_p(stream)))
        return out

    def filter3d_host(self, vol: np.ndarray, radius: int, iterations: int, osbf3=True):
        v = np.ascontiguousarray(vol, dtype=np.float64)
        if v.ndim != 3:
            raise InvalidArgument("expected a (D, H, W) volume")
        d, h, w = v.shape
        out = np.empty_like(v)
        fn = self._lib.osbf_gpu_osbf_3d_host if osbf3 else self._lib.osbf_gpu_box_filter_3d_host
        _check(fn(self.handle, ctypes.c_void_p(v.ctypes.data), ctypes.c_void_p(out.ctypes.data),
                  w, h, d, radius, iterations))
        return out

    def svt_host(self, vol: np.ndarray) -> np.ndarray:
        """Summed-volume table (integral.hpp:98-112 order) of a (D, H, W) host
        volume, built on the GPU; shape (D+1, H+1, W+1) with zero border slabs."""
        v = np.ascontiguousarray(vol, dtype=np.float64)
        if v.ndim != 3:
            raise InvalidArgument("expected a (D, H, W) volume")
        d, h, w = v.shape
        out = np.empty((d + 1, h + 1, w + 1), dtype=np.float64)
        _check(self._lib.osbf_gpu_svt_host(self.handle, ctypes.c_void_p(v.ctypes.data), w, h, d,
                                           ctypes.c_void_p(out.ctypes.data)))
        return out

    def _sat_filter(self, fn, src, radius, iterations, out, stream):
        import torch

        x, batch, h, w = _as_batch(src)
        if out is None:
            out = torch.empty((batch, h, w), dtype=torch.float64, device=x.device)
            ret = out.view(src.shape)
        else:
            ret = out
            out = _check_out(out, x, (batch, h, w))
        if stream is None:
            stream = torch.cuda.current_stream(x.device).cuda_stream
        _check(getattr(self._lib, fn)(
            self.handle, _dtype_code(x), ctypes.c_void_p(x.data_ptr()), x.stride(1), x.stride(0),
            ctypes.c_void_p(out.data_ptr()), out.stride(1), out.stride(0), w, h, batch, radius,
            iterations, ctypes.c_void_p(stream)))
        return ret

    def subwindow_means(self, src, radius: int, mode="exact", stream=None):
        """All-pixel subwindow_means (filters2d.hpp:26-34) and the selection map."""
        import torch

        x, batch, h, w = _as_batch(src)
        means = torch.empty((batch, h, w, 8), dtype=torch.float64, device=x.device)
        sel = torch.empty((batch, h, w), dtype=torch.uint8, device=x.device)
        if stream is None:
            stream = torch.cuda.current_stream(x.device).cuda_stream
        _check(self._lib.osbf_gpu_subwindow_means(
            self.handle, _dtype_code(x), ctypes.c_void_p(x.data_ptr()), x.stride(1), x.stride(0),
            w, h, batch, radius, ctypes.c_void_p(means.data_ptr()), ctypes.c_void_p(sel.data_ptr()),
            _mode_code(mode), ctypes.c_void_p(stream)))
        shape = tuple(src.shape)
        return means.view(*shape, 8), sel.view(shape)

    def sat(self, src, stream=None):
        import torch

        x, batch, h, w = _as_batch(src)
        c = torch.empty((batch, h + 1, w + 1), dtype=torch.float64, device=x.device)
        if stream is None:
            stream = torch.cuda.current_stream(x.device).cuda_stream
        _check(self._lib.osbf_gpu_sat(
            self.handle, _dtype_code(x), ctypes.c_void_p(x.data_ptr()), x.stride(1), x.stride(0),
            w, h, batch, ctypes.c_void_p(c.data_ptr()), ctypes.c_void_p(stream)))
        return c.view(*src.shape[:-2], h + 1, w + 1)

    def step_band(self, src, in_row0: int, out, out_row0: int, out_rows: int,
                  image_height: int, radius: int, mode="fast", stream=None,
                  push_up=None, push_down=None, push_rows: int = 0):
        """One fast pass over a row band (osbf_gpu_step_band).  ``src``: CUDA
        tensor (in_rows, W) holding global rows [in_row0, in_row0+in_rows);
        ``out``: fp64 CUDA tensor whose rows receive global rows
        [out_row0, out_row0 + out_rows).  ``push_up`` / ``push_down``: fp64
        (push_rows, W) views of the neighbours' halo rows (local or peer
        memory) that the pass also writes its first / last ``push_rows`` rows
        into (osbf_gpu_step_band_push: the halo exchange fused into the pass)."""
        import torch

        if src.dim() != 2 or out.dim() != 2 or src.stride(1) != 1 or out.stride(1) != 1:
            raise InvalidArgument("step_band expects 2-D row-major tensors")
        if out.dtype != torch.float64:
            raise InvalidArgument("band output must be float64")
        if out.device != src.device:
            raise InvalidArgument("band output must be on the input's device")
        if out.shape[0] < out_rows or out.shape[1] != src.shape[1]:
            raise InvalidArgument("band output must hold out_rows rows of the input's width")
        if in_row0 > out_row0 or in_row0 + src.shape[0] < out_row0 + out_rows:
            raise InvalidArgument("band input rows must cover the output rows")
        if stream is None:
            stream = torch.cuda.current_stream(src.device).cuda_stream
        pitch = 0
        for t in (push_up, push_down):
            if t is not None:
                if t.dtype != torch.float64 or t.dim() != 2 or t.stride(1) != 1:
                    raise InvalidArgument("push targets must be 2-D row-major float64")
                if t.shape[0] < push_rows or t.shape[1] < src.shape[1]:
                    raise InvalidArgument("push target smaller than push_rows x width")
                if pitch and t.stride(0) != pitch:
                    raise InvalidArgument("push targets must share one row pitch")
                pitch = t.stride(0)
        _check(self._lib.osbf_gpu_step_band_push(
            self.handle, _dtype_code(src), ctypes.c_void_p(src.data_ptr()), src.stride(0), in_row0,
            src.shape[0], ctypes.c_void_p(out.data_ptr()), out.stride(0), out_row0, out_rows,
            src.shape[1], image_height, radius, _mode_code(mode),
            ctypes.c_void_p(push_up.data_ptr() if push_up is not None else 0),
            ctypes.c_void_p(push_down.data_ptr() if push_down is not None else 0),
            push_rows if pitch else 0, pitch, ctypes.c_void_p(stream)))
        return out

    # -- host arrays (the drop-in path: H2D, filter, D2H inside the call) ----
    def osbf_host(self, planes: np.ndarray, radius: int, iterations: int, mode="exact",
                  out: np.ndarray | None = None) -> np.ndarray:
        p = np.ascontiguousarray(planes)
        code = {np.dtype(np.uint8): 0, np.dtype(np.float32): 1, np.dtype(np.float64): 2}.get(p.dtype)
        if code is None:
            p = p.astype(np.float64)
            code = 2
        if p.ndim == 2:
            batch, (h, w) = 1, p.shape
        elif p.ndim == 3:
            batch, h, w = p.shape
        else:
            raise InvalidArgument("expected a (H, W) or (B, H, W) array")
        if out is None:
            out = np.empty(p.shape, dtype=np.float64)
        _check(self._lib.osbf_gpu_osbf_host(
            self.handle, code, ctypes.c_void_p(p.ctypes.data), ctypes.c_void_p(out.ctypes.data),
            w, h, batch, radius, iterations, _mode_code(mode)))
        return out

    def box_filter_host(self, planes: np.ndarray, radius: int, iterations: int) -> np.ndarray:
        """box_filter on host arrays (H, W) or (B, H, W)."""
        return self._sat_filter_host("osbf_gpu_box_filter_host", planes, radius, iterations)

    def fast_osbf_host(self, planes: np.ndarray, radius: int, iterations: int) -> np.ndarray:
        """fast_osbf on host arrays (H, W) or (B, H, W): copy in, filter, copy out."""
        return self._sat_filter_host("osbf_gpu_fast_osbf_host", planes, radius, iterations)

    def _sat_filter_host(self, fn, planes, radius, iterations):
        p = np.ascontiguousarray(planes)
        code = {np.dtype(np.uint8): 0, np.dtype(np.float32): 1, np.dtype(np.float64): 2}.get(p.dtype)
        if code is None:
            p = p.astype(np.float64)
            code = 2
        if p.ndim not in (2, 3):
            raise InvalidArgument("expected a (H, W) or (B, H, W) array")
        batch = 1 if p.ndim == 2 else p.shape[0]
        h, w = p.shape[-2:]
        out = np.empty(p.shape, dtype=np.float64)
        _check(getattr(self._lib, fn)(
            self.handle, code, ctypes.c_void_p(p.ctypes.data), ctypes.c_void_p(out.ctypes.data),
            w, h, batch, radius, iterations))
        return out

    def osbf_step_host(self, plane: np.ndarray, radius: int, mode="exact") -> np.ndarray:
        p = np.ascontiguousarray(plane, dtype=np.float64)
        if p.ndim != 2:
            raise InvalidArgument("expected a (H, W) plane")
        h, w = p.shape
        out = np.empty_like(p)
        _check(self._lib.osbf_gpu_osbf_step_host(
            self.handle, ctypes.c_void_p(p.ctypes.data), ctypes.c_void_p(out.ctypes.data), w, h,
            radius, _mode_code(mode)))
        return out

    def filter_multichannel_host(self, channels, radius: int, iterations: int, mode="exact",
                                 outs=None, variant: "FilterVariant | None" = None):
        chans = [np.ascontiguousarray(c, dtype=np.float64) for c in channels]
        if not chans:
            raise InvalidArgument("MultiChannelImage: channel count must be in [1,4]")
        h, w = chans[0].shape
        for c in chans:
            if c.shape != (h, w):
                raise InvalidArgument("MultiChannelImage: channel dimensions differ")
        if outs is None:
            outs = [np.empty((h, w), dtype=np.float64) for _ in chans]
        ins = (ctypes.c_void_p * len(chans))(*[c.ctypes.data for c in chans])
        ous = (ctypes.c_void_p * len(chans))(*[o.ctypes.data for o in outs])
        if variant is FilterVariant.OsbfFast:
            _check(self._lib.osbf_gpu_filter_multichannel_fast_host(
                self.handle, ins, ous, len(chans), w, h, radius, iterations))
        elif variant is FilterVariant.Box:
            _check(self._lib.osbf_gpu_filter_multichannel_box_host(
                self.handle, ins, ous, len(chans), w, h, radius, iterations))
        else:
            _check(self._lib.osbf_gpu_filter_multichannel_host(
                self.handle, ins, ous, len(chans), w, h, radius, iterations, _mode_code(mode)))
        return outs

    def smooth_raster(self, raster: np.ndarray, filter: str = "osbf", radius: int = 2,
                      iterations: int = 10, out_bits: int = 8, mode="exact") -> np.ndarray:
        """The `osbf smooth` edge (tools/osbf_main.cpp:63-83): decoded PGM/PPM
        samples, (H, W) or (H, W, 3) uint8/uint16, promoted, filtered with
        "osbf" / "fast-osbf" / "box" and quantised (io.hpp:108-115) to
        out_bits 8 or 16 — promotion and quantisation on the GPU."""
        if filter not in _SMOOTH_FILTERS:
            raise InvalidArgument(f"unknown filter: {filter}")
        r = np.ascontiguousarray(raster)
        if r.dtype not in (np.uint8, np.uint16):
            raise InvalidArgument("raster samples must be uint8 or uint16")
        if r.ndim == 2:
            h, w, c = r.shape[0], r.shape[1], 1
        elif r.ndim == 3:
            h, w, c = r.shape
        else:
            raise InvalidArgument("expected an (H, W) or (H, W, C) raster")
        if out_bits not in (8, 16):
            raise InvalidArgument("write_image: bit depth must be 8 or 16")
        out = np.empty(r.shape, dtype=np.uint8 if out_bits == 8 else np.uint16)
        _check(self._lib.osbf_gpu_smooth_raster_host(
            self.handle, ctypes.c_void_p(r.ctypes.data), r.dtype.itemsize, c, w, h,
            _SMOOTH_FILTERS[filter], radius, iterations, _mode_code(mode),
            ctypes.c_void_p(out.ctypes.data), out.dtype.itemsize))
        return out

    def sat_host(self, plane: np.ndarray) -> np.ndarray:
        p = np.ascontiguousarray(plane, dtype=np.float64)
        h, w = p.shape
        c = np.empty((h + 1, w + 1), dtype=np.float64)
        _check(self._lib.osbf_gpu_sat_host(self.handle, ctypes.c_void_p(p.ctypes.data), w, h,
                                           ctypes.c_void_p(c.ctypes.data)))
        return c


def _dtype_code(t) -> int:
    import torch

    code = {torch.uint8: 0, torch.float32: 1, torch.float64: 2}.get(t.dtype)
    if code is None:
        raise InvalidArgument(f"unsupported dtype {t.dtype}")
    return code


def _check_out(out, like, shape):
    """A caller-supplied output: float64, on the input's device, of the
    expected shape (any leading view of it), rows contiguous."""
    import torch

    if out.dtype != torch.float64:
        raise InvalidArgument("out must be float64")
    if not out.is_cuda or out.device != like.device:
        raise InvalidArgument("out must be a CUDA tensor on the input's device")
    if out.numel() != int(np.prod(shape)) or tuple(out.shape)[-2:] != tuple(shape)[-2:]:
        raise InvalidArgument(f"out has shape {tuple(out.shape)}, expected {tuple(shape)}")
    if out.stride(-1) != 1:
        raise InvalidArgument("out rows must be contiguous (stride(-1) == 1)")
    if out.dim() == 3 and out.stride(0) < out.shape[1] * out.stride(1):
        raise InvalidArgument("out planes overlap")
    v = out.view(*shape) if out.dim() != len(shape) else out
    return v


def _as_batch(src):
    if not getattr(src, "is_cuda", False):
        raise InvalidArgument("expected a CUDA tensor (use the *_host methods for host arrays)")
    if src.dim() == 2:
        x = src.unsqueeze(0)
    elif src.dim() == 3:
        x = src
    else:
        raise InvalidArgument("expected a (H, W) or (B, H, W) tensor")
    if x.stride(2) != 1:
        x = x.contiguous()
    b, h, w = x.shape
    if h < 1 or w < 1:
        raise InvalidArgument("ImagePlane: dimensions must be >= 1")
    return x, b, h, w


_default = threading.local()


def default_context(device: int = 0) -> Context:
    ctxs = getattr(_default, "ctxs", None)
    if ctxs is None:
        ctxs = _default.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


# ---------------------------------------------------------------------------
# reference free functions


def _is_tensor(x) -> bool:
    return hasattr(x, "is_cuda") and hasattr(x, "data_ptr")


def osbf(plane, r: int, iterations: int, mode="exact"):
    """filters2d.hpp:91-98 — ``iterations`` Jacobi passes of osbf_step.

    ``iterations < 0`` raises InvalidArgument; ``iterations == 0`` returns a
    copy without checking ``r`` (the reference's behaviour)."""
    if _is_tensor(plane):
        return default_context(plane.device.index or 0).iterate(plane, r, iterations, mode)
    return default_context().osbf_host(np.asarray(plane), r, iterations, mode)


def osbf_step(plane, r: int, mode="exact"):
    """filters2d.hpp:61-88 — one pass; always validates ``r``."""
    if r < 1:
        raise InvalidArgument("osbf_step: radius must be >= 1")
    return osbf(plane, r, 1, mode)


def fast_osbf(plane, r: int, iterations: int):
    """filters2d.hpp:105-154 — paper Algorithm 3, bit-identical.  ``r < 1`` or
    ``iterations < 0`` raise InvalidArgument (the radius even for 0 iterations)."""
    if _is_tensor(plane):
        return default_context(plane.device.index or 0).fast_osbf(plane, r, iterations)
    return default_context().fast_osbf_host(np.asarray(plane), r, iterations)


def box_filter(plane, r: int, iterations: int):
    """filters2d.hpp:38-56 — the classical box filter, bit-identical.  ``r < 1``
    or ``iterations < 0`` raise InvalidArgument (the radius even for 0
    iterations)."""
    if _is_tensor(plane):
        return default_context(plane.device.index or 0).box_filter(plane, r, iterations)
    return default_context().box_filter_host(np.asarray(plane), r, iterations)


def osbf_3d(vol, r: int, iterations: int):
    """filters3d.hpp:78-114 — 14 one-sided regions, bit-identical; numpy or
    CUDA float64 volume of shape (D, H, W)."""
    if _is_tensor(vol):
        return default_context(vol.device.index or 0).osbf_3d(vol, r, iterations)
    return default_context().filter3d_host(np.asarray(vol), r, iterations, osbf3=True)


def box_filter_3d(vol, r: int, iterations: int):
    """filters3d.hpp:55-76 — bit-identical; numpy or CUDA float64 (D, H, W)."""
    if _is_tensor(vol):
        return default_context(vol.device.index or 0).box_filter_3d(vol, r, iterations)
    return default_context().filter3d_host(np.asarray(vol), r, iterations, osbf3=False)


def filter_multichannel(channels, config: FilterConfig, mode="exact"):
    """filters2d.hpp:371-400, OsbfExact / OsbfFast / Box branches: channels
    filtered independently (one batched launch per pass)."""
    config.validate()
    if config.variant not in (FilterVariant.OsbfExact, FilterVariant.OsbfFast,
                              FilterVariant.Box):
        raise InvalidArgument(
            f"filter_multichannel: variant {config.variant.name} is not on the GPU OSBF path")
    chans = list(channels) if not (hasattr(channels, "ndim") and channels.ndim == 3) else channels
    if len(chans) < 1 or len(chans) > 4:
        raise InvalidArgument("MultiChannelImage: channel count must be in [1,4]")
    if _is_tensor(chans) or (len(chans) and _is_tensor(chans[0])):
        import torch

        stack = chans if _is_tensor(chans) else torch.stack(list(chans))
        ctx = default_context(stack.device.index or 0)
        if config.variant is FilterVariant.OsbfFast:
            return ctx.fast_osbf(stack, config.radius, config.iterations)
        if config.variant is FilterVariant.Box:
            return ctx.box_filter(stack, config.radius, config.iterations)
        return ctx.iterate(stack, config.radius, config.iterations, mode)
    return default_context().filter_multichannel_host(chans, config.radius, config.iterations,
                                                      mode, variant=config.variant)


_SMOOTH_FILTERS = {"osbf": 0, "fast-osbf": 1, "box": 2}  # osbf_filter (osbf_gpu.h)


def smooth_raster(raster, filter: str = "osbf", radius: int = 2, iterations: int = 10,
                  out_bits: int = 8, mode="exact"):
    """tools/osbf_main.cpp:63-83 minus the file I/O: promote, filter_multichannel,
    quantise — see Context.smooth_raster."""
    return default_context().smooth_raster(raster, filter, radius, iterations, out_bits, mode)


def build_sat(plane):
    """integral.hpp:16-30 — the (H+1) x (W+1) summed-area table, built on the GPU."""
    if _is_tensor(plane):
        return default_context(plane.device.index or 0).sat(plane)
    return default_context().sat_host(np.asarray(plane))


def subwindow_means(plane, r: int, mode="exact"):
    """filters2d.hpp:26-34 at every pixel: returns (means[..., 8], selected_id)."""
    if r < 1:
        raise InvalidArgument("sub_windows: radius must be >= 1")
    if _is_tensor(plane):
        return default_context(plane.device.index or 0).subwindow_means(plane, r, mode)
    import torch

    t = torch.from_numpy(np.ascontiguousarray(plane)).cuda()
    m, s = default_context().subwindow_means(t, r, mode)
    return m.cpu().numpy(), s.cpu().numpy()
