"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU parity checkers.

* ``Oracle`` wraps ``oracle/liboracle.so`` — the plain-C restatement of the
  reference OSBF path (``osbf_oracle.c``; every function cites the reference
  file:line it follows).
* ``Reference`` wraps ``oracle/_ref/libosbf_ref.so`` — the unmodified
  reference headers (``/root/reference/proj/include``) compiled behind a C
  shim (``ref_shim.cpp``).  It is built here and travels to the GPU box as a
  prebuilt file; nothing reads ``/root/reference`` at run time.

Only ``tests/``, ``__graft_entry__.smoke()`` and the CPU-baseline legs of
``bench.py`` may import this package.  The product path never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libosbf_ref.so")

_dp = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)


def build() -> None:
    """Compile liboracle.so (+ _ref when the reference tree is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _ptr(a: np.ndarray, t=_dp):
    return a.ctypes.data_as(t)


def _as_f64(plane) -> np.ndarray:
    return np.ascontiguousarray(plane, dtype=np.float64)


class CheckerError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: status {status}")
        self.status = status


class Oracle:
    """The C restatement (osbf_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        lib = ctypes.CDLL(path)
        lib.oracle_osbf.argtypes = [_dp, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        lib.oracle_osbf_mt.argtypes = lib.oracle_osbf.argtypes + [ctypes.c_int]
        lib.oracle_osbf_step.argtypes = [_dp, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _u8p]
        lib.oracle_sat_build.argtypes = [_dp, ctypes.c_int, ctypes.c_int, _dp]
        lib.oracle_sat_build.restype = None
        lib.oracle_rect_sum.argtypes = [_dp] + [ctypes.c_int] * 6
        lib.oracle_rect_sum.restype = ctypes.c_double
        lib.oracle_rect_count.argtypes = [ctypes.c_int] * 6
        lib.oracle_rect_count.restype = ctypes.c_longlong
        lib.oracle_rect_mean.argtypes = [_dp] + [ctypes.c_int] * 6 + [_dp]
        lib.oracle_subwindow_means.argtypes = [_dp] + [ctypes.c_int] * 5 + [_dp]
        lib.oracle_sub_windows.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        lib.oracle_fast_osbf.argtypes = lib.oracle_osbf.argtypes
        lib.oracle_box_filter.argtypes = lib.oracle_osbf.argtypes
        lib.oracle_svt_build.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp]
        lib.oracle_svt_build.restype = None
        lib.oracle_osbf_3d.argtypes = [_dp, _dp] + [ctypes.c_int] * 5
        lib.oracle_box_filter_3d.argtypes = lib.oracle_osbf_3d.argtypes
        lib.oracle_quantize.argtypes = [ctypes.c_double, ctypes.c_int]
        lib.oracle_smooth_raster.argtypes = ([ctypes.c_void_p] + [ctypes.c_int] * 7 +
                                             [ctypes.c_void_p, ctypes.c_int])
        self.lib = lib

    def sub_windows(self, r: int):
        buf = (ctypes.c_int * 40)()
        st = self.lib.oracle_sub_windows(r, buf)
        if st:
            raise CheckerError(st, "sub_windows")
        return [tuple(buf[i * 5:(i + 1) * 5]) for i in range(8)]

    def osbf(self, plane, r: int, iterations: int, threads: int = 1) -> np.ndarray:
        p = _as_f64(plane)
        h, w = p.shape
        out = np.empty_like(p)
        st = self.lib.oracle_osbf_mt(_ptr(p), _ptr(out), w, h, r, iterations, threads)
        if st:
            raise CheckerError(st, "osbf")
        return out

    # 3-D: volumes as numpy (D, H, W) arrays (x fastest)
    def svt(self, vol) -> np.ndarray:
        v = np.ascontiguousarray(vol, dtype=np.float64)
        d, h, w = v.shape
        c = np.empty((d + 1, h + 1, w + 1), dtype=np.float64)
        self.lib.oracle_svt_build(_ptr(v), w, h, d, _ptr(c))
        return c

    def osbf_3d(self, vol, r: int, iterations: int) -> np.ndarray:
        return self._f3(self.lib.oracle_osbf_3d, vol, r, iterations, "osbf_3d")

    def box_filter_3d(self, vol, r: int, iterations: int) -> np.ndarray:
        return self._f3(self.lib.oracle_box_filter_3d, vol, r, iterations, "box_filter_3d")

    def _f3(self, fn, vol, r, iterations, name):
        v = np.ascontiguousarray(vol, dtype=np.float64)
        d, h, w = v.shape
        out = np.empty_like(v)
        st = fn(_ptr(v), _ptr(out), w, h, d, r, iterations)
        if st:
            raise CheckerError(st, name)
        return out

    def quantize(self, v: float, maxval: int) -> int:
        """io.hpp:108-115."""
        return self.lib.oracle_quantize(v, maxval)

    def smooth_raster(self, raster, filter: str, r: int, iterations: int,
                      out_bits: int = 8) -> np.ndarray:
        """tools/osbf_main.cpp:63-83 without file I/O: promote, filter, quantise."""
        x = np.ascontiguousarray(raster)
        h, w = x.shape[:2]
        c = 1 if x.ndim == 2 else x.shape[2]
        out = np.empty(x.shape, dtype=np.uint8 if out_bits == 8 else np.uint16)
        st = self.lib.oracle_smooth_raster(x.ctypes.data, x.dtype.itemsize, c, w, h,
                                           SMOOTH_FILTERS[filter], r, iterations, out.ctypes.data,
                                           out.dtype.itemsize)
        if st:
            raise CheckerError(st, "smooth_raster")
        return out

    def box_filter(self, plane, r: int, iterations: int) -> np.ndarray:
        """filters2d.hpp:38-56."""
        p = _as_f64(plane)
        h, w = p.shape
        out = np.empty_like(p)
        st = self.lib.oracle_box_filter(_ptr(p), _ptr(out), w, h, r, iterations)
        if st:
            raise CheckerError(st, "box_filter")
        return out

    def fast_osbf(self, plane, r: int, iterations: int) -> np.ndarray:
        """filters2d.hpp:105-154 (paper Algorithm 3)."""
        p = _as_f64(plane)
        h, w = p.shape
        out = np.empty_like(p)
        st = self.lib.oracle_fast_osbf(_ptr(p), _ptr(out), w, h, r, iterations)
        if st:
            raise CheckerError(st, "fast_osbf")
        return out

    def osbf_step(self, plane, r: int, with_selection: bool = False):
        p = _as_f64(plane)
        h, w = p.shape
        out = np.empty_like(p)
        sel = np.zeros((h, w), dtype=np.uint8)
        st = self.lib.oracle_osbf_step(_ptr(p), _ptr(out), w, h, r, _ptr(sel, _u8p))
        if st:
            raise CheckerError(st, "osbf_step")
        return (out, sel) if with_selection else out

    def sat(self, plane) -> np.ndarray:
        p = _as_f64(plane)
        h, w = p.shape
        c = np.empty((h + 1, w + 1), dtype=np.float64)
        self.lib.oracle_sat_build(_ptr(p), w, h, _ptr(c))
        return c

    def subwindow_means(self, cumsum: np.ndarray, w: int, h: int, x: int, y: int, r: int):
        out = np.empty(8, dtype=np.float64)
        st = self.lib.oracle_subwindow_means(_ptr(cumsum), w, h, x, y, r, _ptr(out))
        if st:
            raise CheckerError(st, "subwindow_means")
        return out

    def rect_mean(self, cumsum, w, h, x0, y0, x1, y1) -> float:
        m = ctypes.c_double()
        st = self.lib.oracle_rect_mean(_ptr(cumsum), w, h, x0, y0, x1, y1, ctypes.byref(m))
        if st:
            raise CheckerError(st, "rect_mean")
        return m.value


class Reference:
    """The unmodified reference headers behind ref_shim.cpp (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        lib = ctypes.CDLL(path)
        lib.ref_osbf.argtypes = [_dp, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        lib.ref_osbf_step.argtypes = [_dp, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        lib.ref_filter_multichannel.argtypes = [_dp, _dp] + [ctypes.c_int] * 5
        lib.ref_filter_multichannel_fast.argtypes = [_dp, _dp] + [ctypes.c_int] * 5
        lib.ref_fast_osbf.argtypes = [_dp, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int]
        lib.ref_box_filter.argtypes = lib.ref_fast_osbf.argtypes
        lib.ref_filter_3d.argtypes = [_dp, _dp] + [ctypes.c_int] * 6
        lib.ref_svt.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp]
        lib.ref_sat.argtypes = [_dp, ctypes.c_int, ctypes.c_int, _dp]
        lib.ref_subwindow_means.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _u8p]
        lib.ref_rect_mean.argtypes = [_dp] + [ctypes.c_int] * 6 + [_dp]
        lib.ref_quantize.argtypes = [ctypes.c_double, ctypes.c_int]
        lib.ref_smooth_file.argtypes = [ctypes.c_char_p, ctypes.c_char_p] + [ctypes.c_int] * 3
        lib.ref_set_max_threads.argtypes = [ctypes.c_int]
        lib.ref_set_max_threads.restype = None
        lib.ref_pin_allocator_for_timing.restype = None
        _ull = ctypes.c_ulonglong
        lib.ref_checkerboard.argtypes = [ctypes.c_int] * 3 + [ctypes.c_double] * 3 + [_ull, _dp, _dp]
        lib.ref_step_volume.argtypes = [ctypes.c_int] * 4 + [ctypes.c_double] * 3 + [_ull, _dp, _dp]
        lib.ref_phantom.argtypes = [ctypes.c_int, ctypes.c_int, _dp]
        lib.ref_psnr.argtypes = [_dp, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_double]
        lib.ref_psnr.restype = ctypes.c_double
        lib.ref_rmse.argtypes = [_dp, _dp, ctypes.c_int, ctypes.c_int]
        lib.ref_rmse.restype = ctypes.c_double
        self.lib = lib

    @staticmethod
    def available(path: str = REF_SO) -> bool:
        return os.path.exists(path)

    # -- acceptance-criterion inputs and metrics (the reference's own code)
    def checkerboard(self, w, h, cell, lo, hi, sigma, seed):
        """(clean, noisy): synth.hpp:52 checkerboard + :94 Gaussian noise."""
        c, n = np.empty((h, w)), np.empty((h, w))
        st = self.lib.ref_checkerboard(w, h, cell, lo, hi, sigma, seed, _ptr(c), _ptr(n))
        if st:
            raise CheckerError(st, "ref checkerboard")
        return c, n

    def step_volume(self, w, h, d, edge, lo, hi, sigma, seed):
        """(clean, noisy) volumes (D, H, W): synth.hpp:81 + :106."""
        c, n = np.empty((d, h, w)), np.empty((d, h, w))
        st = self.lib.ref_step_volume(w, h, d, edge, lo, hi, sigma, seed, _ptr(c), _ptr(n))
        if st:
            raise CheckerError(st, "ref step_volume")
        return c, n

    def phantom(self, w=256, h=256):
        """tests/support/fixtures.hpp:36, the reference's stand-in natural image."""
        p = np.empty((h, w))
        st = self.lib.ref_phantom(w, h, _ptr(p))
        if st:
            raise CheckerError(st, "ref phantom")
        return p

    def psnr(self, a, b, peak=255.0) -> float:
        a, b = _as_f64(a), _as_f64(b)
        return float(self.lib.ref_psnr(_ptr(a), _ptr(b), a.shape[1], a.shape[0], peak))

    def rmse(self, a, b) -> float:
        a, b = _as_f64(a), _as_f64(b)
        return float(self.lib.ref_rmse(_ptr(a), _ptr(b), a.shape[-1], a.size // a.shape[-1]))

    def set_max_threads(self, n: int) -> None:
        self.lib.ref_set_max_threads(n)

    def max_threads(self) -> int:
        return self.lib.ref_max_threads()

    def pin_allocator_for_timing(self) -> None:
        self.lib.ref_pin_allocator_for_timing()

    def osbf(self, plane, r: int, iterations: int) -> np.ndarray:
        p = _as_f64(plane)
        h, w = p.shape
        out = np.empty_like(p)
        st = self.lib.ref_osbf(_ptr(p), _ptr(out), w, h, r, iterations)
        if st:
            raise CheckerError(st, "ref osbf")
        return out

    def osbf_step(self, plane, r: int) -> np.ndarray:
        p = _as_f64(plane)
        h, w = p.shape
        out = np.empty_like(p)
        st = self.lib.ref_osbf_step(_ptr(p), _ptr(out), w, h, r)
        if st:
            raise CheckerError(st, "ref osbf_step")
        return out

    def filter_multichannel(self, planes, r: int, iterations: int,
                            variant: str = "exact") -> np.ndarray:
        p = _as_f64(planes)
        c, h, w = p.shape
        out = np.empty_like(p)
        fn = (self.lib.ref_filter_multichannel if variant == "exact"
              else self.lib.ref_filter_multichannel_fast)
        st = fn(_ptr(p), _ptr(out), c, w, h, r, iterations)
        if st:
            raise CheckerError(st, "ref filter_multichannel")
        return out

    def svt(self, vol) -> np.ndarray:
        v = np.ascontiguousarray(vol, dtype=np.float64)
        d, h, w = v.shape
        c = np.empty((d + 1, h + 1, w + 1), dtype=np.float64)
        st = self.lib.ref_svt(_ptr(v), w, h, d, _ptr(c))
        if st:
            raise CheckerError(st, "ref svt")
        return c

    def osbf_3d(self, vol, r: int, iterations: int) -> np.ndarray:
        return self._f3(vol, r, iterations, 1)

    def box_filter_3d(self, vol, r: int, iterations: int) -> np.ndarray:
        return self._f3(vol, r, iterations, 0)

    def _f3(self, vol, r, iterations, osbf3):
        v = np.ascontiguousarray(vol, dtype=np.float64)
        d, h, w = v.shape
        out = np.empty_like(v)
        st = self.lib.ref_filter_3d(_ptr(v), _ptr(out), w, h, d, r, iterations, osbf3)
        if st:
            raise CheckerError(st, "ref filter_3d")
        return out

    def box_filter(self, plane, r: int, iterations: int) -> np.ndarray:
        p = _as_f64(plane)
        h, w = p.shape
        out = np.empty_like(p)
        st = self.lib.ref_box_filter(_ptr(p), _ptr(out), w, h, r, iterations)
        if st:
            raise CheckerError(st, "ref box_filter")
        return out

    def fast_osbf(self, plane, r: int, iterations: int) -> np.ndarray:
        p = _as_f64(plane)
        h, w = p.shape
        out = np.empty_like(p)
        st = self.lib.ref_fast_osbf(_ptr(p), _ptr(out), w, h, r, iterations)
        if st:
            raise CheckerError(st, "ref fast_osbf")
        return out

    def sat(self, plane) -> np.ndarray:
        p = _as_f64(plane)
        h, w = p.shape
        c = np.empty((h + 1, w + 1), dtype=np.float64)
        st = self.lib.ref_sat(_ptr(p), w, h, _ptr(c))
        if st:
            raise CheckerError(st, "ref sat")
        return c

    def subwindow_means(self, plane, r: int):
        p = _as_f64(plane)
        h, w = p.shape
        out = np.empty((h, w, 8), dtype=np.float64)
        sel = np.zeros((h, w), dtype=np.uint8)
        st = self.lib.ref_subwindow_means(_ptr(p), w, h, r, _ptr(out), _ptr(sel, _u8p))
        if st:
            raise CheckerError(st, "ref subwindow_means")
        return out, sel

    def rect_mean(self, plane, x0, y0, x1, y1) -> float:
        p = _as_f64(plane)
        h, w = p.shape
        m = ctypes.c_double()
        st = self.lib.ref_rect_mean(_ptr(p), w, h, x0, y0, x1, y1, ctypes.byref(m))
        if st:
            raise CheckerError(st, "ref rect_mean")
        return m.value

    def quantize(self, v: float, maxval: int) -> int:
        return self.lib.ref_quantize(v, maxval)

    def smooth_file(self, in_path: str, out_path: str, filter: str, r: int,
                    iterations: int) -> None:
        """cmd_smooth (tools/osbf_main.cpp:63-83) through the reference's own
        read_image / filter_multichannel / write_image."""
        st = self.lib.ref_smooth_file(in_path.encode(), out_path.encode(), SMOOTH_FILTERS[filter],
                                      r, iterations)
        if st:
            raise CheckerError(st, "ref smooth_file")

    def smooth_raster(self, raster, filter: str, r: int, iterations: int, tmpdir: str,
                      maxval: int | None = None) -> np.ndarray:
        """smooth_file on a raster written as binary PGM/PPM (maxval defaults to
        255 for uint8, 65535 for uint16), output read back."""
        x = np.ascontiguousarray(raster)
        if maxval is None:
            maxval = 255 if x.dtype == np.uint8 else 65535
        src = os.path.join(tmpdir, "ref_in.pnm")
        dst = os.path.join(tmpdir, "ref_out.pnm")
        write_pnm(src, x, maxval)
        self.smooth_file(src, dst, filter, r, iterations)
        return read_pnm(dst)[0]


SMOOTH_FILTERS = {"osbf": 0, "fast-osbf": 1, "box": 2}


def write_pnm(path: str, raster: np.ndarray, maxval: int) -> None:
    """Binary P5 (H, W) / P6 (H, W, 3); 2-byte big-endian samples when maxval > 255."""
    x = np.asarray(raster)
    magic = b"P5" if x.ndim == 2 else b"P6"
    h, w = x.shape[:2]
    payload = x.astype(">u2" if maxval > 255 else np.uint8).tobytes()
    with open(path, "wb") as f:
        f.write(magic + b"\n%d %d\n%d\n" % (w, h, maxval) + payload)


def read_pnm(path: str):
    """Binary P5/P6 as written by write_image (io.hpp:187-215) -> (raster, maxval)."""
    data = open(path, "rb").read()
    fields, pos = [], 2
    while len(fields) < 3:
        while data[pos:pos + 1].isspace():
            pos += 1
        start = pos
        while not data[pos:pos + 1].isspace():
            pos += 1
        fields.append(int(data[start:pos]))
    pos += 1
    w, h, maxval = fields
    c = 3 if data[:2] == b"P6" else 1
    dt = np.dtype(">u2") if maxval > 255 else np.dtype(np.uint8)
    x = np.frombuffer(data[pos:pos + w * h * c * dt.itemsize], dtype=dt)
    x = x.astype(np.uint16 if maxval > 255 else np.uint8).reshape((h, w, c) if c == 3 else (h, w))
    return x, maxval
