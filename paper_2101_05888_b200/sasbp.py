"""Thin ctypes binding of libsasbp.so (include/sasbp.h) -- argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module converts numpy
arrays / torch tensors to pointers and status codes to exceptions.  There is no CPU
fallback: if the library is missing or cannot find an sm_100 device, calls raise.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libsasbp.so")

SAS_OK, SAS_E_INVALID, SAS_E_STATE, SAS_E_NOMEM, SAS_E_CUDA, SAS_E_UNSUPPORTED = 0, -1, -2, -3, -4, -5
SAS_FORM_ACCUMULATE = 1
_NAMES = {0: "SAS_OK", -1: "SAS_E_INVALID", -2: "SAS_E_STATE", -3: "SAS_E_NOMEM", -4: "SAS_E_CUDA",
          -5: "SAS_E_UNSUPPORTED"}

EXPORTS = ("sas_bp_create", "sas_bp_destroy", "sas_bp_set_pings", "sas_bp_set_pings_device", "sas_bp_form",
           "sas_bp_form_device", "sas_bp_count_terms", "sas_bp_workspace_bytes", "sas_rangecompress",
           "sas_rangecompress_device", "sas_last_error", "sas_version", "sas_bp_get_plan", "sas_bp_form_streamed", "sas_bp_set_beam", "sas_bp_set_motion", "sas_bp_set_nav", "sas_bp_set_medium",
           "sas_bp_set_weighting", "sas_upsample", "sas_upsample_device", "sas_baseband", "sas_baseband_device",
           "sas_whitening_gain", "sas_whitening_gain_device", "sas_rangecompress_whitened",
           "sas_rangecompress_whitened_device")


class SasError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_NAMES.get(status, status)}: {msg}")
        self.status = status


class sas_bp_plan(ctypes.Structure):
    _fields_ = [("tile", ctypes.c_int32 * 3), ("window", ctypes.c_int32), ("rx_mode", ctypes.c_int32),
                ("tma", ctypes.c_int32), ("batch", ctypes.c_int32), ("ctas_per_sm", ctypes.c_int32),
                ("tail_split", ctypes.c_int32)]


class sas_beam(ctypes.Structure):
    _fields_ = [("az_fwhm", ctypes.c_double), ("el_fwhm", ctypes.c_double), ("bistatic", ctypes.c_int32),
                ("cull", ctypes.c_int32)]


class sas_grid(ctypes.Structure):
    _fields_ = [("origin", ctypes.c_double * 3), ("step_x", ctypes.c_double * 3),
                ("step_y", ctypes.c_double * 3), ("step_z", ctypes.c_double * 3),
                ("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32)]


_lib = None


def load_library(path: Optional[str] = None):
    """Load libsasbp.so (raises OSError loudly if it was not built).  SASBP_LIB overrides the
    path (A/B builds of the same library)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("SASBP_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise OSError(f"libsasbp.so not built at {path}; run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    vp, f32p, f64p = ctypes.c_void_p, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_double)
    i32 = ctypes.c_int32
    sig = {
        "sas_bp_create": ([ctypes.c_double] * 4 + [ctypes.POINTER(sas_grid), ctypes.POINTER(vp)], ctypes.c_int),
        "sas_bp_destroy": ([vp], None),
        "sas_bp_set_pings": ([vp, f32p, i32, i32, i32, f64p, f64p, f64p], ctypes.c_int),
        "sas_bp_set_pings_device": ([vp, vp, i32, i32, i32, f64p, f64p, f64p, vp], ctypes.c_int),
        "sas_bp_form": ([vp, f32p], ctypes.c_int),
        "sas_bp_form_device": ([vp, vp, vp, i32], ctypes.c_int),
        "sas_bp_count_terms": ([vp, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)], ctypes.c_int),
        "sas_bp_workspace_bytes": ([vp], ctypes.c_size_t),
        "sas_rangecompress": ([f32p, i32, i32, i32, f32p, i32, f32p], ctypes.c_int),
        "sas_rangecompress_device": ([vp, i32, i32, i32, vp, i32, vp, vp], ctypes.c_int),
        "sas_last_error": ([], ctypes.c_char_p),
        "sas_version": ([], ctypes.c_char_p),
        "sas_bp_get_plan": ([vp, ctypes.POINTER(sas_bp_plan)], ctypes.c_int),
        "sas_bp_form_streamed": ([vp, f32p, i32, i32, i32, f64p, f64p, f64p, f32p, i32], ctypes.c_int),
        "sas_bp_set_beam": ([vp, ctypes.POINTER(sas_beam), f64p, i32], ctypes.c_int),
        "sas_bp_set_motion": ([vp, f64p, i32], ctypes.c_int),
        "sas_bp_set_nav": ([vp, f64p, i32, i32, i32, ctypes.c_double], ctypes.c_int),
        "sas_bp_set_medium": ([vp, ctypes.c_double, ctypes.c_double], ctypes.c_int),
        "sas_bp_set_weighting": ([vp, i32], ctypes.c_int),
        "sas_upsample": ([f32p, i32, i32, i32, f32p], ctypes.c_int),
        "sas_whitening_gain": ([f32p, i32, i32, i32, ctypes.c_double, f32p], ctypes.c_int),
        "sas_whitening_gain_device": ([vp, i32, i32, i32, ctypes.c_double, vp, vp], ctypes.c_int),
        "sas_rangecompress_whitened": ([f32p, i32, i32, i32, f32p, i32, f32p, i32, f32p], ctypes.c_int),
        "sas_rangecompress_whitened_device": ([vp, i32, i32, i32, vp, i32, vp, i32, vp, vp], ctypes.c_int),
        "sas_upsample_device": ([vp, i32, i32, i32, vp, vp], ctypes.c_int),
        "sas_baseband": ([f32p, i32, i32, i32, ctypes.c_double, ctypes.c_double, f64p, f32p, i32, i32, i32, f32p],
                         ctypes.c_int),
        "sas_baseband_device": ([vp, i32, i32, i32, ctypes.c_double, ctypes.c_double, vp, vp, i32, i32, i32, vp,
                                 vp], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name, None)
        if fn is None:   # an older A/B build without this entry point
            continue
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def _check(st: int):
    if st != SAS_OK:
        raise SasError(st, _lib.sas_last_error().decode())


def version() -> str:
    return load_library().sas_version().decode()


def make_grid(grid) -> sas_grid:
    g = sas_grid()
    for k in ("origin", "step_x", "step_y", "step_z"):
        v = np.asarray(grid[k], dtype=np.float64).reshape(3)
        getattr(g, k)[:] = [float(x) for x in v]
    g.nx, g.ny, g.nz = int(grid["nx"]), int(grid["ny"]), int(grid["nz"])
    return g


def _f64(a, shape):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.size != int(np.prod(shape)):
        raise ValueError(f"expected {shape} float64, got {a.shape}")
    return a


def _ptr(a, ct):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(ct))


def _stream_ptr(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        except ImportError:
            pass
        return None
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _is_torch(x) -> bool:
    return hasattr(x, "data_ptr") and not hasattr(x, "ctypes")


def _dev_ptr(t, nbytes_min: int, dtype: Optional[str] = None):
    """Device pointer of a torch CUDA tensor (complex64 / float32 / float64): device, contiguity,
    dtype (when given, e.g. "complex64") and size checked, so a wrong tensor raises here instead of
    letting the library read or write past it."""
    if not getattr(t, "is_cuda", False):
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    if dtype is not None and str(t.dtype) != "torch." + dtype:
        raise ValueError(f"expected a {dtype} tensor, got {t.dtype}")
    if t.numel() * t.element_size() < nbytes_min:
        raise ValueError("tensor too small")
    return ctypes.c_void_p(t.data_ptr())


def _host_c64_in(x, name: str, ndim: int = 3):
    """(keep-alive object, float* pointer, shape) of host complex64 input (numpy, or a CPU torch
    tensor: dtype / device checked, made contiguous)."""
    if _is_torch(x):
        if x.is_cuda:
            raise ValueError(f"{name}: expected host memory; use the *_device call for CUDA tensors")
        if str(x.dtype) != "torch.complex64":
            raise ValueError(f"{name}: expected complex64, got {x.dtype}")
        keep = x.contiguous()
        ptr = ctypes.cast(ctypes.c_void_p(keep.data_ptr()), ctypes.POINTER(ctypes.c_float))
        shape = tuple(keep.shape)
    else:
        keep = np.ascontiguousarray(x, dtype=np.complex64)
        ptr = keep.view(np.float32).ctypes.data_as(ctypes.POINTER(ctypes.c_float))
        shape = keep.shape
    if len(shape) != ndim:
        raise ValueError(f"{name}: expected {ndim} dimensions, got shape {shape}")
    return keep, ptr, shape


def _host_c64_out(out, shape, name: str = "out"):
    """float* pointer of a caller-provided host output: complex64, C-contiguous, exactly `shape`."""
    if _is_torch(out):
        if out.is_cuda or str(out.dtype) != "torch.complex64" or not out.is_contiguous() \
                or tuple(out.shape) != tuple(shape):
            raise ValueError(f"{name} must be a contiguous host complex64 tensor of shape {tuple(shape)}")
        return ctypes.cast(ctypes.c_void_p(out.data_ptr()), ctypes.POINTER(ctypes.c_float))
    if not isinstance(out, np.ndarray) or out.dtype != np.complex64 or not out.flags.c_contiguous \
            or out.shape != tuple(shape):
        raise ValueError(f"{name} must be a C-contiguous complex64 array of shape {tuple(shape)}")
    return out.view(np.float32).ctypes.data_as(ctypes.POINTER(ctypes.c_float))


class Backprojector:
    """One TDBP plan on the current CUDA device (sas_bp_create ... sas_bp_destroy)."""

    def __init__(self, fc: float, bandwidth: float, fs: float, c: float, grid):
        lib = load_library()
        self._grid = make_grid(grid)
        self.shape = (self._grid.nz, self._grid.ny, self._grid.nx)
        h = ctypes.c_void_p()
        _check(lib.sas_bp_create(fc, bandwidth, fs, c, ctypes.byref(self._grid), ctypes.byref(h)))
        self._h = h
        self.P = self.E = self.Ns = 0
        self._keep = None

    def close(self):
        if getattr(self, "_h", None):
            _lib.sas_bp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _geo(self, P, E, tx, rx, t0):
        tx = _f64(tx, (P, 3))
        rx = _f64(rx, (P, E, 3))
        t0 = None if t0 is None else _f64(t0, (P,))
        return tx, rx, t0

    def set_pings(self, echoes, tx, rx, t0=None):
        """Host echoes complex64 [P][E][Ns] (numpy or CPU torch tensor, pinned or not); copied."""
        keep, ptr, (P, E, Ns) = _host_c64_in(echoes, "echoes")
        tx, rx, t0 = self._geo(P, E, tx, rx, t0)
        _check(_lib.sas_bp_set_pings(self._h, ptr, P, E, Ns, _ptr(tx, ctypes.c_double),
                                     _ptr(rx, ctypes.c_double), _ptr(t0, ctypes.c_double)))
        del keep
        self.P, self.E, self.Ns = P, E, Ns

    def set_pings_device(self, echoes, tx, rx, t0=None, stream=None):
        """Borrow a CUDA complex64 tensor [P][E][Ns] (kept alive by this object)."""
        if len(echoes.shape) != 3:
            raise ValueError(f"echoes: expected [P][E][Ns], got shape {tuple(echoes.shape)}")
        P, E, Ns = echoes.shape
        tx, rx, t0 = self._geo(P, E, tx, rx, t0)
        _check(_lib.sas_bp_set_pings_device(self._h, _dev_ptr(echoes, P * E * Ns * 8, "complex64"), P, E, Ns,
                                            _ptr(tx, ctypes.c_double), _ptr(rx, ctypes.c_double),
                                            _ptr(t0, ctypes.c_double), _stream_ptr(stream)))
        self._keep = echoes
        self.P, self.E, self.Ns = P, E, Ns

    def form(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        """Form into host memory; returns complex64 [nz][ny][nx]."""
        if out is None:
            out = np.empty(self.shape, dtype=np.complex64)
        ptr = _host_c64_out(out, self.shape)
        _check(_lib.sas_bp_form(self._h, ptr))
        return out

    def form_streamed(self, echoes, tx, rx, t0=None, out=None, chunks: int = 0) -> np.ndarray:
        """End to end from host echoes with chunked H2D overlapped with backprojection
        (sas_bp_form_streamed).  `echoes`: complex64 [P][E][Ns] numpy / CPU torch (pin it for
        overlap); returns the image in host memory."""
        ek, eptr, (P, E, Ns) = _host_c64_in(echoes, "echoes")
        if out is None:
            out = np.empty(self.shape, dtype=np.complex64)
        optr = _host_c64_out(out, self.shape)
        tx, rx, t0 = self._geo(P, E, tx, rx, t0)
        _check(_lib.sas_bp_form_streamed(self._h, eptr, P, E, Ns, _ptr(tx, ctypes.c_double), _ptr(rx, ctypes.c_double),
                                         _ptr(t0, ctypes.c_double), optr, int(chunks)))
        del ek
        self.P, self.E, self.Ns = P, E, Ns
        return out

    def form_device(self, image, stream=None, accumulate: bool = False):
        """Form into a CUDA complex64 tensor of the grid shape, asynchronously on `stream`."""
        n = self.shape[0] * self.shape[1] * self.shape[2]
        _check(_lib.sas_bp_form_device(self._h, _dev_ptr(image, n * 8, "complex64"), _stream_ptr(stream),
                                       SAS_FORM_ACCUMULATE if accumulate else 0))
        return image

    def count_terms(self):
        """(dense, in_window) term counts of the current ping set (K3; in_window on device)."""
        d, w = ctypes.c_uint64(), ctypes.c_uint64()
        _check(_lib.sas_bp_count_terms(self._h, ctypes.byref(d), ctypes.byref(w)))
        return int(d.value), int(w.value)

    def set_beam(self, az_fwhm=None, el_fwhm: float = 0.0, bistatic: bool = False, cull: bool = True, axes=None):
        """Gate the sum to the transmit (and, bistatic, receive) FOV cones (NEXT-1); az_fwhm=None
        returns to the dense sum.  axes: [P][2][3] per-ping (along-track, boresight) or None."""
        if az_fwhm is None:
            _check(_lib.sas_bp_set_beam(self._h, None, None, 0))
            return
        b = sas_beam(float(az_fwhm), float(el_fwhm), 1 if bistatic else 0, 1 if cull else 0)
        ax = None if axes is None else np.ascontiguousarray(axes, dtype=np.float64)
        P = 0 if ax is None else ax.shape[0]
        _check(_lib.sas_bp_set_beam(self._h, ctypes.byref(b), _ptr(ax, ctypes.c_double), P))

    def set_motion(self, vel=None):
        """Receivers move with the per-ping platform velocity vel [P][3] during reception
        (NEXT-2); None = stop-and-hop."""
        if vel is None:
            _check(_lib.sas_bp_set_motion(self._h, None, 0))
            return
        v = np.ascontiguousarray(vel, dtype=np.float64).reshape(-1, 3)
        _check(_lib.sas_bp_set_motion(self._h, _ptr(v, ctypes.c_double), v.shape[0]))

    def set_nav(self, lut=None, dt: float = 0.0):
        """Receivers follow tabled trajectories lut [P][E][K][3] (nodes dt seconds apart from the
        transmit; NEXT-2, reading R23); None = no table."""
        if lut is None:
            _check(_lib.sas_bp_set_nav(self._h, None, 0, 0, 0, 0.0))
            return
        a = np.ascontiguousarray(lut, dtype=np.float64)
        if a.ndim != 4 or a.shape[-1] != 3:
            raise ValueError("lut must be float64 [P][E][K][3]")
        _check(_lib.sas_bp_set_nav(self._h, _ptr(a, ctypes.c_double), a.shape[0], a.shape[1], a.shape[2], float(dt)))

    def set_medium(self, zb: float = 0.0, c2: float = 0.0):
        """Flat sediment-water interface z = zb with sediment sound speed c2 (NEXT-3); c2 <= 0 =
        isovelocity."""
        _check(_lib.sas_bp_set_medium(self._h, float(zb), float(c2)))

    def set_weighting(self, spreading: bool = False):
        """Multiply every term by R_tx R_rx (NEXT-4, R18); False = unweighted sum (R6)."""
        _check(_lib.sas_bp_set_weighting(self._h, 1 if spreading else 0))

    def plan(self) -> dict:
        """The execution plan (tile, window, rx_mode, tma, batch) -- sas_bp_get_plan."""
        p = sas_bp_plan()
        _check(_lib.sas_bp_get_plan(self._h, ctypes.byref(p)))
        return {"tile": tuple(p.tile), "window": p.window, "rx_mode": ("series3", "series4", "exact", "refracted")[p.rx_mode]
                if p.rx_mode >= 0 else None, "tma": None if p.tma < 0 else bool(p.tma), "batch": p.batch,
                "ctas_per_sm": p.ctas_per_sm, "tail_split": p.tail_split}

    @property
    def workspace_bytes(self) -> int:
        return int(_lib.sas_bp_workspace_bytes(self._h))


def rangecompress(raw, replica) -> np.ndarray:
    """Host matched filter: out[..., n] = sum_m raw[..., n+m] conj(replica[m]) (K1 on the GPU)."""
    lib = load_library()
    raw = np.ascontiguousarray(raw, dtype=np.complex64)
    rep = np.ascontiguousarray(replica, dtype=np.complex64).ravel()
    shp = raw.shape
    Ns = shp[-1]
    nch = int(np.prod(shp[:-1])) if len(shp) > 1 else 1
    out = np.empty_like(raw)
    f = lambda a: a.view(np.float32).ctypes.data_as(ctypes.POINTER(ctypes.c_float))
    _check(lib.sas_rangecompress(f(raw), nch, 1, Ns, f(rep), rep.size, f(out)))
    return out


def rangecompress_device(raw, replica, out, stream=None):
    """CUDA-tensor matched filter (complex64 [..., Ns] -> out of the same shape)."""
    lib = load_library()
    Ns = raw.shape[-1]
    nch = raw.numel() // Ns
    _check(lib.sas_rangecompress_device(_dev_ptr(raw, raw.numel() * 8), nch, 1, Ns,
                                        _dev_ptr(replica, replica.numel() * 8), replica.numel(),
                                        _dev_ptr(out, raw.numel() * 8), _stream_ptr(stream)))
    return out


def upsample(x, U: int) -> np.ndarray:
    """Host xU band-limited upsampling by the 8-tap windowed sinc (K1b, R19): complex64
    [..., Ns] -> [..., U*Ns] at rate U*fs, same t0."""
    lib = load_library()
    x = np.ascontiguousarray(x, dtype=np.complex64)
    shp = x.shape
    Ns = shp[-1]
    nch = int(np.prod(shp[:-1])) if len(shp) > 1 else 1
    out = np.empty(shp[:-1] + (U * Ns,), dtype=np.complex64)
    f = lambda a: a.view(np.float32).ctypes.data_as(ctypes.POINTER(ctypes.c_float))
    _check(lib.sas_upsample(f(x), nch, Ns, int(U), f(out)))
    return out


def upsample_device(x, U: int, out, stream=None):
    """CUDA-tensor xU upsampling: complex64 [..., Ns] -> out complex64 [..., U*Ns]."""
    lib = load_library()
    Ns = x.shape[-1]
    nch = x.numel() // Ns
    _check(lib.sas_upsample_device(_dev_ptr(x, x.numel() * 8), nch, Ns, int(U), _dev_ptr(out, x.numel() * 8 * U),
                                   _stream_ptr(stream)))
    return out


def _bb_args(t0, h, P):
    t = None if t0 is None else np.ascontiguousarray(t0, dtype=np.float64).reshape(P)
    hh = np.ascontiguousarray(h, dtype=np.float32).ravel()
    return t, hh


def baseband(x, fs_in: float, fc: float, t0, h, D: int, Nout: int) -> np.ndarray:
    """Host basebanding (K0, R20): real float32 [P][E][Nin] at fs_in -> complex64 [P][E][Nout]:
    mix by exp(-j 2 pi fc (t0_p + n/fs_in)), centred FIR h (odd length), keep every D-th sample."""
    lib = load_library()
    x = np.ascontiguousarray(x, dtype=np.float32)
    P, E, Nin = x.shape
    t, hh = _bb_args(t0, h, P)
    out = np.empty((P, E, int(Nout)), dtype=np.complex64)
    _check(lib.sas_baseband(_ptr(x, ctypes.c_float), P, E, Nin, float(fs_in), float(fc), _ptr(t, ctypes.c_double),
                            _ptr(hh, ctypes.c_float), hh.size, int(D), int(Nout),
                            out.view(np.float32).ctypes.data_as(ctypes.POINTER(ctypes.c_float))))
    return out


def baseband_device(x, fs_in: float, fc: float, t0, h, D: int, out, stream=None):
    """CUDA-tensor basebanding: float32 [P][E][Nin] -> out complex64 [P][E][Nout]; t0 (float64
    [P] CUDA tensor or None) and h (float32 [Nh] CUDA tensor) on the device; asynchronous."""
    lib = load_library()
    P, E, Nin = x.shape
    Nout = out.shape[-1]
    t0p = None if t0 is None else _dev_ptr(t0, P * 8)
    _check(lib.sas_baseband_device(_dev_ptr(x, x.numel() * 4), P, E, Nin, float(fs_in), float(fc), t0p,
                                   _dev_ptr(h, h.numel() * 4), h.numel(), int(D), int(Nout),
                                   _dev_ptr(out, P * E * Nout * 8), _stream_ptr(stream)))
    return out


def whitening_gain(raw, M: int, gamma: float) -> np.ndarray:
    """Eq. 9 whitening power gain G [M] (float32) of complex64 [..., Ns] (R21; GPU periodogram)."""
    lib = load_library()
    raw = np.ascontiguousarray(raw, dtype=np.complex64)
    Ns = raw.shape[-1]
    nch = raw.size // Ns
    G = np.empty(int(M), dtype=np.float32)
    f = lambda a: a.view(np.float32).ctypes.data_as(ctypes.POINTER(ctypes.c_float))
    _check(lib.sas_whitening_gain(f(raw), nch, Ns, int(M), float(gamma), f(G)))
    return G


def whitening_gain_device(raw, M: int, gamma: float, G, stream=None):
    """CUDA-tensor variant: G float32 [M] on the device (NaN for an all-zero batch)."""
    lib = load_library()
    Ns = raw.shape[-1]
    _check(lib.sas_whitening_gain_device(_dev_ptr(raw, raw.numel() * 8), raw.numel() // Ns, Ns, int(M), float(gamma),
                                         _dev_ptr(G, int(M) * 4), _stream_ptr(stream)))
    return G


def rangecompress_whitened(raw, replica, G) -> np.ndarray:
    """Host whitened matched filter (R21 + R14): sqrt(G) frequency-sampling FIR, then the replica."""
    lib = load_library()
    raw = np.ascontiguousarray(raw, dtype=np.complex64)
    rep = np.ascontiguousarray(replica, dtype=np.complex64).ravel()
    g = np.ascontiguousarray(G, dtype=np.float32).ravel()
    Ns = raw.shape[-1]
    nch = raw.size // Ns
    out = np.empty_like(raw)
    f = lambda a: a.view(np.float32).ctypes.data_as(ctypes.POINTER(ctypes.c_float))
    _check(lib.sas_rangecompress_whitened(f(raw), nch, 1, Ns, f(rep), rep.size, f(g), g.size, f(out)))
    return out


def rangecompress_whitened_device(raw, replica, G, out, stream=None):
    """CUDA-tensor whitened matched filter (G a float32 CUDA tensor [M])."""
    lib = load_library()
    Ns = raw.shape[-1]
    nch = raw.numel() // Ns
    _check(lib.sas_rangecompress_whitened_device(_dev_ptr(raw, raw.numel() * 8), nch, 1, Ns,
                                                 _dev_ptr(replica, replica.numel() * 8), replica.numel(),
                                                 _dev_ptr(G, G.numel() * 4), G.numel(),
                                                 _dev_ptr(out, raw.numel() * 8), _stream_ptr(stream)))
    return out
