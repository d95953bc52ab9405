"""fp64 CPU oracle for the TDBP hot path (arXiv 2101.05888) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2101_05888_b200``) never imports it; the two share no code.

What is computed is documented in ``oracle/oracle.c`` (the definition of
SURVEY §8(c), PAPER.md Eq. (eqn:backprojection) P:89-92).  This module is only
ctypes marshalling plus the gcc build of ``liboracle.so``.

Parity status: every function here is pinned (tests/test_oracle_pins.py):
``tdbp_points`` / ``tdbp_grid`` by closed forms, hand-computed mono/bistatic
delays, zero-extension values, point-target physics and invariants;
``rangecompress`` by the autocorrelation-peak, shift and mainlobe pins;
``tdbp_points_gated`` (NEXT-1, reading R15) by the wide-open special case (= dense),
the azimuth / elevation boundary examples, monotonicity in the beamwidth, rigid-rotation
invariance and the config-1 target under the generator's own beam; the NEXT-4 variants
``tdbp_points_weighted`` (R18), ``upsample`` / ``lanczos4`` (R19) and ``baseband`` (R20) by
closed forms, interpolating / band-limited reproduction properties and config-1 physics;
``whitening_gain`` / ``rangecompress_whitened`` (R21) by the SPEC's hand examples (flat ->
0 dB, P = [1, 4] -> [0, -6.02] dB), the gamma limit, G = 1 -> plain compression and spectral
flattening of coloured noise.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2, OpenMP, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        f64p = ctypes.POINTER(ctypes.c_double)
        f32p = ctypes.POINTER(ctypes.c_float)
        i64p = ctypes.POINTER(ctypes.c_int64)
        lib.oracle_tdbp_points.argtypes = [f32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                           f64p, f64p, f64p, ctypes.c_double, ctypes.c_double,
                                           ctypes.c_double, f64p, ctypes.c_int64, f64p, i64p]
        lib.oracle_tdbp_points.restype = ctypes.c_int
        lib.oracle_tdbp_grid_pixels.argtypes = [f32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                                f64p, f64p, f64p, ctypes.c_double, ctypes.c_double,
                                                ctypes.c_double, f64p, f64p, f64p, f64p, i64p,
                                                ctypes.c_int64, f64p, i64p]
        lib.oracle_tdbp_grid_pixels.restype = ctypes.c_int
        lib.oracle_tdbp_points_gated.argtypes = [f32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                                 f64p, f64p, f64p, ctypes.c_double, ctypes.c_double,
                                                 ctypes.c_double, f64p, ctypes.c_double, ctypes.c_double,
                                                 ctypes.c_int32, f64p, ctypes.c_int64, f64p, i64p]
        lib.oracle_tdbp_points_gated.restype = ctypes.c_int
        lib.oracle_tdbp_points_motion.argtypes = [f32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                                  f64p, f64p, f64p, f64p, ctypes.c_double, ctypes.c_double,
                                                  ctypes.c_double, f64p, ctypes.c_int64, f64p, i64p]
        lib.oracle_tdbp_points_motion.restype = ctypes.c_int
        lib.oracle_delay_moving.argtypes = [f64p, f64p, f64p, f64p, ctypes.c_double]
        lib.oracle_delay_moving.restype = ctypes.c_double
        lib.oracle_tdbp_points_nav.argtypes = [f32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, f64p, f64p,
                                               ctypes.c_int32, ctypes.c_double, f64p, ctypes.c_double,
                                               ctypes.c_double, ctypes.c_double, f64p, ctypes.c_int64, f64p, i64p]
        lib.oracle_tdbp_points_nav.restype = ctypes.c_int
        lib.oracle_nav_eval.argtypes = [f64p, ctypes.c_int32, ctypes.c_double, ctypes.c_double, f64p]
        lib.oracle_nav_eval.restype = None
        lib.oracle_delay_nav.argtypes = [f64p, f64p, f64p, ctypes.c_int32, ctypes.c_double, ctypes.c_double]
        lib.oracle_delay_nav.restype = ctypes.c_double
        lib.oracle_tdbp_points_gated_nav.argtypes = [f32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, f64p, f64p,
                                                     f64p, ctypes.c_int32, ctypes.c_double, f64p, ctypes.c_double,
                                                     ctypes.c_double, ctypes.c_double, f64p, ctypes.c_double,
                                                     ctypes.c_double, ctypes.c_int32, f64p, ctypes.c_int64, f64p, i64p]
        lib.oracle_tdbp_points_gated_nav.restype = ctypes.c_int
        lib.oracle_tdbp_points_refracted.argtypes = [f32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                                     f64p, f64p, f64p, ctypes.c_double, ctypes.c_double,
                                                     ctypes.c_double, ctypes.c_double, ctypes.c_double, f64p,
                                                     ctypes.c_int64, f64p, i64p]
        lib.oracle_tdbp_points_refracted.restype = ctypes.c_int
        lib.oracle_travel_refracted.argtypes = [f64p, f64p, ctypes.c_double, ctypes.c_double, ctypes.c_double]
        lib.oracle_travel_refracted.restype = ctypes.c_double
        lib.oracle_rangecompress.argtypes = [f32p, ctypes.c_int64, ctypes.c_int32, f32p,
                                             ctypes.c_int32, f64p]
        lib.oracle_rangecompress.restype = ctypes.c_int
        lib.oracle_tdbp_points_weighted.argtypes = lib.oracle_tdbp_points.argtypes
        lib.oracle_tdbp_points_weighted.restype = ctypes.c_int
        lib.oracle_lanczos4.argtypes = [ctypes.c_double]
        lib.oracle_lanczos4.restype = ctypes.c_double
        lib.oracle_upsample.argtypes = [f32p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, f64p]
        lib.oracle_upsample.restype = ctypes.c_int
        lib.oracle_baseband.argtypes = [f32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                                        ctypes.c_double, f64p, f32p, ctypes.c_int32, ctypes.c_int32,
                                        ctypes.c_int32, f64p]
        lib.oracle_baseband.restype = ctypes.c_int
        lib.oracle_whitening_gain.argtypes = [f32p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                                              f64p, f64p]
        lib.oracle_whitening_gain.restype = ctypes.c_int
        lib.oracle_rangecompress_whitened.argtypes = [f32p, ctypes.c_int64, ctypes.c_int32, f32p, ctypes.c_int32,
                                                      f64p, ctypes.c_int32, f64p]
        lib.oracle_rangecompress_whitened.restype = ctypes.c_int
        lib.oracle_tdbp_points_gated_weighted.argtypes = [f32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                                          f64p, f64p, f64p, ctypes.c_double, ctypes.c_double,
                                                          ctypes.c_double, f64p, ctypes.c_double, ctypes.c_double,
                                                          ctypes.c_int32, f64p, ctypes.c_int64, f64p]
        lib.oracle_tdbp_points_gated_weighted.restype = ctypes.c_int
        lib.oracle_tdbp_points_gated_motion.argtypes = [f32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                                        f64p, f64p, f64p, f64p, ctypes.c_double, ctypes.c_double,
                                                        ctypes.c_double, f64p, ctypes.c_double, ctypes.c_double,
                                                        ctypes.c_int32, f64p, ctypes.c_int64, f64p, i64p]
        lib.oracle_tdbp_points_gated_motion.restype = ctypes.c_int
        lib.oracle_tdbp_points_gated_refracted.argtypes = [f32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                                           f64p, f64p, f64p, ctypes.c_double, ctypes.c_double,
                                                           ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                                           f64p, ctypes.c_double, ctypes.c_double, ctypes.c_int32,
                                                           f64p, ctypes.c_int64, f64p, i64p]
        lib.oracle_tdbp_points_gated_refracted.restype = ctypes.c_int
        lib.oracle_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct)) if a is not None else None


def _echo_arrays(echoes, tx, rx, t0):
    echoes = np.ascontiguousarray(echoes)
    if echoes.dtype == np.complex64:
        echoes = echoes.view(np.float32).reshape(echoes.shape + (2,))
    if echoes.dtype != np.float32 or echoes.ndim != 4 or echoes.shape[-1] != 2:
        raise ValueError("echoes must be complex64 [P][E][Ns] or float32 [P][E][Ns][2]")
    P, E, Ns = echoes.shape[:3]
    tx = np.ascontiguousarray(tx, dtype=np.float64).reshape(P, 3)
    rx = np.ascontiguousarray(rx, dtype=np.float64).reshape(P, E, 3)
    t0 = None if t0 is None else np.ascontiguousarray(t0, dtype=np.float64).reshape(P)
    return echoes, P, E, Ns, tx, rx, t0


def tdbp_points(echoes, tx, rx, t0, fc, fs, c, pts, with_count=False):
    """I(x) at explicit fp64 points ``pts[N][3]``; returns complex128 [N] (and N_u counts)."""
    lib = _load()
    echoes, P, E, Ns, tx, rx, t0 = _echo_arrays(echoes, tx, rx, t0)
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
    N = pts.shape[0]
    out = np.zeros((N, 2), dtype=np.float64)
    cnt = np.zeros(N, dtype=np.int64) if with_count else None
    rc = lib.oracle_tdbp_points(_p(echoes, ctypes.c_float), P, E, Ns, _p(tx, ctypes.c_double),
                                _p(rx, ctypes.c_double), _p(t0, ctypes.c_double), float(fc),
                                float(fs), float(c), _p(pts, ctypes.c_double), N,
                                _p(out, ctypes.c_double), _p(cnt, ctypes.c_int64))
    if rc != 0:
        raise ValueError("oracle_tdbp_points: invalid arguments")
    res = out[:, 0] + 1j * out[:, 1]
    return (res, cnt) if with_count else res


def tdbp_points_gated(echoes, tx, rx, t0, fc, fs, c, pts, az, el=0.0, bistatic=False, axes=None,
                      with_count=False):
    """Gated TDBP (NEXT-1): only terms whose point lies in the tx (and, bistatic, rx) FOV cone.
    axes: [P][2][3] per-ping along-track axis a and boresight b (NED), None = (+x, +y)."""
    lib = _load()
    echoes, P, E, Ns, tx, rx, t0 = _echo_arrays(echoes, tx, rx, t0)
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
    ax = None if axes is None else np.ascontiguousarray(axes, dtype=np.float64).reshape(P, 2, 3)
    N = pts.shape[0]
    out = np.zeros((N, 2), dtype=np.float64)
    cnt = np.zeros(N, dtype=np.int64) if with_count else None
    rc = lib.oracle_tdbp_points_gated(_p(echoes, ctypes.c_float), P, E, Ns, _p(tx, ctypes.c_double),
                                      _p(rx, ctypes.c_double), _p(t0, ctypes.c_double), float(fc), float(fs),
                                      float(c), _p(ax, ctypes.c_double), float(az), float(el),
                                      1 if bistatic else 0, _p(pts, ctypes.c_double), N,
                                      _p(out, ctypes.c_double), _p(cnt, ctypes.c_int64))
    if rc != 0:
        raise ValueError("oracle_tdbp_points_gated: invalid arguments")
    res = out[:, 0] + 1j * out[:, 1]
    return (res, cnt) if with_count else res


def tdbp_points_motion(echoes, tx, rx, t0, vel, fc, fs, c, pts, with_count=False):
    """TDBP with the receiver moving at the per-ping velocity vel [P][3] during reception (NEXT-2)."""
    lib = _load()
    echoes, P, E, Ns, tx, rx, t0 = _echo_arrays(echoes, tx, rx, t0)
    vel = np.ascontiguousarray(vel, dtype=np.float64).reshape(P, 3)
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
    N = pts.shape[0]
    out = np.zeros((N, 2), dtype=np.float64)
    cnt = np.zeros(N, dtype=np.int64) if with_count else None
    rc = lib.oracle_tdbp_points_motion(_p(echoes, ctypes.c_float), P, E, Ns, _p(tx, ctypes.c_double),
                                       _p(rx, ctypes.c_double), _p(t0, ctypes.c_double), _p(vel, ctypes.c_double),
                                       float(fc), float(fs), float(c), _p(pts, ctypes.c_double), N,
                                       _p(out, ctypes.c_double), _p(cnt, ctypes.c_int64))
    if rc != 0:
        raise ValueError("oracle_tdbp_points_motion: invalid arguments")
    res = out[:, 0] + 1j * out[:, 1]
    return (res, cnt) if with_count else res


def tdbp_points_nav(echoes, tx, lut, dt, t0, fc, fs, c, pts, with_count=False):
    """TDBP with each receiver on its tabled trajectory lut [P][E][K][3] (nodes dt apart from the
    transmit; NEXT-2, reading R23)."""
    lib = _load()
    echoes = np.ascontiguousarray(echoes, dtype=np.complex64)
    P, E, Ns = echoes.shape
    tx = np.ascontiguousarray(tx, dtype=np.float64).reshape(P, 3)
    lut = np.ascontiguousarray(lut, dtype=np.float64)
    K = lut.shape[-2]
    lut = lut.reshape(P, E, K, 3)
    t0a = None if t0 is None else np.ascontiguousarray(t0, dtype=np.float64).reshape(P)
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
    N = pts.shape[0]
    out = np.zeros((N, 2), dtype=np.float64)
    cnt = np.zeros(N, dtype=np.int64) if with_count else None
    rc = lib.oracle_tdbp_points_nav(_p(echoes.view(np.float32), ctypes.c_float), P, E, Ns, _p(tx, ctypes.c_double),
                                    _p(lut, ctypes.c_double), K, float(dt),
                                    None if t0a is None else _p(t0a, ctypes.c_double), float(fc), float(fs), float(c),
                                    _p(pts, ctypes.c_double), N, _p(out, ctypes.c_double),
                                    None if cnt is None else _p(cnt, ctypes.c_int64))
    if rc != 0:
        raise ValueError("oracle_tdbp_points_nav: invalid arguments")
    res = out[:, 0] + 1j * out[:, 1]
    return (res, cnt) if with_count else res


def tdbp_points_gated_nav(echoes, tx, rx, lut, dt, t0, fc, fs, c, pts, az, el=0.0, bistatic=False, axes=None,
                          with_count=False):
    """Gated (R15) TDBP with tabled receiver trajectories (R23); gate on the recorded positions (R22)."""
    lib = _load()
    echoes, P, E, Ns, tx, rx, t0 = _echo_arrays(echoes, tx, rx, t0)
    lut = np.ascontiguousarray(lut, dtype=np.float64)
    K = lut.shape[-2]
    lut = lut.reshape(P, E, K, 3)
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
    ax = None if axes is None else np.ascontiguousarray(axes, dtype=np.float64).reshape(P, 2, 3)
    N = pts.shape[0]
    out = np.zeros((N, 2), dtype=np.float64)
    cnt = np.zeros(N, dtype=np.int64) if with_count else None
    rc = lib.oracle_tdbp_points_gated_nav(_p(echoes, ctypes.c_float), P, E, Ns, _p(tx, ctypes.c_double),
                                          _p(rx, ctypes.c_double), _p(lut, ctypes.c_double), K, float(dt),
                                          _p(t0, ctypes.c_double), float(fc), float(fs), float(c),
                                          _p(ax, ctypes.c_double), float(az), float(el), 1 if bistatic else 0,
                                          _p(pts, ctypes.c_double), N, _p(out, ctypes.c_double),
                                          _p(cnt, ctypes.c_int64))
    if rc != 0:
        raise ValueError("oracle_tdbp_points_gated_nav: invalid arguments")
    res = out[:, 0] + 1j * out[:, 1]
    return (res, cnt) if with_count else res


def nav_eval(lut, dt, t):
    """The R23 trajectory interpolant of one (ping, element) table lut [K][3] at time t."""
    lut = np.ascontiguousarray(lut, dtype=np.float64).reshape(-1, 3)
    r = np.zeros(3)
    _load().oracle_nav_eval(_p(lut, ctypes.c_double), lut.shape[0], float(dt), float(t), _p(r, ctypes.c_double))
    return r


def delay_nav(x, tx, lut, dt, c):
    """The R23 two-way delay of one point / transmitter / receiver table."""
    a = [np.ascontiguousarray(q, dtype=np.float64).reshape(3) for q in (x, tx)]
    lut = np.ascontiguousarray(lut, dtype=np.float64).reshape(-1, 3)
    return float(_load().oracle_delay_nav(_p(a[0], ctypes.c_double), _p(a[1], ctypes.c_double),
                                          _p(lut, ctypes.c_double), lut.shape[0], float(dt), float(c)))


def tdbp_points_refracted(echoes, tx, rx, t0, zb, c2, fc, fs, c, pts, with_count=False):
    """TDBP through a flat sediment-water interface z = zb (sediment speed c2, water speed c)."""
    lib = _load()
    echoes, P, E, Ns, tx, rx, t0 = _echo_arrays(echoes, tx, rx, t0)
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
    N = pts.shape[0]
    out = np.zeros((N, 2), dtype=np.float64)
    cnt = np.zeros(N, dtype=np.int64) if with_count else None
    rc = lib.oracle_tdbp_points_refracted(_p(echoes, ctypes.c_float), P, E, Ns, _p(tx, ctypes.c_double),
                                          _p(rx, ctypes.c_double), _p(t0, ctypes.c_double), float(zb), float(c2),
                                          float(fc), float(fs), float(c), _p(pts, ctypes.c_double), N,
                                          _p(out, ctypes.c_double), _p(cnt, ctypes.c_int64))
    if rc != 0:
        raise ValueError("oracle_tdbp_points_refracted: invalid arguments")
    res = out[:, 0] + 1j * out[:, 1]
    return (res, cnt) if with_count else res


def travel_refracted(x, s, zb, c1, c2):
    lib = _load()
    a = [np.ascontiguousarray(q, dtype=np.float64).reshape(3) for q in (x, s)]
    return float(lib.oracle_travel_refracted(_p(a[0], ctypes.c_double), _p(a[1], ctypes.c_double), float(zb),
                                             float(c1), float(c2)))


def delay_moving(x, tx, rx, v, c):
    lib = _load()
    a = [np.ascontiguousarray(q, dtype=np.float64).reshape(3) for q in (x, tx, rx, v)]
    return float(lib.oracle_delay_moving(*[_p(q, ctypes.c_double) for q in a], float(c)))


def grid_points(grid, idx=None):
    """Pixel centres (reading R8) of index triples idx [N][3] (None = full grid, z-y-x order)."""
    if idx is None:
        iz, iy, ix = np.meshgrid(np.arange(grid["nz"]), np.arange(grid["ny"]), np.arange(grid["nx"]), indexing="ij")
        idx = np.stack([ix.ravel(), iy.ravel(), iz.ravel()], axis=1)
    idx = np.asarray(idx, dtype=np.float64).reshape(-1, 3)
    g = {k: np.asarray(grid[k], dtype=np.float64) for k in ("origin", "step_x", "step_y", "step_z")}
    return (g["origin"][None] + idx[:, :1] * g["step_x"][None] + idx[:, 1:2] * g["step_y"][None]
            + idx[:, 2:3] * g["step_z"][None])


def tdbp_grid(echoes, tx, rx, t0, fc, fs, c, grid, idx=None, with_count=False):
    """I at grid pixels.  ``grid`` is a dict with origin, step_x, step_y, step_z (3-vectors)
    and nx, ny, nz.  ``idx`` is an int64 [N][3] array of (ix, iy, iz); None = full grid,
    returned as [nz][ny][nx]."""
    lib = _load()
    echoes, P, E, Ns, tx, rx, t0 = _echo_arrays(echoes, tx, rx, t0)
    full = idx is None
    if full:
        iz, iy, ix = np.meshgrid(np.arange(grid["nz"]), np.arange(grid["ny"]), np.arange(grid["nx"]),
                                 indexing="ij")
        idx = np.stack([ix.ravel(), iy.ravel(), iz.ravel()], axis=1)
    idx = np.ascontiguousarray(idx, dtype=np.int64).reshape(-1, 3)
    N = idx.shape[0]
    vec = {k: np.ascontiguousarray(grid[k], dtype=np.float64).reshape(3)
           for k in ("origin", "step_x", "step_y", "step_z")}
    out = np.zeros((N, 2), dtype=np.float64)
    cnt = np.zeros(N, dtype=np.int64) if with_count else None
    rc = lib.oracle_tdbp_grid_pixels(_p(echoes, ctypes.c_float), P, E, Ns, _p(tx, ctypes.c_double),
                                     _p(rx, ctypes.c_double), _p(t0, ctypes.c_double), float(fc),
                                     float(fs), float(c), _p(vec["origin"], ctypes.c_double),
                                     _p(vec["step_x"], ctypes.c_double),
                                     _p(vec["step_y"], ctypes.c_double),
                                     _p(vec["step_z"], ctypes.c_double), _p(idx, ctypes.c_int64), N,
                                     _p(out, ctypes.c_double), _p(cnt, ctypes.c_int64))
    if rc != 0:
        raise ValueError("oracle_tdbp_grid_pixels: invalid arguments")
    res = out[:, 0] + 1j * out[:, 1]
    if full:
        res = res.reshape(grid["nz"], grid["ny"], grid["nx"])
        if cnt is not None:
            cnt = cnt.reshape(grid["nz"], grid["ny"], grid["nx"])
    return (res, cnt) if with_count else res


def rangecompress(raw, replica):
    """Direct fp64 correlation y[n] = sum_m x[n+m] conj(r[m]) per channel; raw complex64 [..., Ns]."""
    lib = _load()
    raw = np.ascontiguousarray(raw, dtype=np.complex64)
    replica = np.ascontiguousarray(replica, dtype=np.complex64).ravel()
    shape = raw.shape
    Ns = shape[-1]
    nch = int(np.prod(shape[:-1])) if len(shape) > 1 else 1
    out = np.zeros((nch, Ns, 2), dtype=np.float64)
    rc = lib.oracle_rangecompress(_p(raw.view(np.float32), ctypes.c_float), nch, Ns,
                                  _p(replica.view(np.float32), ctypes.c_float), replica.size,
                                  _p(out, ctypes.c_double))
    if rc != 0:
        raise ValueError("oracle_rangecompress: invalid arguments")
    return (out[..., 0] + 1j * out[..., 1]).reshape(shape)


def tdbp_points_weighted(echoes, tx, rx, t0, fc, fs, c, pts, with_count=False):
    """Spreading-compensated TDBP (NEXT-4, R18): every term times R_tx * R_rx."""
    lib = _load()
    echoes, P, E, Ns, tx, rx, t0 = _echo_arrays(echoes, tx, rx, t0)
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
    N = pts.shape[0]
    out = np.zeros((N, 2), dtype=np.float64)
    cnt = np.zeros(N, dtype=np.int64) if with_count else None
    rc = lib.oracle_tdbp_points_weighted(_p(echoes, ctypes.c_float), P, E, Ns, _p(tx, ctypes.c_double),
                                         _p(rx, ctypes.c_double), _p(t0, ctypes.c_double), float(fc),
                                         float(fs), float(c), _p(pts, ctypes.c_double), N,
                                         _p(out, ctypes.c_double), _p(cnt, ctypes.c_int64))
    if rc != 0:
        raise ValueError("oracle_tdbp_points_weighted: invalid arguments")
    res = out[:, 0] + 1j * out[:, 1]
    return (res, cnt) if with_count else res


def tdbp_points_gated_weighted(echoes, tx, rx, t0, fc, fs, c, pts, az, el=0.0, bistatic=False, axes=None):
    """Gated (R15) and spreading-weighted (R18) TDBP at explicit points."""
    lib = _load()
    echoes, P, E, Ns, tx, rx, t0 = _echo_arrays(echoes, tx, rx, t0)
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
    ax = None if axes is None else np.ascontiguousarray(axes, dtype=np.float64).reshape(P, 2, 3)
    N = pts.shape[0]
    out = np.zeros((N, 2), dtype=np.float64)
    rc = lib.oracle_tdbp_points_gated_weighted(_p(echoes, ctypes.c_float), P, E, Ns, _p(tx, ctypes.c_double),
                                               _p(rx, ctypes.c_double), _p(t0, ctypes.c_double), float(fc), float(fs),
                                               float(c), _p(ax, ctypes.c_double), float(az), float(el),
                                               1 if bistatic else 0, _p(pts, ctypes.c_double), N,
                                               _p(out, ctypes.c_double))
    if rc != 0:
        raise ValueError("oracle_tdbp_points_gated_weighted: invalid arguments")
    return out[:, 0] + 1j * out[:, 1]


def tdbp_points_gated_motion(echoes, tx, rx, t0, vel, fc, fs, c, pts, az, el=0.0, bistatic=False, axes=None,
                             with_count=False):
    """Gated (R15) TDBP with the moving-receiver delay (R16); gate on transmit-time positions (R22)."""
    lib = _load()
    echoes, P, E, Ns, tx, rx, t0 = _echo_arrays(echoes, tx, rx, t0)
    vel = np.ascontiguousarray(vel, dtype=np.float64).reshape(P, 3)
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
    ax = None if axes is None else np.ascontiguousarray(axes, dtype=np.float64).reshape(P, 2, 3)
    N = pts.shape[0]
    out = np.zeros((N, 2), dtype=np.float64)
    cnt = np.zeros(N, dtype=np.int64) if with_count else None
    rc = lib.oracle_tdbp_points_gated_motion(_p(echoes, ctypes.c_float), P, E, Ns, _p(tx, ctypes.c_double),
                                             _p(rx, ctypes.c_double), _p(t0, ctypes.c_double),
                                             _p(vel, ctypes.c_double), float(fc), float(fs), float(c),
                                             _p(ax, ctypes.c_double), float(az), float(el), 1 if bistatic else 0,
                                             _p(pts, ctypes.c_double), N, _p(out, ctypes.c_double),
                                             _p(cnt, ctypes.c_int64))
    if rc != 0:
        raise ValueError("oracle_tdbp_points_gated_motion: invalid arguments")
    res = out[:, 0] + 1j * out[:, 1]
    return (res, cnt) if with_count else res


def tdbp_points_gated_refracted(echoes, tx, rx, t0, zb, c2, fc, fs, c, pts, az, el=0.0, bistatic=False,
                                axes=None, with_count=False):
    """Gated (R15) TDBP with the Fermat delay through a flat interface (R17); straight line-of-sight
    gate from the recorded sensor positions (R22)."""
    lib = _load()
    echoes, P, E, Ns, tx, rx, t0 = _echo_arrays(echoes, tx, rx, t0)
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
    ax = None if axes is None else np.ascontiguousarray(axes, dtype=np.float64).reshape(P, 2, 3)
    N = pts.shape[0]
    out = np.zeros((N, 2), dtype=np.float64)
    cnt = np.zeros(N, dtype=np.int64) if with_count else None
    rc = lib.oracle_tdbp_points_gated_refracted(_p(echoes, ctypes.c_float), P, E, Ns, _p(tx, ctypes.c_double),
                                                _p(rx, ctypes.c_double), _p(t0, ctypes.c_double), float(zb),
                                                float(c2), float(fc), float(fs), float(c), _p(ax, ctypes.c_double),
                                                float(az), float(el), 1 if bistatic else 0,
                                                _p(pts, ctypes.c_double), N, _p(out, ctypes.c_double),
                                                _p(cnt, ctypes.c_int64))
    if rc != 0:
        raise ValueError("oracle_tdbp_points_gated_refracted: invalid arguments")
    res = out[:, 0] + 1j * out[:, 1]
    return (res, cnt) if with_count else res


def lanczos4(s) -> float:
    """The 8-tap interpolation kernel L(s) = sinc(s) sinc(s/4), |s| < 4 (R19)."""
    return float(_load().oracle_lanczos4(float(s)))


def upsample(x, U):
    """xU band-limited upsampling by the 8-tap kernel (R19); x complex64 [..., Ns] ->
    complex128 [..., U*Ns] at rate U*fs, same t0."""
    lib = _load()
    x = np.ascontiguousarray(x, dtype=np.complex64)
    shape = x.shape
    Ns = shape[-1]
    nch = int(np.prod(shape[:-1])) if len(shape) > 1 else 1
    out = np.zeros((nch, U * Ns, 2), dtype=np.float64)
    rc = lib.oracle_upsample(_p(x.view(np.float32), ctypes.c_float), nch, Ns, int(U), _p(out, ctypes.c_double))
    if rc != 0:
        raise ValueError("oracle_upsample: invalid arguments")
    return (out[..., 0] + 1j * out[..., 1]).reshape(shape[:-1] + (U * Ns,))


def baseband(x, fs_in, fc, t0, h, D, Nout):
    """Real passband [P][E][Nin] -> complex baseband [P][E][Nout] (R20): mix by
    exp(-j 2 pi fc (t0_p + n/fs_in)), centred FIR h (odd length), keep every D-th sample."""
    lib = _load()
    x = np.ascontiguousarray(x, dtype=np.float32)
    if x.ndim != 3:
        raise ValueError("x must be float32 [P][E][Nin]")
    P, E, Nin = x.shape
    h = np.ascontiguousarray(h, dtype=np.float32).ravel()
    t0 = None if t0 is None else np.ascontiguousarray(t0, dtype=np.float64).reshape(P)
    out = np.zeros((P, E, Nout, 2), dtype=np.float64)
    rc = lib.oracle_baseband(_p(x, ctypes.c_float), P, E, Nin, float(fs_in), float(fc), _p(t0, ctypes.c_double),
                             _p(h, ctypes.c_float), h.size, int(D), int(Nout), _p(out, ctypes.c_double))
    if rc != 0:
        raise ValueError("oracle_baseband: invalid arguments")
    return out[..., 0] + 1j * out[..., 1]


def whitening_gain(raw, M, gamma):
    """Eq. 9 whitening gain (R21): batch-mean M-point periodogram P of complex64 [..., Ns] and
    G = h(1/(gamma mean P + P)), max G = 1.  Returns (G, P), fp64 [M] each."""
    lib = _load()
    raw = np.ascontiguousarray(raw, dtype=np.complex64)
    Ns = raw.shape[-1]
    nch = int(np.prod(raw.shape[:-1])) if raw.ndim > 1 else 1
    G = np.zeros(M, dtype=np.float64)
    P = np.zeros(M, dtype=np.float64)
    rc = lib.oracle_whitening_gain(_p(raw.view(np.float32), ctypes.c_float), nch, Ns, int(M), float(gamma),
                                   _p(G, ctypes.c_double), _p(P, ctypes.c_double))
    if rc == -2:
        raise ValueError("oracle_whitening_gain: no spectrum (all-zero batch)")
    if rc != 0:
        raise ValueError("oracle_whitening_gain: invalid arguments")
    return G, P


def rangecompress_whitened(raw, replica, G):
    """Whitening FIR (frequency sampling of G over one centred period) then the matched filter
    (R21 + R14); complex64 [..., Ns] -> complex128 of the same shape."""
    lib = _load()
    raw = np.ascontiguousarray(raw, dtype=np.complex64)
    replica = np.ascontiguousarray(replica, dtype=np.complex64).ravel()
    G = np.ascontiguousarray(G, dtype=np.float64).ravel()
    shape = raw.shape
    Ns = shape[-1]
    nch = int(np.prod(shape[:-1])) if len(shape) > 1 else 1
    out = np.zeros((nch, Ns, 2), dtype=np.float64)
    rc = lib.oracle_rangecompress_whitened(_p(raw.view(np.float32), ctypes.c_float), nch, Ns,
                                           _p(replica.view(np.float32), ctypes.c_float), replica.size,
                                           _p(G, ctypes.c_double), G.size, _p(out, ctypes.c_double))
    if rc != 0:
        raise ValueError("oracle_rangecompress_whitened: invalid arguments")
    return (out[..., 0] + 1j * out[..., 1]).reshape(shape)


def num_threads() -> int:
    return int(_load().oracle_num_threads())
