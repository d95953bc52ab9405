"""Seeded synthetic scenarios for the TDBP hot path (inputs only).

This module is the ONE place both the CUDA path's tests/bench and the oracle get
their inputs from.  It contains the scene/trajectory recipe of SURVEY §8(d)
("Synthetic inputs") and DESIGN.md §"Input recipe", the Eq. 2 attitude rotation
(PAPER.md eqn:rollpitchyaw) used to place lever arms, and a C
forward-model echo synthesiser (synth.c).  It holds none of the backprojection
method's arithmetic (no interpolation, no phase ramp, no accumulation).

Configs (BASELINE.json ``configs``):
  1  single point target, 64 pings, 1 tx + 4 rx, 2048 samples, 128x128 2D (oracle in seconds)
  2  2D stripmap, 1000 pings, 32 rx, 5 targets + speckle, 4096x4096 (the bench workload)
  3  high-motion (sway/heave/yaw/roll/pitch), 2000 pings, 32 rx, 8192x4096
  4  3D near-field volumetric, 8x32 downward rx array, 1000 pings, 512x512x128
  5  full swath 16384^2, 4000 pings x 64 rx (58.7 GB of echoes; definition only)
Every config also has a ``reduced`` form (same physics, fewer pings/elements and a
small ragged grid) that the oracle evaluates in seconds.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "synth.c")
_LIB = os.path.join(_HERE, "libsynth.so")
_lib = None

C_WATER = 1500.0


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        f64p = ctypes.POINTER(ctypes.c_double)
        lib.synth_echoes.argtypes = [ctypes.POINTER(ctypes.c_float), ctypes.c_int32, ctypes.c_int32,
                                     ctypes.c_int32, f64p, f64p, f64p, f64p, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_int32, f64p, f64p, ctypes.c_int64, ctypes.c_double, f64p,
                                     ctypes.c_int32, ctypes.c_double, ctypes.c_double]
        lib.synth_echoes.restype = ctypes.c_int
        _lib = lib
    return _lib


def rotation_matrix(roll: float, pitch: float, yaw: float) -> np.ndarray:
    """Eq. (eqn:rollpitchyaw), written out literally.

    phi = roll, theta = pitch, psi = yaw (radians); maps body-frame vectors to NED.
    """
    ph, th, ps = roll, pitch, yaw
    c, s = np.cos, np.sin
    return np.array([
        [c(th) * c(ps), c(ps) * s(th) * s(ph) - c(ph) * s(ps), c(ph) * c(ps) * s(th) + s(ph) * s(ps)],
        [c(th) * s(ps), c(ph) * c(ps) + s(th) * s(ph) * s(ps), c(ph) * s(th) * s(ps) - c(ps) * s(ph)],
        [-s(th), c(th) * s(ph), c(th) * c(ph)],
    ])


@dataclasses.dataclass
class Scenario:
    """One seeded synthetic collection + imaging grid (all SI units, NED metres)."""
    name: str
    fc: float
    bandwidth: float
    fs: float
    c: float
    tx: np.ndarray            # [P][3]
    rx: np.ndarray            # [P][E][3]
    t0: np.ndarray            # [P] seconds after transmit of sample 0
    Ns: int
    grid: dict                # origin, step_x, step_y, step_z (3-vectors), nx, ny, nz
    targets: np.ndarray       # [T][3] point targets (sigma = 1)
    target_pixels: np.ndarray  # [T][3] (ix, iy, iz) of each target
    scat: np.ndarray          # [S][3] all scatterers (targets first)
    sigma: np.ndarray         # [S] complex128 amplitudes
    sin_half_beam: float      # generator gate; 0 = omni
    body_rot: Optional[np.ndarray] = None  # [P][3][3]
    half_support: int = 16
    nav_nominal: Optional[tuple] = None   # (tx, rx) unperturbed nav (cfg 3)
    vel: Optional[np.ndarray] = None      # [P][3] platform velocity during reception (None = stop-and-hop)
    medium: Optional[tuple] = None        # (zb, c2): flat sediment interface z = zb, sediment speed c2

    @property
    def P(self):
        return self.tx.shape[0]

    @property
    def E(self):
        return self.rx.shape[1]

    @property
    def n_pixels(self):
        return self.grid["nx"] * self.grid["ny"] * self.grid["nz"]

    @property
    def dense_terms(self):
        return self.n_pixels * self.P * self.E

    def echoes(self) -> np.ndarray:
        """complex64 [P][E][Ns] range-compressed basebanded echoes (forward model, synth.c)."""
        lib = _load()
        P, E, Ns = self.P, self.E, self.Ns
        out = np.zeros((P, E, Ns, 2), dtype=np.float32)
        f64 = lambda a: np.ascontiguousarray(a, dtype=np.float64)
        tx, rx, t0, scat = f64(self.tx), f64(self.rx), f64(self.t0), f64(self.scat)
        sig = f64(np.stack([self.sigma.real, self.sigma.imag], axis=1))
        rot = f64(self.body_rot.reshape(P, 9)) if self.body_rot is not None else None
        vel = f64(self.vel.reshape(P, 3)) if self.vel is not None else None
        ptr = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if a is not None else None
        rc = lib.synth_echoes(out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), P, E, Ns, ptr(tx),
                              ptr(rx), ptr(t0), ptr(rot), self.fc, self.bandwidth, self.fs, self.c,
                              self.half_support, ptr(scat), ptr(sig), scat.shape[0],
                              self.sin_half_beam, ptr(vel), 1 if self.medium else 0,
                              float(self.medium[0]) if self.medium else 0.0,
                              float(self.medium[1]) if self.medium else 0.0)
        if rc != 0:
            raise ValueError("synth_echoes failed")
        return out.view(np.complex64).reshape(P, E, Ns)

    def subset_pings(self, idx) -> "Scenario":
        """The same scene and grid observed by a subset of the pings (for bounded test sizes)."""
        idx = np.asarray(idx)
        return dataclasses.replace(self, name=f"{self.name}[{len(idx)} pings]", tx=self.tx[idx], rx=self.rx[idx],
                                   t0=self.t0[idx],
                                   body_rot=None if self.body_rot is None else self.body_rot[idx],
                                   vel=None if self.vel is None else self.vel[idx],
                                   nav_nominal=None if self.nav_nominal is None else
                                   (self.nav_nominal[0][idx], self.nav_nominal[1][idx]))

    def pixel_centre(self, idx) -> np.ndarray:
        idx = np.asarray(idx, dtype=np.float64).reshape(-1, 3)
        g = self.grid
        return (np.asarray(g["origin"])[None] + idx[:, :1] * np.asarray(g["step_x"])[None]
                + idx[:, 1:2] * np.asarray(g["step_y"])[None] + idx[:, 2:3] * np.asarray(g["step_z"])[None])

    def sample_pixels(self, n_random: int, window: int = 15, seed: int = 0) -> np.ndarray:
        """SURVEY §8(c) compared-pixel set: n_random seeded pixels + a window^2 (window^3 in 3D)
        patch around every point target, clipped to the grid.  int64 [N][3]."""
        g = self.grid
        rng = np.random.default_rng(seed)
        rnd = np.stack([rng.integers(0, g["nx"], n_random), rng.integers(0, g["ny"], n_random),
                        rng.integers(0, g["nz"], n_random)], axis=1)
        h = window // 2
        parts = [rnd]
        for t in self.target_pixels:
            rz = range(-h, h + 1) if g["nz"] > 1 else [0]
            o = np.array([(dx, dy, dz) for dz in rz for dy in range(-h, h + 1) for dx in range(-h, h + 1)])
            q = t[None] + o
            keep = ((q[:, 0] >= 0) & (q[:, 0] < g["nx"]) & (q[:, 1] >= 0) & (q[:, 1] < g["ny"])
                    & (q[:, 2] >= 0) & (q[:, 2] < g["nz"]))
            parts.append(q[keep])
        return np.ascontiguousarray(np.concatenate(parts, axis=0).astype(np.int64))


def grid_dict(origin, step, n):
    """Axis-aligned grid: pixel (0,0,0) centred at ``origin`` (reading R8)."""
    sx, sy, sz = step
    return {"origin": np.asarray(origin, dtype=np.float64), "step_x": np.array([sx, 0.0, 0.0]),
            "step_y": np.array([0.0, sy, 0.0]), "step_z": np.array([0.0, 0.0, sz]),
            "nx": int(n[0]), "ny": int(n[1]), "nz": int(n[2])}


def _snap(grid, pts):
    """Snap points to the nearest pixel centre; return (points, pixel indices)."""
    o = np.asarray(grid["origin"])
    st = np.array([grid["step_x"][0], grid["step_y"][1], grid["step_z"][2]])
    st = np.where(st == 0, 1.0, st)
    idx = np.rint((np.asarray(pts, dtype=np.float64) - o[None]) / st[None]).astype(np.int64)
    return o[None] + idx * st[None], idx


def _speckle(rng, n, lo, hi, rms):
    pos = rng.uniform(lo, hi, size=(n, 3))
    sig = (rng.normal(size=n) + 1j * rng.normal(size=n)) * (rms / np.sqrt(2.0))
    return pos, sig


def _ar1(rng, n, std, a=0.99):
    """Band-limited random walk: stationary AR(1) with the given standard deviation."""
    x = np.zeros(n)
    w = rng.normal(size=n) * std * np.sqrt(1 - a * a)
    x[0] = rng.normal() * std
    for i in range(1, n):
        x[i] = a * x[i - 1] + w[i]
    return x


def stripmap(name, *, P, E, D, fc, B, fs, altitude, track, grid, Ns, t0, targets, n_speckle,
             speckle_rms=0.05, motion=None, seed=0, c=C_WATER, half_support=16):
    """Side-looking (starboard, +y) stripmap collection; element lever arms along body +x at
    pitch D centred on the transmitter; hard azimuth fan-beam gate FWHM 0.886*lambda/D."""
    rng = np.random.default_rng(seed)
    xs = np.linspace(track[0], track[1], P)
    base = np.stack([xs, np.zeros(P), np.full(P, -altitude)], axis=1)
    lever = np.stack([(np.arange(E) - (E - 1) / 2.0) * D, np.zeros(E), np.zeros(E)], axis=1)
    nominal_tx = base.copy()
    nominal_rx = base[:, None, :] + lever[None]
    rot = None
    if motion is not None:
        pp = np.arange(P)
        sway = motion["sway"] * np.sin(2 * np.pi * pp / 137.0) + _ar1(rng, P, motion["sway_rw"])
        heave = motion["heave"] * np.sin(2 * np.pi * pp / 91.0) + _ar1(rng, P, motion["heave_rw"])
        yaw = np.deg2rad(motion["yaw_deg"]) * np.sin(2 * np.pi * pp / 211.0) + _ar1(
            rng, P, np.deg2rad(motion["yaw_rw_deg"]))
        roll = _ar1(rng, P, np.deg2rad(motion["roll_deg"]))
        pitch = _ar1(rng, P, np.deg2rad(motion["pitch_deg"]))
        base = base + np.stack([np.zeros(P), sway, heave], axis=1)
        rot = np.stack([rotation_matrix(roll[i], pitch[i], yaw[i]) for i in range(P)])
        tx = base.copy()
        rx = base[:, None, :] + np.einsum("pij,ej->pei", rot, lever)
    else:
        tx = nominal_tx.copy()
        rx = nominal_rx.copy()
    tpos, tpix = _snap(grid, targets)
    g = grid
    lo = np.asarray(g["origin"]) - 0.5 * np.array([g["step_x"][0], g["step_y"][1], 0.0])
    hi = lo + np.array([g["nx"] * g["step_x"][0], g["ny"] * g["step_y"][1], 0.0])
    spos, ssig = _speckle(rng, n_speckle, lo, hi, speckle_rms)
    lam = c / fc
    theta = 0.886 * lam / D
    return Scenario(name=name, fc=fc, bandwidth=B, fs=fs, c=c, tx=tx, rx=rx,
                    t0=np.full(P, float(t0)), Ns=int(Ns), grid=g, targets=tpos, target_pixels=tpix,
                    scat=np.concatenate([tpos, spos], axis=0),
                    sigma=np.concatenate([np.ones(len(tpos), dtype=np.complex128), ssig]),
                    sin_half_beam=float(np.sin(theta / 2)), body_rot=rot, half_support=half_support,
                    nav_nominal=(nominal_tx, nominal_rx) if motion is not None else None)


HF = dict(fc=120e3, B=30e3, fs=120e3, D=0.04)   # lambda = 12.5 mm, fs = 4B


def _cfg1(reduced=False, seed=1001):
    tgt = np.array([[2.56, 11.18, 0.0]])
    step = 0.0025
    n = 128 if not reduced else 48
    origin = tgt[0] - np.array([n // 2 * step, n // 2 * step, 0.0])
    grid = grid_dict(origin, (step, step, 1.0), (n, n, 1))
    P = 64
    xs = 2.56 + (np.arange(P) - (P - 1) / 2.0) * 0.08
    return stripmap("cfg1", P=P, E=4, **HF, altitude=10.0, track=(xs[0], xs[-1]), grid=grid,
                    Ns=2048, t0=0.012, targets=tgt, n_speckle=0, seed=seed)


def _cfg2(reduced=False, seed=1002):
    if not reduced:
        grid = grid_dict((0.0, 20.0, 0.0), (0.01, 0.01, 1.0), (4096, 4096, 1))
        fr = [(0.25, 0.25), (0.75, 0.25), (0.5, 0.5), (0.25, 0.75), (0.75, 0.75)]
        tg = np.array([[f[0] * 40.96, 20.0 + f[1] * 40.96, 0.0] for f in fr])
        return stripmap("cfg2", P=1000, E=32, **HF, altitude=10.0, track=(-8.6, 49.6), grid=grid,
                        Ns=10240, t0=2 * 20.0 / C_WATER, targets=tg, n_speckle=1 << 16, seed=seed)
    # reduced: 200 x 150 ragged grid (several 32x32 tiles + tails), 40 pings x 8 elements
    grid = grid_dict((19.0, 30.0, 0.0), (0.01, 0.01, 1.0), (200, 150, 1))
    tg = np.array([[19.5, 30.6, 0.0], [20.4, 31.1, 0.0]])
    return stripmap("cfg2r", P=40, E=8, **HF, altitude=10.0, track=(15.0, 24.0), grid=grid,
                    Ns=4096, t0=2 * 20.0 / C_WATER, targets=tg, n_speckle=512, seed=seed)


MOTION3 = dict(sway=0.3, sway_rw=0.1, heave=0.1, heave_rw=0.03, yaw_deg=3.0, yaw_rw_deg=0.5,
               roll_deg=1.0, pitch_deg=1.0)


def _cfg3(reduced=False, seed=1003):
    if not reduced:
        grid = grid_dict((0.0, 20.0, 0.0), (0.01, 0.01, 1.0), (8192, 4096, 1))
        fr = [(0.25, 0.25), (0.75, 0.25), (0.5, 0.5), (0.25, 0.75), (0.75, 0.75)]
        tg = np.array([[f[0] * 81.92, 20.0 + f[1] * 40.96, 0.0] for f in fr])
        return stripmap("cfg3", P=2000, E=32, **HF, altitude=10.0, track=(-8.6, 90.52), grid=grid,
                        Ns=16384, t0=2 * 20.0 / C_WATER, targets=tg, n_speckle=1 << 16,
                        motion=MOTION3, seed=seed)
    grid = grid_dict((19.0, 24.0, 0.0), (0.01, 0.01, 1.0), (96, 130, 1))
    tg = np.array([[19.4, 24.6, 0.0]])
    return stripmap("cfg3r", P=48, E=8, **HF, altitude=10.0, track=(14.0, 25.0), grid=grid,
                    Ns=4096, t0=2 * 20.0 / C_WATER, targets=tg, n_speckle=256, motion=MOTION3,
                    seed=seed)


def _cfg4(reduced=False, seed=1004):
    """Near-field 3D sub-bottom (P:307-319 analog): downward-looking 8x32 rx array at
    lambda/2 = 3 cm + 1 tx at centre, 2 m altitude, 25 x 40 raster over 6 x 6 m."""
    rng = np.random.default_rng(seed)
    fc, B, fs = 25e3, 20e3, 80e3
    nl, npl = (25, 40) if not reduced else (4, 5)
    P = nl * npl
    pp = np.arange(P)
    if not reduced:
        xs = 0.075 + (pp % npl) * 0.15
        ys = 0.12 + (pp // npl) * 0.24
        grid = grid_dict((0.44, 0.44, 0.0), (0.01, 0.01, 0.01), (512, 512, 128))
        ax, ay = 8, 32
        n_speckle = 1 << 9
        tg = np.array([[1.5, 1.5, 0.11], [1.5, 4.5, 0.11], [4.5, 1.5, 0.11], [4.5, 4.5, 0.11],
                       [3.0, 2.0, 0.5], [3.0, 4.0, 0.5]])
    else:
        xs = 2.7 + (pp % npl) * 0.15
        ys = 2.64 + (pp // npl) * 0.24
        grid = grid_dict((2.8, 2.9, 0.05), (0.01, 0.01, 0.01), (40, 36, 20))
        ax, ay = 4, 8
        n_speckle = 64
        tg = np.array([[3.0, 3.1, 0.11]])
    tx = np.stack([xs, ys, np.full(P, -2.0)], axis=1)
    ii, jj = np.meshgrid(np.arange(ax), np.arange(ay), indexing="ij")
    lever = np.stack([(ii.ravel() - (ax - 1) / 2) * 0.03, (jj.ravel() - (ay - 1) / 2) * 0.03,
                      np.zeros(ax * ay)], axis=1)
    rx = tx[:, None, :] + lever[None]
    tpos, tpix = _snap(grid, tg)
    g = grid
    lo = np.asarray(g["origin"]) - 0.5 * np.array([g["step_x"][0], g["step_y"][1], g["step_z"][2]])
    hi = lo + np.array([g["nx"] * g["step_x"][0], g["ny"] * g["step_y"][1], g["nz"] * g["step_z"][2]])
    spos, ssig = _speckle(rng, n_speckle, lo, hi, 0.05)
    return Scenario(name="cfg4" if not reduced else "cfg4r", fc=fc, bandwidth=B, fs=fs, c=C_WATER,
                    tx=tx, rx=rx, t0=np.full(P, 2.53e-3), Ns=1024, grid=grid, targets=tpos,
                    target_pixels=tpix, scat=np.concatenate([tpos, spos], axis=0),
                    sigma=np.concatenate([np.ones(len(tpos), dtype=np.complex128), ssig]),
                    sin_half_beam=0.0)


def _cfg5(reduced=False, seed=1005):
    if not reduced:
        grid = grid_dict((0.0, 20.0, 0.0), (0.01, 0.01, 1.0), (16384, 16384, 1))
        fr = [(0.25, 0.25), (0.75, 0.25), (0.5, 0.5), (0.25, 0.75), (0.75, 0.75)]
        tg = np.array([[f[0] * 163.84, 20.0 + f[1] * 163.84, 0.0] for f in fr])
        return stripmap("cfg5", P=4000, E=64, **HF, altitude=15.0, track=(-25.7, 189.54), grid=grid,
                        Ns=28672, t0=2 * 24.5 / C_WATER, targets=tg, n_speckle=1 << 16, seed=seed)
    grid = grid_dict((60.0, 150.0, 0.0), (0.01, 0.01, 1.0), (70, 97, 1))
    tg = np.array([[60.3, 150.5, 0.0]])
    return stripmap("cfg5r", P=24, E=16, **HF, altitude=15.0, track=(48.0, 72.0), grid=grid,
                    Ns=28672, t0=2 * 24.5 / C_WATER, targets=tg, n_speckle=128, seed=seed)


_BUILDERS = {1: _cfg1, 2: _cfg2, 3: _cfg3, 4: _cfg4, 5: _cfg5}


def scenario(cid: int, reduced: bool = False, seed: Optional[int] = None) -> Scenario:
    """Config ``cid`` (1..5) of BASELINE.json; seed defaults to 1000 + cid."""
    b = _BUILDERS[cid]
    return b(reduced=reduced) if seed is None else b(reduced=reduced, seed=seed)


def random_case(seed: int, P=3, E=2, Ns=256, n=(9, 7, 3), fc=40e3, fs=50e3, c=C_WATER, offset=(0.0, 0.0, 0.0)):
    """Tiny random geometry + white complex echoes (brute-force / invariant tests).
    The grid is placed so the pixel delays fall inside the recorded window."""
    rng = np.random.default_rng(seed)
    off = np.asarray(offset, dtype=np.float64)
    grid = grid_dict(off + np.array([1.0, 2.0, 0.5]), (0.013, 0.011, 0.017), n)
    tx = off + np.stack([rng.uniform(0, 0.5, P), rng.uniform(-0.3, 0.3, P), rng.uniform(-1.2, -0.8, P)], axis=1)
    rx = tx[:, None, :] + rng.uniform(-0.2, 0.2, size=(P, E, 3))
    # window covering the two-way delays
    t0 = np.full(P, 2.0 * 1.5 / c) + rng.uniform(0, 1e-4, P)
    ech = ((rng.normal(size=(P, E, Ns)) + 1j * rng.normal(size=(P, E, Ns))) / np.sqrt(2)).astype(np.complex64)
    return dict(echoes=ech, tx=tx, rx=rx, t0=t0, fc=fc, fs=fs, c=c, grid=grid)


def nav_table(s: "Scenario", K: int = 8, accel: float = 0.5, yaw_rate_deg: float = 2.0, vel=None, seed: int = 0):
    """Seeded tabled receiver trajectories for the scenario's pings (input for NEXT-2 reading R23,
    the paper's position look-up table): K nodes dt apart from each transmit covering the
    record (dt = (max t0 + Ns/fs) / (K - 1)); receiver (p, e) starts at rx[p, e] and moves as
        r(t) = rx + v_p t + a_p t^2 / 2 + (Rz(w_p t) - I)(rx - tx_p)
    (platform velocity v_p -- the scenario's vel, else the given / a seeded one --, a seeded
    acceleration a_p, and the lever arm turning at a seeded yaw rate w_p).  Returns (lut [P][E][K][3], dt)."""
    rng = np.random.default_rng(seed)
    P, E = s.P, s.E
    T = float(np.max(s.t0)) + s.Ns / s.fs
    dt = T / (K - 1)
    if vel is None:
        vel = s.vel if s.vel is not None else rng.normal(size=(P, 3)) * np.array([1.0, 0.3, 0.1])
    vel = np.asarray(vel, dtype=np.float64).reshape(P, 3)
    acc = rng.normal(size=(P, 3)) * accel
    w = np.deg2rad(yaw_rate_deg) * rng.normal(size=P)
    t = np.arange(K) * dt
    lever = s.rx - s.tx[:, None, :]                                  # [P][E][3]
    ang = w[:, None] * t[None, :]                                     # [P][K]
    cs, sn = np.cos(ang) - 1.0, np.sin(ang)
    dlx = cs[:, None, :] * lever[:, :, None, 0] - sn[:, None, :] * lever[:, :, None, 1]
    dly = sn[:, None, :] * lever[:, :, None, 0] + cs[:, None, :] * lever[:, :, None, 1]
    lut = (s.rx[:, :, None, :] + vel[:, None, None, :] * t[None, None, :, None]
           + 0.5 * acc[:, None, None, :] * (t * t)[None, None, :, None])
    lut[..., 0] += dlx
    lut[..., 1] += dly
    return np.ascontiguousarray(lut), dt
