"""Randomised GPU-vs-oracle parity (-m gpu): 48 seeded random small problems stressing the plan
logic -- rotated (non axis-aligned) grids, 2D and 3D, sensors far away or inside / next to the
grid (near-field exact legs), delays inside, straddling and outside the record, fc/fs ratios from
0.3 to 3, ragged tile edges -- through the dense, weighted and moving-receiver paths."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
TOL = 1e-3


@pytest.fixture(scope="module")
def pk(require_gpu):
    import torch
    torch.cuda.set_device(0)
    from paper_2101_05888_b200 import _build
    _build.build()
    import paper_2101_05888_b200 as pkg
    return pkg


def _rot(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    a, b, c, d = q
    return np.array([[a * a + b * b - c * c - d * d, 2 * (b * c - a * d), 2 * (b * d + a * c)],
                     [2 * (b * c + a * d), a * a - b * b + c * c - d * d, 2 * (c * d - a * b)],
                     [2 * (b * d - a * c), 2 * (c * d + a * b), a * a - b * b - c * c + d * d]])


def _case(seed):
    rng = np.random.default_rng(5000 + seed)
    c = 1500.0
    fs = float(rng.choice([20e3, 50e3, 120e3]))
    fc = fs * float(rng.uniform(0.3, 3.0))
    nz = 1 if seed % 2 == 0 else int(rng.integers(2, 6))
    n = (int(rng.integers(1, 41)), int(rng.integers(1, 41)), nz)
    R = _rot(rng) if seed % 3 else np.eye(3)
    st = rng.uniform(0.004, 0.02, size=3)
    origin = rng.uniform(-1, 1, size=3) * 5
    grid = {"origin": origin, "step_x": R[:, 0] * st[0], "step_y": R[:, 1] * st[1],
            "step_z": R[:, 2] * st[2] if nz > 1 else np.array([0.0, 0.0, 1.0]), "nx": n[0], "ny": n[1], "nz": nz}
    P, E = int(rng.integers(1, 8)), int(rng.integers(1, 5))
    centre = origin + 0.5 * (n[0] * grid["step_x"] + n[1] * grid["step_y"] + (nz - 1) * grid["step_z"])
    near = seed % 4 == 1   # sensors inside / next to the grid
    spread = 0.3 if near else 1.0
    off = np.zeros(3) if near else rng.normal(size=3) * 3
    tx = centre + off + rng.normal(size=(P, 3)) * spread
    rx = tx[:, None, :] + rng.normal(size=(P, E, 3)) * 0.1
    Ns = int(rng.integers(50, 700))
    d = np.linalg.norm(centre[None] - tx, axis=1)
    tau = 2 * d / c
    shift = rng.uniform(-0.6, 0.6) * Ns / fs if seed % 5 == 2 else 0.0   # straddle / miss the record
    t0 = tau - 0.5 * Ns / fs + shift
    ech = ((rng.normal(size=(P, E, Ns)) + 1j * rng.normal(size=(P, E, Ns))) / np.sqrt(2)).astype(np.complex64)
    vel = rng.normal(size=(P, 3)) * 2.0
    return grid, tx, rx, t0, ech, fc, fs, c, vel


def _idx(g):
    iz, iy, ix = np.meshgrid(np.arange(g["nz"]), np.arange(g["ny"]), np.arange(g["nx"]), indexing="ij")
    return np.stack([ix.ravel(), iy.ravel(), iz.ravel()], axis=1)


def _cmp(got, ref, label):
    got = np.asarray(got).ravel()
    assert np.all(np.isfinite(got)), label
    scale = np.max(np.abs(ref))
    if scale == 0:
        assert np.max(np.abs(got)) == 0, label
        return
    assert np.max(np.abs(got - ref)) <= TOL * scale, (label, np.max(np.abs(got - ref)) / scale)


@pytest.mark.parametrize("seed", range(48))
def test_random_problem(pk, seed):
    grid, tx, rx, t0, ech, fc, fs, c, vel = _case(seed)
    idx = _idx(grid)
    pts = oracle.grid_points(grid, idx)
    mode = ("dense", "weighted", "motion")[seed % 3]
    with pk.Backprojector(fc, fs / 4, fs, c, grid) as bp:
        if mode == "weighted":
            bp.set_weighting(True)
        if mode == "motion":
            bp.set_motion(vel)
        bp.set_pings(ech, tx, rx, t0)
        got = bp.form()
        _, inwin = bp.count_terms()
    if mode == "dense":
        ref, cnt = oracle.tdbp_points(ech, tx, rx, t0, fc, fs, c, pts, with_count=True)
        assert inwin == int(cnt.sum()), (seed, inwin, int(cnt.sum()))
    elif mode == "weighted":
        ref = oracle.tdbp_points_weighted(ech, tx, rx, t0, fc, fs, c, pts)
    else:
        ref = oracle.tdbp_points_motion(ech, tx, rx, t0, vel, fc, fs, c, pts)
    _cmp(got, ref, f"seed {seed} {mode} grid {grid['nx']}x{grid['ny']}x{grid['nz']} P{len(tx)}")
