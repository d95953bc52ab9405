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
        ref, cnt = oracle.tdbp_points_motion(ech, tx, rx, t0, vel, fc, fs, c, pts, with_count=True)
        # fp32 delays decide terms exactly at u = -1 or Ns differently from fp64 only on ties
        assert abs(inwin - int(cnt.sum())) <= max(2, int(1e-4 * cnt.sum())), (seed, inwin, int(cnt.sum()))
    _cmp(got, ref, f"seed {seed} {mode} grid {grid['nx']}x{grid['ny']}x{grid['nz']} P{len(tx)}")


@pytest.mark.parametrize("seed", range(0, 48, 3))
def test_random_problem_cp_async(pk, seed, monkeypatch):
    """The same random dense problems through the cp.async staging path (SASBP_NO_TMA=1)."""
    monkeypatch.setenv("SASBP_NO_TMA", "1")
    grid, tx, rx, t0, ech, fc, fs, c, _ = _case(seed)
    pts = oracle.grid_points(grid, _idx(grid))
    with pk.Backprojector(fc, fs / 4, fs, c, grid) as bp:
        bp.set_pings(ech, tx, rx, t0)
        assert bp.plan()["tma"] is False
        got = bp.form()
    ref = oracle.tdbp_points(ech, tx, rx, t0, fc, fs, c, pts)
    _cmp(got, ref, f"cp.async seed {seed}")


def _axes(rng, P):
    a = rng.normal(size=(P, 3))
    a /= np.linalg.norm(a, axis=1, keepdims=True)
    b = rng.normal(size=(P, 3))
    b -= (b * a).sum(1, keepdims=True) * a
    b /= np.linalg.norm(b, axis=1, keepdims=True)
    return np.stack([a, b], axis=1)


@pytest.mark.parametrize("seed", range(24))
def test_random_gated(pk, seed):
    """Random beams: azimuth 0.1-1.5 rad, optional elevation, bistatic or not, per-ping axes or the
    default, culling on or off; the gate decisions are fp64 on both sides (R15)."""
    grid, tx, rx, t0, ech, fc, fs, c, _ = _case(100 + seed)
    rng = np.random.default_rng(7000 + seed)
    P = len(tx)
    az = float(rng.uniform(0.1, 1.5))
    el = float(rng.uniform(0.2, 2.0)) if seed % 3 == 0 else 0.0
    bistatic = bool(seed % 2)
    axes = _axes(rng, P) if seed % 4 < 2 else None
    cull = seed % 5 != 0
    idx = _idx(grid)
    pts = oracle.grid_points(grid, idx)
    with pk.Backprojector(fc, fs / 4, fs, c, grid) as bp:
        bp.set_pings(ech, tx, rx, t0)
        bp.set_beam(az, el, bistatic, cull, axes)
        got = bp.form()
        _, inc = bp.count_terms()
    ref, cnt = oracle.tdbp_points_gated(ech, tx, rx, t0, fc, fs, c, pts, az, el, bistatic, axes, with_count=True)
    assert inc == int(cnt.sum()), (seed, inc, int(cnt.sum()))
    _cmp(got, ref, f"gated seed {seed}")


@pytest.mark.parametrize("seed", range(12))
def test_random_refracted(pk, seed):
    """Random flat interfaces through or below the volume, sediment faster or slower than water."""
    grid, tx, rx, t0, ech, fc, fs, c, _ = _case(200 + 2 * seed + 1)   # odd -> 3D grids
    rng = np.random.default_rng(8000 + seed)
    zs = max(tx[:, 2].max(), rx[:, :, 2].max())
    pts_all = oracle.grid_points(grid, _idx(grid))
    zb = float(zs + rng.uniform(0.01, 1.0) * max(1e-3, pts_all[:, 2].max() - zs)) if pts_all[:, 2].max() > zs \
        else float(zs + 0.05)
    c2 = float(rng.choice([1450.0, 1600.0, 1750.0]))
    with pk.Backprojector(fc, fs / 4, fs, c, grid) as bp:
        bp.set_pings(ech, tx, rx, t0)
        try:
            bp.set_medium(zb, c2)
        except pk.SasError:
            pytest.skip("window for this sediment speed exceeds shared memory")
        got = bp.form()
    ref = oracle.tdbp_points_refracted(ech, tx, rx, t0, zb, c2, fc, fs, c, pts_all)
    _cmp(got, ref, f"refracted seed {seed}")


@pytest.mark.parametrize("seed", range(12))
def test_random_conditioning(pk, seed):
    """Random sizes for K1 (both paths), K1b, K0 and the whitening pair."""
    rng = np.random.default_rng(9000 + seed)
    nch, Ns = int(rng.integers(1, 7)), int(rng.integers(1, 5000))
    x = ((rng.normal(size=(nch, Ns)) + 1j * rng.normal(size=(nch, Ns))) / np.sqrt(2)).astype(np.complex64)
    Nr = int(rng.integers(1, 2100))
    rep = ((rng.normal(size=Nr) + 1j * rng.normal(size=Nr)) / np.sqrt(2 * Nr)).astype(np.complex64)
    r = oracle.rangecompress(x, rep)
    assert np.max(np.abs(pk.rangecompress(x, rep) - r)) <= 2e-5 * max(np.max(np.abs(r)), 1e-30)
    U = int(rng.integers(1, 17))
    u = oracle.upsample(x, U)
    assert np.max(np.abs(pk.upsample(x, U) - u)) <= 2e-5 * np.max(np.abs(u))
    D = int(rng.integers(1, 40))
    Nh = int(rng.integers(0, 200)) * 2 + 1
    h = rng.normal(size=Nh).astype(np.float32)
    xr = rng.normal(size=(1, nch, max(Ns, 1))).astype(np.float32)
    Nout = int(rng.integers(1, max(2, Ns // D + 3)))
    t0 = np.array([float(rng.uniform(0, 0.05))])
    fcb = float(rng.uniform(1e3, 200e3))
    b = oracle.baseband(xr, 480e3, fcb, t0, h, D, Nout)
    bg = pk.baseband(xr, 480e3, fcb, t0, h, D, Nout)
    assert np.max(np.abs(bg - b)) <= 2e-5 * max(np.max(np.abs(b)), 1e-30) or np.max(np.abs(b)) == 0
    M = int(rng.choice([1, 2, 16, 32, 48, 64, 128, 256]))
    if np.max(np.abs(x)) > 0:
        G, _ = oracle.whitening_gain(x, M, 0.05)
        Gg = pk.whitening_gain(x, M, 0.05)
        assert np.max(np.abs(Gg - G)) <= 2e-5
        if Nr + M - 1 <= 8192 and nch * Ns * Nr * M <= 3e8:   # the oracle cascade is O(Ns Nr M)
            w = oracle.rangecompress_whitened(x, rep, G.astype(np.float32).astype(np.float64))
            wg = pk.rangecompress_whitened(x, rep, G.astype(np.float32))
            assert np.max(np.abs(wg - w)) <= 2e-5 * max(np.max(np.abs(w)), 1e-30)


@pytest.mark.parametrize("seed", range(8))
def test_random_partition_accumulate_streamed(pk, seed):
    """Ping-partition additivity through SAS_FORM_ACCUMULATE on borrowed (device) echoes, an
    8-byte-but-not-16-byte aligned device pointer (cp.async staging), and form_streamed with a
    random chunk count -- all against the single dense form."""
    import torch
    grid, tx, rx, t0, ech, fc, fs, c, _ = _case(300 + seed)
    P = len(tx)
    rng = np.random.default_rng(9500 + seed)
    with pk.Backprojector(fc, fs / 4, fs, c, grid) as bp:
        bp.set_pings(ech, tx, rx, t0)
        ref = bp.form()
        # partition the pings, accumulate on the device
        cut = int(rng.integers(0, P + 1))
        img = torch.zeros(bp.shape, dtype=torch.complex64, device="cuda")
        first = True
        for sl in (slice(0, cut), slice(cut, P)):
            if sl.stop - sl.start == 0:
                continue
            e_d = torch.from_numpy(np.ascontiguousarray(ech[sl])).cuda()
            bp.set_pings_device(e_d, tx[sl], rx[sl], t0[sl])
            bp.form_device(img, accumulate=not first)
            first = False
        torch.cuda.synchronize()
        part = img.cpu().numpy()
        # misaligned (8-byte) borrowed pointer -> cp.async staging
        buf = torch.empty(ech.size + 1, dtype=torch.complex64, device="cuda")
        view = buf[1:].view(ech.shape)
        view.copy_(torch.from_numpy(ech))
        bp.set_pings_device(view, tx, rx, t0)
        mis = torch.empty(bp.shape, dtype=torch.complex64, device="cuda")
        bp.form_device(mis)
        torch.cuda.synchronize()
        tma_mis = bp.plan()["tma"]
        st = bp.form_streamed(ech, tx, rx, t0, chunks=int(rng.integers(0, 5)))
    assert tma_mis is False
    scale = np.max(np.abs(ref))
    if scale == 0:
        return
    assert np.max(np.abs(part - ref)) <= 1e-5 * scale
    assert np.max(np.abs(mis.cpu().numpy() - ref)) <= 1e-6 * scale
    assert np.max(np.abs(st - ref)) <= 1e-5 * scale


@pytest.mark.parametrize("seed", range(8))
def test_random_gated_weighted(pk, seed):
    grid, tx, rx, t0, ech, fc, fs, c, _ = _case(400 + seed)
    rng = np.random.default_rng(9700 + seed)
    az = float(rng.uniform(0.2, 1.5))
    bistatic = bool(seed % 2)
    pts = oracle.grid_points(grid, _idx(grid))
    with pk.Backprojector(fc, fs / 4, fs, c, grid) as bp:
        bp.set_pings(ech, tx, rx, t0)
        bp.set_weighting(True)
        bp.set_beam(az, 0.0, bistatic, True)
        got = bp.form()
    ref = oracle.tdbp_points_gated_weighted(ech, tx, rx, t0, fc, fs, c, pts, az=az, bistatic=bistatic)
    _cmp(got, ref, f"gated weighted seed {seed}")


def _case_many(seed):
    """Stripmap-like problems with many channels (multi-batch pipelines: prologue groups, the
    constant ring, mbarrier phases, culled batches) on small grids."""
    rng = np.random.default_rng(11000 + seed)
    c, fs = 1500.0, float(rng.choice([40e3, 120e3]))
    fc = fs * float(rng.uniform(0.5, 2.0))
    P, E = int(rng.integers(20, 90)), int(rng.integers(1, 9))
    nx, ny = int(rng.integers(8, 70)), int(rng.integers(8, 70))
    step = float(rng.uniform(0.005, 0.02))
    y0 = float(rng.uniform(5, 20))
    grid = {"origin": np.array([0.0, y0, 0.0]), "step_x": np.array([step, 0, 0]), "step_y": np.array([0, step, 0]),
            "step_z": np.array([0, 0, 1.0]), "nx": nx, "ny": ny, "nz": 1}
    xs = np.linspace(-3, 3 + nx * step, P)
    tx = np.stack([xs, np.zeros(P), np.full(P, -5.0)], axis=1) + rng.normal(size=(P, 3)) * 0.02
    rx = tx[:, None, :] + np.stack([(np.arange(E) - (E - 1) / 2) * 0.03, np.zeros(E), np.zeros(E)], axis=1)[None]
    ctr = np.array([nx * step / 2, y0 + ny * step / 2, 0.0])
    d = np.linalg.norm(ctr[None] - tx, axis=1)
    Ns = int(rng.integers(300, 1500))
    t0 = 2 * d / c - 0.5 * Ns / fs + rng.uniform(-0.2, 0.2) * Ns / fs
    ech = ((rng.normal(size=(P, E, Ns)) + 1j * rng.normal(size=(P, E, Ns))) / np.sqrt(2)).astype(np.complex64)
    return grid, tx, rx, t0, ech, fc, fs, c


@pytest.mark.parametrize("seed", range(10))
def test_random_many_channels(pk, seed):
    grid, tx, rx, t0, ech, fc, fs, c = _case_many(seed)
    pts = oracle.grid_points(grid, _idx(grid))
    gated = seed % 2 == 1
    az = 0.3 + 0.05 * seed
    with pk.Backprojector(fc, fs / 4, fs, c, grid) as bp:
        bp.set_pings(ech, tx, rx, t0)
        if gated:
            bp.set_beam(az, 0.0, seed % 4 == 3, True)
        got = bp.form()
    if gated:
        ref = oracle.tdbp_points_gated(ech, tx, rx, t0, fc, fs, c, pts, az, 0.0, seed % 4 == 3)
    else:
        ref = oracle.tdbp_points(ech, tx, rx, t0, fc, fs, c, pts)
    _cmp(got, ref, f"many channels seed {seed} P{len(tx)} E{rx.shape[1]} gated={gated}")
