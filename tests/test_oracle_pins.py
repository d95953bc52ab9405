"""Pins of the fp64 oracle against what the paper and mathematics fix (not against itself).

Each test names the passage / reading it follows (SURVEY §8(c) pins):
closed forms and hand-derived values (tests/golden/closed_form.json), zero-extension
values, point-target physics of config 1 (tests/golden/cfg1_physics.json), invariants
(linearity, ping order, ping partition, translation, axis permutation), and the
range-compression pins (autocorrelation peak, shift, mainlobe).
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _ramp(Ns, a=(1.0, 2.0), b=(2.0 ** -10, -(2.0 ** -11))):
    n = np.arange(Ns, dtype=np.float64)
    d = (a[0] + b[0] * n) + 1j * (a[1] + b[1] * n)
    d32 = d.astype(np.complex64)
    assert np.array_equal(d32.astype(np.complex128), d)  # exactly representable
    return d32


@pytest.mark.parametrize("case", _load("closed_form.json")["cases"], ids=lambda c: c["name"])
def test_closed_form_single_term(case):
    """P = E = 1: I(x) = ehat(u) exp(+j 2 pi fc tau) with u, tau hand-derived (Eq. 1 delay P:89; R1-R4)."""
    g = _load("closed_form.json")
    Ns = g["ramp"]["Ns"]
    d = _ramp(Ns)
    ech = d.reshape(1, 1, Ns)
    val, cnt = oracle.tdbp_points(ech, np.array([case["tx"]]), np.array([[case["rx"]]]),
                                  np.array([case["t0"]]), case["fc"], case["fs"], case["c"],
                                  np.array([case["x"]]), with_count=True)
    u, cyc = case["u"], case["cycles"]
    ehat = (1.0 + u / 1024.0) + 1j * (2.0 - u / 2048.0)  # ramp is exact under linear interpolation
    expected = ehat * np.exp(2j * np.pi * (cyc - np.floor(cyc)))
    assert abs(val[0] - expected) <= 1e-9 * abs(expected)
    assert cnt[0] == 1


def test_bistatic_sign_is_plus_j():
    """The 3-4-5 case has fc*tau = 600.25 cycles: the ramp exp(+j..) gives +j * ehat; the opposite
    sign convention would give -j * ehat (R3)."""
    case = [c for c in _load("closed_form.json")["cases"] if c["name"] == "bistatic_345_sign"][0]
    d = _ramp(4096).reshape(1, 1, 4096)
    val = oracle.tdbp_points(d, np.array([case["tx"]]), np.array([[case["rx"]]]), None, case["fc"],
                             case["fs"], case["c"], np.array([case["x"]]))[0]
    ehat = (1.0 + 720 / 1024.0) + 1j * (2.0 - 720 / 2048.0)
    assert abs(val - 1j * ehat) < 1e-9
    assert abs(val + 1j * ehat) > 1.0


def test_zero_extension_values_and_counts():
    """R2: d[n] = 0 outside 0..Ns-1, so ehat is continuous in u; N_u counts u in (-1, Ns)."""
    z = _load("closed_form.json")["zero_extension"]
    Ns = z["Ns"]
    ech = np.ones((1, 1, Ns), dtype=np.complex64)
    for case in z["cases"]:
        val, cnt = oracle.tdbp_points(ech, np.zeros((1, 3)), np.zeros((1, 1, 3)), np.array([case["t0"]]),
                                      z["fc"], z["fs"], z["c"], np.array([[z["R"], 0.0, 0.0]]),
                                      with_count=True)
        assert abs(val[0] - case["value"]) < 1e-9, case
        assert cnt[0] == case["in_window"], case


def test_lerp_exact_at_integer_and_on_ramps():
    """R1: at integer u the interpolant returns d[k]; on linear data it is exact for any u."""
    Ns = 64
    rng = np.random.default_rng(3)
    d = (rng.normal(size=Ns) + 1j * rng.normal(size=Ns)).astype(np.complex64)
    c, fs, fc = 1500.0, 1000.0, 1000.0  # R = 15 -> tau = 0.02 s, fc tau = 20 cycles (phase 1)
    for k in [0, 1, 17, 63]:
        t0 = 0.02 - k / fs
        val = oracle.tdbp_points(d.reshape(1, 1, Ns), np.zeros((1, 3)), np.zeros((1, 1, 3)),
                                 np.array([t0]), fc, fs, c, np.array([[15.0, 0, 0]]))[0]
        assert abs(val - complex(d[k])) < 1e-9


def _numpy_bruteforce(echoes, tx, rx, t0, fc, fs, c, pts):
    """Independent cross-check (a second, vectorised implementation -- not a pin by itself)."""
    P, E, Ns = echoes.shape
    d = np.concatenate([echoes.astype(np.complex128), np.zeros((P, E, 2))], axis=2)
    out = np.zeros(len(pts), dtype=np.complex128)
    for i, x in enumerate(pts):
        rt = np.linalg.norm(x[None] - tx, axis=1)[:, None]
        rr = np.linalg.norm(x[None, None] - rx, axis=2)
        tau = (rt + rr) / c
        u = (tau - t0[:, None]) * fs
        k = np.floor(u).astype(np.int64)
        a = u - k
        def at(n):
            ok = (n >= 0) & (n < Ns)
            nn = np.where(ok, n, Ns)
            return np.take_along_axis(d, nn[..., None], axis=2)[..., 0] * ok
        eh = (1 - a) * at(k) + a * at(k + 1)
        out[i] = np.sum(eh * np.exp(2j * np.pi * fc * tau))
    return out


def test_cross_check_numpy_bruteforce():
    r = synth.random_case(11)
    g = r["grid"]
    img = oracle.tdbp_grid(r["echoes"], r["tx"], r["rx"], r["t0"], r["fc"], r["fs"], r["c"], g)
    iz, iy, ix = np.meshgrid(np.arange(g["nz"]), np.arange(g["ny"]), np.arange(g["nx"]), indexing="ij")
    pts = (g["origin"][None] + ix.ravel()[:, None] * g["step_x"] + iy.ravel()[:, None] * g["step_y"]
           + iz.ravel()[:, None] * g["step_z"])
    ref = _numpy_bruteforce(r["echoes"], r["tx"], r["rx"], r["t0"], r["fc"], r["fs"], r["c"], pts)
    assert np.max(np.abs(img.ravel() - ref)) <= 1e-12 * np.max(np.abs(ref)) * 10


# ---------------------------------------------------------------- invariants

def _img(r, echoes=None, tx=None, rx=None, t0=None, grid=None):
    return oracle.tdbp_grid(r["echoes"] if echoes is None else echoes, r["tx"] if tx is None else tx,
                            r["rx"] if rx is None else rx, r["t0"] if t0 is None else t0, r["fc"],
                            r["fs"], r["c"], r["grid"] if grid is None else grid)


def test_linearity():
    """reconstruct(a e1 + e2) = a reconstruct(e1) + reconstruct(e2)."""
    r1, r2 = synth.random_case(5), synth.random_case(6)
    a = np.float32(0.75)
    e12 = (a * r1["echoes"] + r2["echoes"]).astype(np.complex64)
    lhs = _img(r1, echoes=e12)
    rhs = a * _img(r1) + _img(r1, echoes=r2["echoes"])
    assert np.max(np.abs(lhs - rhs)) <= 1e-6 * np.max(np.abs(lhs))  # complex64 rounding of e12


def test_ping_order_invariance():
    """the sum over pings is order-free."""
    r = synth.random_case(7, P=5)
    perm = np.array([3, 0, 4, 1, 2])
    a = _img(r)
    b = _img(r, echoes=r["echoes"][perm], tx=r["tx"][perm], rx=r["rx"][perm], t0=r["t0"][perm])
    assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(a))


def test_ping_partition_additivity():
    """I(A u B) = I(A) + I(B) (the multi-GPU ping-shard identity)."""
    r = synth.random_case(8, P=6)
    A, B = np.array([0, 2, 5]), np.array([1, 3, 4])
    full = _img(r)
    part = lambda s: _img(r, echoes=r["echoes"][s], tx=r["tx"][s], rx=r["rx"][s], t0=r["t0"][s])
    assert np.max(np.abs(full - (part(A) + part(B)))) <= 1e-12 * np.max(np.abs(full))


def test_translation_invariance():
    """Shifting every position and the grid origin by (1e4, -3e3, 0) m leaves I unchanged."""
    off = np.array([1e4, -3e3, 0.0])
    r = synth.random_case(9)
    g2 = dict(r["grid"])
    g2["origin"] = r["grid"]["origin"] + off
    a = _img(r)
    b = _img(r, tx=r["tx"] + off, rx=r["rx"] + off[None, None], grid=g2)
    assert np.max(np.abs(a - b)) <= 1e-7 * np.max(np.abs(a))


def test_axis_permutation():
    """Cyclically permuting (x, y, z) for every position and grid vector gives the same image:
    the delay uses all three coordinates symmetrically (catches an index typo)."""
    r = synth.random_case(10)
    perm = [1, 2, 0]
    g = r["grid"]
    g2 = dict(g)
    for k in ("origin", "step_x", "step_y", "step_z"):
        g2[k] = np.asarray(g[k])[perm]
    a = _img(r)
    b = _img(r, tx=r["tx"][:, perm], rx=r["rx"][:, :, perm], grid=g2)
    assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(a))


def test_element_reciprocity():
    """Swapping the roles of tx and rx (monostatic-pair reciprocity of the delay)."""
    r = synth.random_case(12, E=1)
    a = _img(r)
    b = _img(r, tx=r["rx"][:, 0, :], rx=r["tx"][:, None, :])
    assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(a))


# ---------------------------------------------------------------- physics (config 1)

def _minus3db_width(xs, mag):
    """-3 dB (half-power) width of the main lobe of |I| sampled on a fine line."""
    i0 = int(np.argmax(mag))
    thr = mag[i0] / np.sqrt(2.0)
    i = i0
    while mag[i] > thr:
        i -= 1
    left = xs[i] + (thr - mag[i]) * (xs[i + 1] - xs[i]) / (mag[i + 1] - mag[i])
    j = i0
    while mag[j] > thr:
        j += 1
    right = xs[j - 1] + (thr - mag[j - 1]) * (xs[j] - xs[j - 1]) / (mag[j] - mag[j - 1])
    return right - left


@pytest.fixture(scope="module")
def cfg1():
    s = synth.scenario(1)
    return s, s.echoes()


def test_cfg1_point_target_focus(cfg1):
    """Config 1: peak at the true pixel, phase ~ 0 (R3), magnitude within the
    in-beam bound (Eq. 1 amplitudes) -- tests/golden/cfg1_physics.json."""
    s, e = cfg1
    gold = _load("cfg1_physics.json")
    img = oracle.tdbp_grid(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, s.grid)[0]
    mag = np.abs(img)
    iy, ix = np.unravel_index(np.argmax(mag), mag.shape)
    tp = gold["target_pixel"]
    assert abs(ix - tp[0]) <= gold["peak_position_tol_px"] and abs(iy - tp[1]) <= gold["peak_position_tol_px"]
    assert abs(np.angle(img[iy, ix])) <= gold["peak_phase_tol_rad"]
    x = s.targets[0]
    rt = np.linalg.norm(x[None] - s.tx, axis=1)
    rr = np.linalg.norm(x[None, None] - s.rx, axis=2)
    inbeam = np.abs((x[None] - s.tx)[:, 0]) <= rt * s.sin_half_beam
    bound = np.sum((1.0 / (rt[:, None] * rr))[inbeam])
    ratio = mag[iy, ix] / bound
    assert gold["peak_over_bound_min"] <= ratio <= 1.0, ratio


def test_cfg1_resolution_widths(cfg1):
    """-3 dB widths on fine lines through the target formed directly by TDBP (no image
    interpolation): along-track ~ D/2, ground range ~ 0.886 c/(2B) * R/y (north star)."""
    s, e = cfg1
    gold = _load("cfg1_physics.json")
    x0 = s.targets[0]
    offs = np.arange(-0.06, 0.06 + 1e-12, 0.0002)
    line_x = x0[None] + offs[:, None] * np.array([1.0, 0, 0])[None]
    line_y = x0[None] + offs[:, None] * np.array([0, 1.0, 0])[None]
    ax = np.abs(oracle.tdbp_points(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, line_x))
    ay = np.abs(oracle.tdbp_points(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, line_y))
    wx, wy = _minus3db_width(offs, ax), _minus3db_width(offs, ay)
    assert abs(wx / gold["along_track_width_m"] - 1) <= gold["along_track_rel_tol"], wx
    assert abs(wy / gold["ground_range_width_m"] - 1) <= gold["ground_range_rel_tol"], wy


def test_two_targets_resolved():
    """two scatterers 4x the along-track resolution apart give two peaks, each at its
    true position, with a > 3 dB dip between them."""
    base = synth.scenario(1)
    tg = np.array([[2.52, 11.18, 0.0], [2.60, 11.18, 0.0]])  # 8 cm = 4 x 2 cm apart
    s = synth.stripmap("two", P=base.P, E=base.E, **synth.HF, altitude=10.0,
                       track=(base.tx[0, 0], base.tx[-1, 0]), grid=base.grid, Ns=base.Ns, t0=0.012,
                       targets=tg, n_speckle=0)
    e = s.echoes()
    offs = np.arange(-0.08, 0.08 + 1e-12, 0.0005)
    line = np.array([2.56, 11.18, 0.0])[None] + offs[:, None] * np.array([1.0, 0, 0])[None]
    a = np.abs(oracle.tdbp_points(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, line))
    left, right = a[offs < 0], a[offs > 0]
    pl, pr = offs[offs < 0][np.argmax(left)], offs[offs > 0][np.argmax(right)]
    assert abs(pl - (-0.04)) <= 0.0025 and abs(pr - 0.04) <= 0.0025  # half a 5 mm... pixel
    mid = a[np.argmin(np.abs(offs))]
    assert mid < min(left.max(), right.max()) / np.sqrt(2)


# ---------------------------------------------------------------- range compression (row a1)

def _lfm(fs, B, T):
    n = int(round(T * fs))
    t = np.arange(n) / fs - T / 2
    return np.exp(1j * np.pi * (B / T) * t ** 2).astype(np.complex64)


def test_rangecompress_autocorrelation_peak():
    """replica through its own matched filter peaks at lag 0 with value = energy."""
    r = _lfm(120e3, 30e3, 2e-3)
    x = np.zeros(1024, dtype=np.complex64)
    x[:r.size] = r
    y = oracle.rangecompress(x[None], r)[0]
    energy = np.sum(np.abs(r.astype(np.complex128)) ** 2)
    assert np.argmax(np.abs(y)) == 0
    assert abs(y[0] - energy) <= 1e-9 * energy


def test_rangecompress_shift_and_mainlobe():
    """delay by k -> peak at lag k; -3 dB mainlobe ~ 1/B within 20 %."""
    fs, B = 120e3, 30e3
    r = _lfm(fs, B, 2e-3)
    k = 300
    x = np.zeros(2048, dtype=np.complex64)
    x[k:k + r.size] = r
    y = np.abs(oracle.rangecompress(x[None], r)[0])
    assert np.argmax(y) == k
    # fine mainlobe via a sub-sample delayed analytic copy is overkill; sample-level width:
    # interpolate the half-power crossing on the sampled |y|
    w = _minus3db_width(np.arange(y.size) / fs, y)
    assert abs(w * B - 1.0) <= 0.2, w * B


def test_rangecompress_definition_small():
    """Brute force on a tiny case: y[n] = sum_m x[n+m] conj(r[m]) with x zero past the end."""
    rng = np.random.default_rng(4)
    x = (rng.normal(size=(2, 9)) + 1j * rng.normal(size=(2, 9))).astype(np.complex64)
    r = (rng.normal(size=4) + 1j * rng.normal(size=4)).astype(np.complex64)
    y = oracle.rangecompress(x, r)
    for ch in range(2):
        for n in range(9):
            ref = sum(complex(x[ch, n + m]) * np.conj(complex(r[m])) for m in range(4) if n + m < 9)
            assert abs(y[ch, n] - ref) < 1e-9


# ---------------------------------------------------------------- generator (Eq. 2) pins

def test_rotation_eq2_examples():
    """S:124-126 + the sign conventions printed under Eq. 2."""
    assert np.allclose(synth.rotation_matrix(0, 0, 0) @ [1, 2, 3], [1, 2, 3])
    assert np.allclose(synth.rotation_matrix(0, 0, np.pi / 2) @ [1, 0, 0], [0, 1, 0], atol=1e-12)
    rng = np.random.default_rng(0)
    for _ in range(100):
        R = synth.rotation_matrix(*rng.uniform(-np.pi, np.pi, 3))
        assert np.allclose(R.T @ R, np.eye(3), atol=1e-12)
        assert abs(np.linalg.det(R) - 1) < 1e-12
    # positive roll lowers the starboard side (+y body -> +z down)
    assert (synth.rotation_matrix(0.1, 0, 0) @ [0, 1, 0])[2] > 0
    # positive pitch raises the bow (+x body -> -z, up)
    assert (synth.rotation_matrix(0, 0.1, 0) @ [1, 0, 0])[2] < 0


def test_nominal_nav_defocuses_high_motion():
    """S:798 analog: imaging the high-motion collection (config 3, reduced) with the nominal,
    unperturbed navigation instead of the true one loses at least 3 dB of target peak --
    the method needs the per-ping, per-element positions (R5), not a straight-line track."""
    s = synth.scenario(3, reduced=True)
    e = s.echoes()
    idx = s.sample_pixels(0, window=9)
    true_img = oracle.tdbp_grid(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, s.grid, idx=idx)
    ntx, nrx = s.nav_nominal
    nom_img = oracle.tdbp_grid(e, ntx, nrx, s.t0, s.fc, s.fs, s.c, s.grid, idx=idx)
    loss_db = 20 * np.log10(np.max(np.abs(true_img)) / np.max(np.abs(nom_img)))
    assert loss_db >= 3.0, loss_db


# ---------------------------------------------------------------- gated TDBP (NEXT-1, reading R15)

def test_gate_wide_open_equals_dense():
    """With the azimuth test disabled (az >= pi) and no elevation test the gate admits every
    term: the gated sum reduces to the pinned dense definition."""
    r = synth.random_case(21)
    pts = oracle.grid_points(r["grid"])
    dense = oracle.tdbp_points(r["echoes"], r["tx"], r["rx"], r["t0"], r["fc"], r["fs"], r["c"], pts)
    for bist in (False, True):
        g = oracle.tdbp_points_gated(r["echoes"], r["tx"], r["rx"], r["t0"], r["fc"], r["fs"], r["c"], pts,
                                     az=np.pi, el=0.0, bistatic=bist)
        assert np.array_equal(g, dense)


@pytest.mark.parametrize("az,inside", [(0.3, True), (0.3, False), (1.2, True), (1.2, False)])
def test_gate_azimuth_boundary(az, inside):
    """S:150-152 examples: a point at azimuth FWHM/2 - 1e-6 rad is in the FOV, at FWHM/2 + 1e-6
    it is not (sensor at the origin, a = +x, b = +y, single term with ramp data)."""
    Ns = 4096
    d = ((1.0 + np.arange(Ns) / 1024.0) + 1j * 0.5).astype(np.complex64).reshape(1, 1, Ns)
    alpha = az / 2 + (-1e-6 if inside else 1e-6)
    R = 15.0
    x = np.array([[R * np.sin(alpha), R * np.cos(alpha), 0.0]])
    args = (d, np.zeros((1, 3)), np.zeros((1, 1, 3)), None, 120e3, 120e3, 1500.0, x)
    dense = oracle.tdbp_points(*args)[0]
    g = oracle.tdbp_points_gated(*args, az=az)[0]
    assert abs(dense) > 1.0
    assert (g == dense) if inside else (g == 0)


def test_gate_elevation_and_behind():
    """Elevation sector |angle(v, b) in the (b, c) plane| <= el/2 and v.b > 0 (in front)."""
    Ns = 4096
    d = np.ones((1, 1, Ns), dtype=np.complex64)
    args = (d, np.zeros((1, 3)), np.zeros((1, 1, 3)), None, 120e3, 120e3, 1500.0)
    el = 0.5
    # c = a x b = x x y = +z (down); a point depressed by el/2 -/+ 1e-6 below boresight
    for delta, ok in ((-1e-6, True), (1e-6, False)):
        ang = el / 2 + delta
        x = np.array([[0.0, 15.0 * np.cos(ang), 15.0 * np.sin(ang)]])
        g = oracle.tdbp_points_gated(*args, x, az=np.pi, el=el)[0]
        assert (g != 0) == ok
    behind = np.array([[0.0, -15.0, 0.0]])
    assert oracle.tdbp_points_gated(*args, behind, az=np.pi, el=el)[0] == 0
    assert oracle.tdbp_points_gated(*args, behind, az=np.pi, el=0.0)[0] != 0   # no elevation test


def test_gate_monotone_in_beamwidth():
    """Shrinking the FWHM never admits more terms."""
    s = synth.scenario(2, reduced=True)
    e = s.echoes()
    pts = oracle.grid_points(s.grid, s.sample_pixels(200, window=3))
    prev = None
    for az in (np.pi, 1.0, 0.5, 0.277, 0.1):
        _, cnt = oracle.tdbp_points_gated(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, pts, az=az, bistatic=True,
                                          with_count=True)
        if prev is not None:
            assert np.all(cnt <= prev)
        prev = cnt


def test_gate_rigid_rotation_invariance():
    """Rotating positions, ping axes and grid rigidly leaves the gated image unchanged
    (frame invariance of the FOV test)."""
    r = synth.random_case(22, P=4, E=3)
    Rm = synth.rotation_matrix(0.3, -0.2, 1.1)
    rng = np.random.default_rng(5)
    centre = oracle.grid_points(r["grid"]).mean(axis=0)
    axes = []
    for p in range(4):   # boresight roughly at the grid, along-track axis perpendicular to it
        b = centre - r["tx"][p] + rng.normal(size=3) * 0.2
        b /= np.linalg.norm(b)
        a = np.cross(b, rng.normal(size=3)); a /= np.linalg.norm(a)
        axes.append([a, b])
    axes = np.array(axes)
    pts = oracle.grid_points(r["grid"])
    kw = dict(az=0.15, el=2.0, bistatic=True)
    g1, cnt = oracle.tdbp_points_gated(r["echoes"], r["tx"], r["rx"], r["t0"], r["fc"], r["fs"], r["c"], pts,
                                       axes=axes, with_count=True, **kw)
    g2 = oracle.tdbp_points_gated(r["echoes"], r["tx"] @ Rm.T, r["rx"] @ Rm.T, r["t0"], r["fc"], r["fs"], r["c"],
                                  pts @ Rm.T, axes=axes @ Rm.T, **kw)
    assert 0 < cnt.sum() < 4 * 3 * len(pts)             # the gate is active on this grid
    assert np.max(np.abs(g1 - g2)) <= 1e-9 * np.max(np.abs(g1))


def test_gate_cfg1_target_matches_generator_beam():
    """Config 1 with the generator's own hard beam (az = 0.886 lambda / D, tested at tx): at the
    target the gated sum equals the dense sum -- out-of-beam pings carry no echo of it -- and the
    gated image still focuses there with phase ~ 0."""
    s = synth.scenario(1)
    e = s.echoes()
    az = 2 * np.arcsin(s.sin_half_beam)
    x = s.targets
    dense = oracle.tdbp_points(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, x)[0]
    gated = oracle.tdbp_points_gated(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, x, az=az)[0]
    assert abs(gated - dense) <= 1e-12 * abs(dense)
    pts = oracle.grid_points(s.grid, s.sample_pixels(0, window=9))
    gi = np.abs(oracle.tdbp_points_gated(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, pts, az=az))
    assert np.argmax(gi) == np.argmin(np.linalg.norm(pts - x, axis=1))


# ---------------------------------------------------------------- moving receiver (NEXT-2, reading R16)

@pytest.mark.parametrize("x,v,closed", [
    ((30.0, 0, 0), (2.0, 0, 0), lambda R, c, v: 2 * R / (c + v)),            # moving towards the pixel
    ((-30.0, 0, 0), (2.0, 0, 0), lambda R, c, v: 2 * R / (c - v)),           # moving away
    ((0, 30.0, 0), (2.0, 0, 0), lambda R, c, v: 2 * R * c / (c * c - v * v)),  # broadside
])
def test_moving_receiver_delay_closed_forms(x, v, closed):
    """tau = (|x - tx| + |x - rx - v tau|)/c with tx = rx = 0 has closed forms on the motion axis
    and broadside (quadratic (c tau - R)^2 = R^2 + v^2 tau^2)."""
    c = 1500.0
    tau = oracle.delay_moving(x, [0, 0, 0], [0, 0, 0], v, c)
    assert abs(tau - closed(30.0, c, 2.0)) <= 1e-15


def test_moving_receiver_zero_velocity_is_stop_and_hop():
    r = synth.random_case(31)
    pts = oracle.grid_points(r["grid"])
    a = oracle.tdbp_points(r["echoes"], r["tx"], r["rx"], r["t0"], r["fc"], r["fs"], r["c"], pts)
    b = oracle.tdbp_points_motion(r["echoes"], r["tx"], r["rx"], r["t0"], np.zeros((r["tx"].shape[0], 3)),
                                  r["fc"], r["fs"], r["c"], pts)
    assert np.array_equal(a, b)


def test_moving_receiver_focus_cfg1():
    """Config 1 recorded with the platform moving at 2 m/s along track during reception: the
    moving-receiver delay focuses the target at its true pixel with phase ~ 0 and full gain;
    the stop-and-hop delay (R5) loses more than 6 dB on the same data."""
    s = synth.scenario(1)
    s.vel = np.tile([2.0, 0.0, 0.0], (s.P, 1))
    e = s.echoes()
    idx = s.sample_pixels(0, window=9)
    pts = oracle.grid_points(s.grid, idx)
    img = oracle.tdbp_points_motion(e, s.tx, s.rx, s.t0, s.vel, s.fc, s.fs, s.c, pts)
    k = int(np.argmax(np.abs(img)))
    assert tuple(idx[k]) == tuple(s.target_pixels[0])
    assert abs(np.angle(img[k])) <= 1e-2
    x = s.targets[0]
    rt = np.linalg.norm(x[None] - s.tx, axis=1)
    rr = np.linalg.norm(x[None, None] - s.rx, axis=2)
    inbeam = np.abs((x[None] - s.tx)[:, 0]) <= rt * s.sin_half_beam
    bound = np.sum((1.0 / (rt[:, None] * rr))[inbeam])
    assert 0.96 <= abs(img[k]) / bound <= 1.01
    sh = oracle.tdbp_points(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, x[None])[0]
    assert 20 * np.log10(abs(img[k]) / abs(sh)) >= 6.0


# ---------------------------------------------------------------- sediment refraction (NEXT-3, reading R17)

def test_refraction_normal_incidence_closed_form():
    """Sensor straight above the voxel: t = h1/c1 + h2/c2 (Snell at normal incidence)."""
    t = oracle.travel_refracted([0.3, -0.2, 0.5], [0.3, -0.2, -2.0], 0.0, 1500.0, 1700.0)
    assert abs(t - (2.0 / 1500.0 + 0.5 / 1700.0)) <= 1e-17


def test_refraction_reduces_to_straight_path():
    """Equal sound speeds, or a voxel above the interface, give the straight path |x - s| / c1."""
    rng = np.random.default_rng(1)
    for _ in range(20):
        s = np.array([*rng.uniform(-2, 2, 2), rng.uniform(-3, -0.5)])
        x = np.array([*rng.uniform(-2, 2, 2), rng.uniform(0.01, 1.5)])
        assert abs(oracle.travel_refracted(x, s, 0.0, 1500.0, 1500.0) - np.linalg.norm(x - s) / 1500.0) <= 1e-15
        xa = np.array([x[0], x[1], -0.3])
        t = oracle.travel_refracted(xa, s, 0.0, 1500.0, 1700.0)
        assert abs(t - np.linalg.norm(xa - s) / 1500.0) <= 1e-15 * t


def test_refraction_is_fermat_minimum_and_snell():
    """Brute force over interface points: the oracle time is the minimum (Fermat), and at the
    minimiser sin(theta1)/c1 = sin(theta2)/c2 (Snell)."""
    c1, c2 = 1500.0, 1650.0
    s = np.array([0.2, -0.4, -1.8])
    x = np.array([1.7, 0.9, 0.45])
    D = np.hypot(*(x[:2] - s[:2]))
    h1, h2 = -s[2], x[2]
    xi = np.linspace(0, D, 200001)
    tt = np.sqrt(xi ** 2 + h1 ** 2) / c1 + np.sqrt((D - xi) ** 2 + h2 ** 2) / c2
    k = np.argmin(tt)
    t = oracle.travel_refracted(x, s, 0.0, c1, c2)
    assert t <= tt.min() + 1e-15 and tt.min() - t <= 1e-12
    xs = xi[k]
    s1, s2 = xs / np.hypot(xs, h1), (D - xs) / np.hypot(D - xs, h2)
    assert abs(s1 / c1 - s2 / c2) <= 1e-3 * s1 / c1


def test_refraction_focuses_buried_target():
    """A target 0.20 m below the seabed in fast sediment (c2 = 1700 m/s): imaging with the
    refracted delay focuses it at its true voxel; straight water-speed rays place it shallower
    (apparent depth ~ h c1/c2), the P:317 motivation for the interface model."""
    s = synth.scenario(4, reduced=True)
    g = dict(s.grid)
    tgt = np.array([[3.0, 3.1, 0.20]])
    pos, pix = synth._snap(g, tgt)
    s.scat, s.sigma = pos, np.ones(1, dtype=np.complex128)      # the target alone (no speckle)
    s.targets, s.target_pixels = pos, pix
    s.medium = (0.0, 1700.0)
    e = s.echoes()
    idx = s.sample_pixels(0, window=11)
    pts = oracle.grid_points(g, idx)
    a = np.abs(oracle.tdbp_points_refracted(e, s.tx, s.rx, s.t0, 0.0, 1700.0, s.fc, s.fs, s.c, pts))
    b = np.abs(oracle.tdbp_points(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, pts))
    assert tuple(idx[np.argmax(a)]) == tuple(pix[0])
    assert idx[np.argmax(b)][2] < pix[0][2] - 1          # straight rays: shallower by > 1 voxel
