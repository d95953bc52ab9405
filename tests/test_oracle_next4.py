"""Pins of the NEXT-4 oracle functions (interpolation and conditioning
variants) against closed forms, the mathematics of the kernels and config-1 physics:

* ``tdbp_points_weighted`` -- spreading weight R_tx R_rx (R18; Eq. 1 amplitude P:89);
* ``lanczos4`` / ``upsample`` -- 8-tap windowed-sinc xU upsampling (R19);
* ``baseband`` -- real passband -> complex baseband, mix + FIR + decimate (R20).
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


def _ramp(Ns):
    n = np.arange(Ns, dtype=np.float64)
    return ((1.0 + n / 1024.0) + 1j * (2.0 - n / 2048.0)).astype(np.complex64)


# ---------------------------------------------------------------- R18 spreading weight

@pytest.mark.parametrize("case", _load("closed_form.json")["cases"], ids=lambda c: c["name"])
def test_weighted_closed_form(case):
    """P = E = 1: I_w(x) = R_tx R_rx ehat(u) exp(+j 2 pi fc tau), R_tx R_rx hand-derived."""
    w = _load("next4.json")["weight_cases"]["weights"][case["name"]]
    Ns = 4096
    ech = _ramp(Ns).reshape(1, 1, Ns)
    val = oracle.tdbp_points_weighted(ech, np.array([case["tx"]]), np.array([[case["rx"]]]),
                                      np.array([case["t0"]]), case["fc"], case["fs"], case["c"],
                                      np.array([case["x"]]))[0]
    u, cyc = case["u"], case["cycles"]
    ehat = (1.0 + u / 1024.0) + 1j * (2.0 - u / 2048.0)
    expected = w * ehat * np.exp(2j * np.pi * (cyc - np.floor(cyc)))
    assert abs(val - expected) <= 1e-9 * abs(expected)


def test_weighted_cfg1_peak_counts_in_beam_terms():
    """Echoes carry sigma / (R_tx R_rx) (Eq. 1); the weight cancels it at the target, so the
    peak is the number of in-beam terms times the compressed-pulse peak (1) up to the linear
    interpolation loss (<= 2.6 % at fs = 4B, cfg1_physics.json), phase ~ 0, and the unweighted
    image's peak pixel is unchanged."""
    s = synth.scenario(1)
    e = s.echoes()
    x = s.targets[0]
    offs = np.arange(-3, 4) * s.grid["step_x"][0]
    pts = np.array([[x[0] + a, x[1] + b, 0.0] for b in offs for a in offs])
    vw = oracle.tdbp_points_weighted(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, pts)
    rt = np.linalg.norm(x[None] - s.tx, axis=1)
    n_in = int(np.sum(np.abs((x[None] - s.tx)[:, 0]) <= rt * s.sin_half_beam)) * s.E
    i0 = len(pts) // 2
    assert int(np.argmax(np.abs(vw))) == i0
    assert 0.97 * n_in <= abs(vw[i0]) <= n_in
    assert abs(np.angle(vw[i0])) <= 1e-2


def test_weighted_is_linear_in_weights():
    """Translating every position and the points leaves R_tx, R_rx and the image unchanged;
    scaling the echoes scales I_w (linearity)."""
    r = synth.random_case(7)
    e = r["echoes"]
    pts = oracle.grid_points(r["grid"])
    a = oracle.tdbp_points_weighted(e, r["tx"], r["rx"], r["t0"], r["fc"], r["fs"], r["c"], pts)
    sh = np.array([1.0e3, -3.0e2, 0.0])
    b = oracle.tdbp_points_weighted(e, r["tx"] + sh, r["rx"] + sh, r["t0"], r["fc"], r["fs"], r["c"], pts + sh)
    assert np.max(np.abs(a - b)) <= 1e-9 * np.max(np.abs(a))
    c2 = oracle.tdbp_points_weighted((2.0 * e).astype(np.complex64), r["tx"], r["rx"], r["t0"], r["fc"], r["fs"],
                                     r["c"], pts)
    assert np.max(np.abs(c2 - 2.0 * a)) <= 1e-12 * np.max(np.abs(a))


# ---------------------------------------------------------------- R19 8-tap windowed sinc

def test_lanczos4_hand_values():
    g = _load("next4.json")["lanczos4"]
    for s, v in g["values"]:
        assert abs(oracle.lanczos4(s) - v) <= g["tol"], s


def test_upsample_identity_and_interpolating():
    """U = 1 is the identity; the r = 0 phase of any U returns the input samples (L(m) = delta_m)."""
    rng = np.random.default_rng(11)
    x = (rng.normal(size=(3, 97)) + 1j * rng.normal(size=(3, 97))).astype(np.complex64)
    y1 = oracle.upsample(x, 1)
    assert np.max(np.abs(y1 - x)) <= 1e-14 * np.max(np.abs(x))
    for U in (2, 3, 4, 8):
        y = oracle.upsample(x, U)
        assert y.shape == (3, 97 * U)
        assert np.max(np.abs(y[:, ::U] - x)) <= 1e-14 * np.max(np.abs(x))


@pytest.mark.parametrize("f", [0.02, 0.05, 0.1, -0.08])
def test_upsample_reproduces_band_limited_exponentials(f):
    """A complex exponential well inside the band is interpolated to the continuous one
    (windowed-sinc passband error < 5e-3 for |f| <= 0.1 cycles/sample); an index, sign or
    phase error would be O(1)."""
    U, Ns = 4, 128
    n = np.arange(Ns)
    x = np.exp(2j * np.pi * f * n).astype(np.complex64)
    y = oracle.upsample(x, U)
    t = np.arange(U * Ns) / U
    inner = (t >= 4) & (t <= Ns - 5)
    assert np.max(np.abs(y - np.exp(2j * np.pi * f * t))[inner]) <= 5e-3


def test_upsample_impulse_response_is_the_symmetric_kernel_support():
    """Upsampling delta[n0] gives the kernel sampled at j/U: symmetric about n0, zero at the
    other input instants, zero at |j/U - n0| >= 4 (8 taps)."""
    U, Ns, n0 = 4, 40, 20
    x = np.zeros(Ns, dtype=np.complex64)
    x[n0] = 1.0
    y = oracle.upsample(x, U)
    j = np.arange(U * Ns) - U * n0
    assert abs(y[U * n0] - 1.0) <= 1e-15
    for k in range(1, 4 * U):
        assert abs(y[U * n0 + k] - y[U * n0 - k]) <= 1e-15
    assert np.all(np.abs(y[(j % U == 0) & (j != 0)]) <= 1e-15)
    assert np.all(np.abs(y[np.abs(j) >= 4 * U]) == 0.0)
    assert np.all(np.abs(y[(np.abs(j) < 4 * U) & (j % U != 0)]) > 1e-4)


def test_upsample_dc_gain():
    """The 8-tap window's partition of unity: a constant is reproduced within 0.5 %."""
    x = np.ones(64, dtype=np.complex64)
    y = oracle.upsample(x, 8)
    assert np.max(np.abs(y[8 * 4: 8 * 59] - 1.0)) <= 5e-3


def _cfg1_at(fs_ratio):
    """Config 1 recorded at fs = fs_ratio * B (the generator's compressed sinc pulse)."""
    base = synth.scenario(1)
    fs = fs_ratio * base.bandwidth
    Ns = int(np.ceil(2048 * fs / base.fs / 8) * 8)
    hf = dict(synth.HF)
    hf["fs"] = fs
    s = synth.stripmap("cfg1_fs", P=base.P, E=base.E, **hf, altitude=10.0, track=(base.tx[0, 0], base.tx[-1, 0]),
                       grid=base.grid, Ns=Ns, t0=0.012, targets=base.targets, n_speckle=0)
    return s, s.echoes()


def test_upsampling_recovers_focus_at_low_sampling_rate():
    """Config 1 recorded at fs = 1.25 B: linear interpolation of the critically-sampled sinc pulse
    loses ~15 % of the peak (mean sinc loss at up to 0.4 samples of offset), while x4 8-tap
    upsampling followed by the same linear TDBP at 4 fs loses < 3 % (S:396's design: 'band-
    limited via 8-tap windowed-sinc on the upsampled (x4) compressed series')."""
    s, e = _cfg1_at(1.25)
    x = s.targets[0]
    rt = np.linalg.norm(x[None] - s.tx, axis=1)
    rr = np.linalg.norm(x[None, None] - s.rx, axis=2)
    inbeam = np.abs((x[None] - s.tx)[:, 0]) <= rt * s.sin_half_beam
    bound = np.sum((1.0 / (rt[:, None] * rr))[inbeam])
    lin = abs(oracle.tdbp_points(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, x[None])[0]) / bound
    eu = oracle.upsample(e, 4).astype(np.complex64)
    up = oracle.tdbp_points(eu, s.tx, s.rx, s.t0, s.fc, 4 * s.fs, s.c, x[None])[0]
    assert lin < 0.92, lin
    assert 0.97 <= abs(up) / bound <= 1.0, abs(up) / bound
    assert abs(np.angle(up)) <= 1e-2


# ---------------------------------------------------------------- R20 basebanding

def test_baseband_hand_values():
    g = _load("next4.json")["baseband"]
    fc, fs = g["fc"], g["fs_in"]
    x = np.array(g["a"]["x"], dtype=np.float32).reshape(1, 1, -1)
    ya = oracle.baseband(x, fs, fc, None, [1.0], 1, 5)[0, 0]
    assert np.max(np.abs(ya - (np.array(g["a"]["y_re"]) + 1j * np.array(g["a"]["y_im"])))) <= 1e-12
    yb = oracle.baseband(x, fs, fc, np.array([g["b"]["t0"]]), [1.0], 1, 5)[0, 0]
    assert np.max(np.abs(yb - (np.array(g["b"]["y_re"]) + 1j * np.array(g["b"]["y_im"])))) <= 1e-9
    c = g["c"]
    xi = np.zeros((1, 1, c["Nin"]), dtype=np.float32)
    xi[0, 0, c["n0"]] = 1.0
    yc = oracle.baseband(xi, fs, fc, None, c["h"], c["D"], c["Nout"])[0, 0]
    assert np.max(np.abs(yc - (np.array(c["y_re"]) + 1j * np.array(c["y_im"])))) <= 1e-12


def _lowpass(n_half, cutoff):
    """Hann-windowed sinc low-pass, cutoff in cycles/sample, unit DC gain (test-side design)."""
    k = np.arange(-n_half, n_half + 1)
    h = 2 * cutoff * np.sinc(2 * cutoff * k) * (0.5 + 0.5 * np.cos(np.pi * k / (n_half + 1)))
    return h / h.sum()


def test_baseband_tone_is_the_analytic_signal():
    """A passband tone a cos(2 pi (fc + d) t + th) mixes to (a/2) exp(j(2 pi d t + th)) plus an image
    at -(2 fc + d) that the low-pass removes: with taps 2h (unit DC gain h) the output is
    a exp(j(2 pi d t_m + th)) at t_m = t0 + m D / fs_in, within the filter's ripple."""
    fs_in, fc, D = 480e3, 120e3, 4
    d, th, a, t0 = 7.5e3, 0.7, 0.8, 0.0123
    Nin = 4096
    t = t0 + np.arange(Nin) / fs_in
    x = (a * np.cos(2 * np.pi * (fc + d) * t + th)).astype(np.float32).reshape(1, 1, Nin)
    h = 2.0 * _lowpass(48, 0.08)   # pass |f| <= 0.05 fs_in (24 kHz), stop the image at 0.5 fs_in
    Nout = Nin // D
    y = oracle.baseband(x, fs_in, fc, np.array([t0]), h, D, Nout)[0, 0]
    tm = t0 + np.arange(Nout) * D / fs_in
    inner = slice(16, Nout - 16)
    ref = a * np.exp(1j * (2 * np.pi * d * tm + th))
    assert np.max(np.abs(y - ref)[inner]) <= 1e-2 * a


def test_baseband_channel_layout_and_t0_per_ping():
    """Channel (p, e) uses t0_p (R4): the same data under two pings differ by exp(-j 2 pi fc dt0)."""
    rng = np.random.default_rng(5)
    x1 = rng.normal(size=(1, 1, 256)).astype(np.float32)
    x = np.repeat(np.repeat(x1, 2, axis=0), 3, axis=1)
    fc, fs = 30e3, 120e3
    t0 = np.array([0.001, 0.001 + 1.0 / (8 * fc)])
    h = _lowpass(8, 0.2)
    y = oracle.baseband(x, fs, fc, t0, h, 2, 128)
    assert np.max(np.abs(y[0] - y[0, :1])) == 0.0
    assert np.max(np.abs(y[1] - y[0] * np.exp(-2j * np.pi / 8))) <= 1e-9 * np.max(np.abs(y))


# ---------------------------------------------------------------- R21 spectral whitening

def test_whitening_gain_hand_values():
    g = _load("next4.json")["whitening"]
    # (a) unit impulse at every block start: flat periodogram -> 0 dB everywhere
    M, B = 16, 5
    x = np.zeros((3, M * B), dtype=np.complex64)
    x[:, ::M] = 1.0
    G, P = oracle.whitening_gain(x, M, 0.0)
    assert np.max(np.abs(P - 1.0)) <= 1e-12 and np.max(np.abs(G - 1.0)) <= 1e-12
    # (b) P = [1, 4], gamma = 0 -> G = [1, 1/4] = [0, -6.02] dB
    b = g["b"]
    xb = np.tile(np.array(b["block"], dtype=np.complex64), 7).reshape(1, -1)
    G, P = oracle.whitening_gain(xb, b["M"], 0.0)
    assert np.allclose(P, b["P"], atol=1e-12) and np.allclose(G, b["G"], atol=1e-12)
    assert np.allclose(10 * np.log10(G), b["dB"], atol=1e-4)
    # (c) gamma = 1
    G, _ = oracle.whitening_gain(xb, b["M"], g["c"]["gamma"])
    assert np.allclose(G, g["c"]["G"], atol=1e-7)
    # (d) gamma -> infinity: no shaping
    G, _ = oracle.whitening_gain(xb, b["M"], 1e12)
    assert np.max(np.abs(G - 1.0)) <= 1e-11


def test_whitening_gain_partial_block_and_zero_batch():
    """Ns < M: one zero-padded block; an all-zero batch has no spectrum (error)."""
    x = np.zeros((2, 5), dtype=np.complex64)
    x[:, 0] = 1.0
    G, P = oracle.whitening_gain(x, 8, 0.0)
    assert np.allclose(P, 1.0) and np.allclose(G, 1.0)
    with pytest.raises(ValueError):
        oracle.whitening_gain(np.zeros((2, 64), dtype=np.complex64), 8, 0.0)


def test_whitened_compression_with_unit_gain_is_plain_compression():
    """G = 1: w = delta[i], the cascade is exactly the matched filter of R14."""
    rng = np.random.default_rng(21)
    x = ((rng.normal(size=(2, 300)) + 1j * rng.normal(size=(2, 300))) / np.sqrt(2)).astype(np.complex64)
    r = ((rng.normal(size=17) + 1j * rng.normal(size=17))).astype(np.complex64)
    for M in (1, 2, 16):
        y = oracle.rangecompress_whitened(x, r, np.ones(M))
        assert np.max(np.abs(y - oracle.rangecompress(x, r))) <= 1e-12 * np.max(np.abs(y))


def test_whitening_flattens_coloured_noise():
    """Coloured noise (white noise through a 2-tap low-pass, spectrum 4 cos^2(pi f)): after the
    whitening FIR with the estimated gain (gamma = 0) the batch periodogram's max/min ratio falls
    by more than 10x (Eq. 9's purpose: 'flatten the spectrum'); the impulse replica r = [1] makes
    the compression the identity."""
    rng = np.random.default_rng(5)
    n = (rng.normal(size=(8, 4097)) + 1j * rng.normal(size=(8, 4097))) / np.sqrt(2)
    x = (n[:, 1:] + 0.8 * n[:, :-1]).astype(np.complex64)
    M = 32
    G, P = oracle.whitening_gain(x, M, 0.0)
    assert P.max() / P.min() > 30
    xw = oracle.rangecompress_whitened(x, np.array([1.0], dtype=np.complex64), G).astype(np.complex64)
    _, Pw = oracle.whitening_gain(xw, M, 0.0)
    assert (Pw.max() / Pw.min()) * 10 < P.max() / P.min()
    assert Pw.max() / Pw.min() < 3.0


def test_gated_weighted_reduces_to_its_parts():
    """The combined gate + weight: a wide-open beam equals the weighted sum; with weights the
    gated sum of the config-1 target equals the in-beam count (as the weighted dense one, since the
    generator's echoes carry only in-beam scatterer terms)."""
    r = synth.random_case(9)
    e = r["echoes"]
    pts = oracle.grid_points(r["grid"])
    a = oracle.tdbp_points_gated_weighted(e, r["tx"], r["rx"], r["t0"], r["fc"], r["fs"], r["c"], pts, az=4.0)
    b = oracle.tdbp_points_weighted(e, r["tx"], r["rx"], r["t0"], r["fc"], r["fs"], r["c"], pts)
    assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(b))
    s = synth.scenario(1)
    e1 = s.echoes()
    x = s.targets[0][None]
    az = 2 * np.arcsin(s.sin_half_beam)
    g = oracle.tdbp_points_gated_weighted(e1, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, x, az=az)[0]
    w = oracle.tdbp_points_weighted(e1, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, x)[0]
    assert abs(g - w) <= 1e-3 * abs(w)
