"""GPU-vs-oracle parity of the NEXT-4 interpolation / conditioning variants through the C ABI
(-m gpu): spreading weight R_tx R_rx in K2 (R18), 8-tap windowed-sinc xU upsampling (K1b, R19)
and passband basebanding (K0, R20).  Same bar as tests/test_gpu_parity.py for images
(max|err| <= 1e-3 max|I|, <= 1e-2 rad at peaks); the conditioning kernels are plain fp32
filters compared element by element at 2e-5 of the oracle's max."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL_MAG = 1e-3
TOL_PHASE = 1e-2
TOL_FILT = 2e-5


@pytest.fixture(scope="module")
def bpmod(require_gpu):
    import torch
    torch.cuda.set_device(0)
    from paper_2101_05888_b200 import _build
    _build.build()
    import paper_2101_05888_b200 as pkg
    return pkg


def _check(got, ref, label=""):
    scale = np.max(np.abs(ref))
    assert scale > 0, f"{label}: oracle output is all zero -- the case tests nothing"
    err = np.max(np.abs(got - ref))
    assert err <= TOL_MAG * scale, f"{label}: max|err| = {err:.3e} > {TOL_MAG} * {scale:.3e}"
    return err / scale


def _at(img, idx):
    return img[idx[:, 2], idx[:, 1], idx[:, 0]]


def _grid_idx(g):
    iz, iy, ix = np.meshgrid(np.arange(g["nz"]), np.arange(g["ny"]), np.arange(g["nx"]), indexing="ij")
    return np.stack([ix.ravel(), iy.ravel(), iz.ravel()], axis=1)


def _weighted_ref(s, e, idx):
    pts = oracle.grid_points(s.grid, idx)
    return oracle.tdbp_points_weighted(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, pts)


def _weighted_form(bpmod, s, e, beam=None):
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(e, s.tx, s.rx, s.t0)
        bp.set_weighting(True)
        if beam is not None:
            bp.set_beam(beam)
        return bp.form(), bp.plan()


# ------------------------------------------------------------------ R18 spreading weight

@pytest.mark.parametrize("cid", [1, 2, 3, 4])
def test_weighted_full_image(bpmod, cid):
    """Full images of config 1 and the reduced configs 2-4 (series and near-field exact modes)."""
    s = synth.scenario(cid, reduced=(cid != 1))
    e = s.echoes()
    got, plan = _weighted_form(bpmod, s, e)
    idx = _grid_idx(s.grid)
    ref = _weighted_ref(s, e, idx)
    _check(_at(got, idx), ref, label=f"weighted {s.name} ({plan['rx_mode']})")
    pk = s.target_pixels
    pref = _weighted_ref(s, e, pk)
    dph = np.angle(_at(got, pk) * np.conj(pref))
    assert np.max(np.abs(dph)) <= TOL_PHASE


def test_weighted_cfg1_focus_counts_in_beam_terms(bpmod):
    """The weight cancels the 1/(R_tx R_rx) echo amplitude at the target: the GPU peak is at the
    target pixel and holds >= 0.97 of the in-beam term count (oracle pin)."""
    s = synth.scenario(1)
    img, _ = _weighted_form(bpmod, s, s.echoes())
    img = img[0]
    iy, ix = np.unravel_index(np.argmax(np.abs(img)), img.shape)
    assert (ix, iy) == tuple(s.target_pixels[0][:2])
    x = s.targets[0]
    rt = np.linalg.norm(x[None] - s.tx, axis=1)
    n_in = int(np.sum(np.abs((x[None] - s.tx)[:, 0]) <= rt * s.sin_half_beam)) * s.E
    assert 0.97 * n_in <= abs(img[iy, ix]) <= n_in * (1 + 1e-5)


def test_weighted_gated_matches_weighted_oracle_in_cone(bpmod):
    """Weight and gate together: reduced config 2 with the generator's beam; the gated weighted
    oracle is the weighted oracle on gated terms -- checked through linearity: for a beam wide
    open the result equals the dense weighted image bitwise."""
    s = synth.scenario(2, reduced=True)
    e = s.echoes()
    dense, _ = _weighted_form(bpmod, s, e)
    opened, _ = _weighted_form(bpmod, s, e, beam=3.5)
    assert np.array_equal(dense, opened)


def test_weighted_full_size_cfg2_sampled(bpmod):
    """Full config-2 size (the bench workload) with the weight on: sampled pixels vs the oracle."""
    s = synth.scenario(2)
    e = s.echoes()
    got, _ = _weighted_form(bpmod, s, e)
    idx = s.sample_pixels(1024, window=5, seed=9)
    _check(_at(got, idx), _weighted_ref(s, e, idx), label="weighted cfg2 full")


def test_weighting_off_is_bitwise_dense(bpmod):
    s = synth.scenario(1)
    e = s.echoes()
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(e, s.tx, s.rx, s.t0)
        a = bp.form()
        bp.set_weighting(True)
        bp.set_weighting(False)
        b = bp.form()
    assert np.array_equal(a, b)


def test_set_weighting_errors(bpmod):
    s = synth.scenario(1)
    e = s.echoes()
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(e, s.tx, s.rx, s.t0)
        assert bpmod.load_library().sas_bp_set_weighting(bp._h, 2) == bpmod.sasbp.SAS_E_INVALID
        bp.set_weighting(True)
        bp.set_motion(np.zeros((s.P, 3)))
        with pytest.raises(bpmod.SasError) as ei:
            bp.form()
        assert ei.value.status == bpmod.sasbp.SAS_E_UNSUPPORTED
        bp.set_motion(None)
        bp.set_medium(1.0, 1700.0)
        with pytest.raises(bpmod.SasError) as ei:
            bp.form()
        assert ei.value.status == bpmod.sasbp.SAS_E_UNSUPPORTED


# ------------------------------------------------------------------ R19 xU upsampling

@pytest.mark.parametrize("U,Ns", [(1, 100), (2, 1), (2, 1023), (3, 1025), (4, 7), (4, 3000), (5, 2049), (8, 777),
                                  (16, 130)])
def test_upsample_vs_oracle(bpmod, U, Ns):
    rng = np.random.default_rng(U * 1000 + Ns)
    x = ((rng.normal(size=(3, 2, Ns)) + 1j * rng.normal(size=(3, 2, Ns))) / np.sqrt(2)).astype(np.complex64)
    got = bpmod.upsample(x, U)
    ref = oracle.upsample(x, U)
    assert got.shape == ref.shape
    assert np.max(np.abs(got - ref)) <= TOL_FILT * np.max(np.abs(ref))


def test_upsample_device_matches_host(bpmod):
    import torch
    rng = np.random.default_rng(2)
    x = ((rng.normal(size=(5, 4000)) + 1j * rng.normal(size=(5, 4000))) / np.sqrt(2)).astype(np.complex64)
    xd = torch.from_numpy(x).cuda()
    out = torch.empty((5, 16000), dtype=torch.complex64, device="cuda")
    bpmod.upsample_device(xd, 4, out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), bpmod.upsample(x, 4))


def test_upsample_errors(bpmod):
    x = np.zeros((2, 8), dtype=np.complex64)
    for U in (0, 17):
        with pytest.raises(bpmod.SasError):
            bpmod.upsample(x, U)


def _cfg1_at(fs_ratio):
    base = synth.scenario(1)
    fs = fs_ratio * base.bandwidth
    Ns = int(np.ceil(2048 * fs / base.fs / 8) * 8)
    hf = dict(synth.HF)
    hf["fs"] = fs
    s = synth.stripmap("cfg1_fs", P=base.P, E=base.E, **hf, altitude=10.0, track=(base.tx[0, 0], base.tx[-1, 0]),
                       grid=base.grid, Ns=Ns, t0=0.012, targets=base.targets, n_speckle=0)
    return s, s.echoes()


def test_upsample_then_backproject_cfg1_low_rate(bpmod):
    """Config 1 recorded at fs = 1.25 B, x4 upsampled on the GPU, linear TDBP at 4 fs on the GPU,
    vs the oracle chain (oracle upsampling + oracle TDBP); focus at the target (R19 pin)."""
    s, e = _cfg1_at(1.25)
    eu = bpmod.upsample(e, 4)
    with bpmod.Backprojector(s.fc, s.bandwidth, 4 * s.fs, s.c, s.grid) as bp:
        bp.set_pings(eu, s.tx, s.rx, s.t0)
        got = bp.form()
    ou = oracle.upsample(e, 4).astype(np.complex64)
    ref = oracle.tdbp_grid(ou, s.tx, s.rx, s.t0, s.fc, 4 * s.fs, s.c, s.grid)
    _check(got, ref, label="upsample -> backproject")
    img = got[0]
    iy, ix = np.unravel_index(np.argmax(np.abs(img)), img.shape)
    assert (ix, iy) == tuple(s.target_pixels[0][:2])
    assert abs(np.angle(img[iy, ix])) <= TOL_PHASE


# ------------------------------------------------------------------ R20 basebanding

def _lowpass(n_half, cutoff):
    k = np.arange(-n_half, n_half + 1)
    h = 2 * cutoff * np.sinc(2 * cutoff * k) * (0.5 + 0.5 * np.cos(np.pi * k / (n_half + 1)))
    return (h / h.sum()).astype(np.float32)


@pytest.mark.parametrize("P,E,Nin,D,Nh,Nout", [(1, 1, 1, 1, 1, 1), (2, 3, 4096, 4, 65, 1024), (3, 2, 5000, 4, 33, 1300),
                                               (1, 4, 999, 1, 7, 999), (2, 2, 3000, 37, 255, 90),
                                               (1, 2, 20000, 2, 1023, 10000), (2, 1, 700, 3, 1, 300), (1, 1, 3000, 64, 129, 47),
                                               (1, 1, 70000, 300, 601, 233)])
@pytest.mark.parametrize("path", ["blocked", "simple"])
def test_baseband_vs_oracle(bpmod, P, E, Nin, D, Nh, Nout, path, monkeypatch):
    """Both kernels (register-blocked polyphase default; the simple one for huge decimations)."""
    if path == "simple":
        monkeypatch.setenv("SASBP_BB_SIMPLE", "1")
    rng = np.random.default_rng(P * 7 + Nin + D + Nh)
    x = rng.normal(size=(P, E, Nin)).astype(np.float32)
    h = (2.0 * _lowpass((Nh - 1) // 2, 0.4 / D)) if Nh > 1 else np.array([1.0], dtype=np.float32)
    t0 = 0.0123 + 1e-4 * np.arange(P)
    fs, fc = 480e3, 120e3 + 17.0
    got = bpmod.baseband(x, fs, fc, t0, h, D, Nout)
    ref = oracle.baseband(x, fs, fc, t0, h, D, Nout)
    assert np.max(np.abs(got - ref)) <= TOL_FILT * max(np.max(np.abs(ref)), 1e-30) or np.max(np.abs(ref)) == 0


def test_baseband_device_t0(bpmod):
    """Device variant with a device t0 array (per-ping carrier phase computed on the GPU)."""
    import torch
    rng = np.random.default_rng(4)
    x = rng.normal(size=(3, 2, 2048)).astype(np.float32)
    h = 2.0 * _lowpass(16, 0.1)
    t0 = np.array([0.0123, 0.0456, 0.0789])
    out = torch.empty((3, 2, 512), dtype=torch.complex64, device="cuda")
    bpmod.baseband_device(torch.from_numpy(x).cuda(), 480e3, 120e3 + 3.0, torch.from_numpy(t0).cuda(),
                          torch.from_numpy(h).cuda(), 4, out)
    torch.cuda.synchronize()
    ref = oracle.baseband(x, 480e3, 120e3 + 3.0, t0, h, 4, 512)
    assert np.max(np.abs(out.cpu().numpy() - ref)) <= TOL_FILT * np.max(np.abs(ref))


def test_baseband_device_and_t0_none(bpmod):
    import torch
    rng = np.random.default_rng(3)
    x = rng.normal(size=(2, 3, 4096)).astype(np.float32)
    h = 2.0 * _lowpass(24, 0.1)
    out = torch.empty((2, 3, 1024), dtype=torch.complex64, device="cuda")
    bpmod.baseband_device(torch.from_numpy(x).cuda(), 480e3, 120e3, None, torch.from_numpy(h).cuda(), 4, out)
    torch.cuda.synchronize()
    ref = oracle.baseband(x, 480e3, 120e3, None, h, 4, 1024)
    assert np.max(np.abs(out.cpu().numpy() - ref)) <= TOL_FILT * np.max(np.abs(ref))


def test_baseband_errors(bpmod):
    x = np.zeros((1, 1, 16), dtype=np.float32)
    for kw in (dict(h=np.ones(2)), dict(D=0), dict(fs=-1.0), dict(h=np.ones(1025))):
        a = dict(fs=480e3, h=np.ones(3), D=2)
        a.update(kw)
        with pytest.raises(bpmod.SasError):
            bpmod.baseband(x, a["fs"], 120e3, None, a["h"], a["D"], 8)


def test_baseband_tone_then_backproject_shape(bpmod):
    """End to end: passband tone -> GPU baseband equals the analytic signal (R20 pin, on the GPU)."""
    fs_in, fc, D = 480e3, 120e3, 4
    d, th, a, t0 = 7.5e3, 0.7, 0.8, 0.0123
    Nin = 4096
    t = t0 + np.arange(Nin) / fs_in
    x = (a * np.cos(2 * np.pi * (fc + d) * t + th)).astype(np.float32).reshape(1, 1, Nin)
    h = 2.0 * _lowpass(48, 0.08)
    y = bpmod.baseband(x, fs_in, fc, np.array([t0]), h, D, Nin // D)[0, 0]
    tm = t0 + np.arange(Nin // D) * D / fs_in
    inner = slice(16, Nin // D - 16)
    assert np.max(np.abs(y - a * np.exp(1j * (2 * np.pi * d * tm + th)))[inner]) <= 1e-2 * a


# ------------------------------------------------------------------ R21 spectral whitening

def _coloured(seed, nch=6, Ns=5000):
    rng = np.random.default_rng(seed)
    n = (rng.normal(size=(nch, Ns + 1)) + 1j * rng.normal(size=(nch, Ns + 1))) / np.sqrt(2)
    return (n[:, 1:] + 0.8 * n[:, :-1]).astype(np.complex64)


@pytest.mark.parametrize("M,gamma,Ns", [(1, 0.0, 100), (2, 0.0, 999), (32, 0.0, 5000), (64, 0.1, 3000),
                                        (256, 1.0, 4096), (64, 0.0, 40), (48, 0.2, 2000), (4, 0.0, 4099), (16, 0.0, 3001),
                                        (128, 0.0, 1000)])
@pytest.mark.parametrize("path", ["reg", "radix2", "dft"])
def test_whitening_gain_vs_oracle(bpmod, M, gamma, Ns, path, monkeypatch):
    """The three periodogram kernels: register FFT (M = 16 R), shared-memory radix-2 (power-of-two
    M) and the direct DFT (any even M)."""
    if path == "dft":
        monkeypatch.setenv("SASBP_WH_DFT", "1")
    if path == "radix2":
        monkeypatch.setenv("SASBP_WH_RADIX2", "1")
    x = _coloured(M + Ns, Ns=Ns)
    got = bpmod.whitening_gain(x, M, gamma)
    ref, _ = oracle.whitening_gain(x, M, gamma)
    assert np.max(np.abs(got - ref)) <= 2e-5


def test_whitening_gain_errors(bpmod):
    with pytest.raises(bpmod.SasError):
        bpmod.whitening_gain(np.zeros((2, 128), dtype=np.complex64), 16, 0.0)
    for M in (0, 3, 258):
        with pytest.raises(bpmod.SasError):
            bpmod.whitening_gain(np.ones((2, 128), dtype=np.complex64), M, 0.0)


@pytest.mark.parametrize("M,Ns,Nr,path", [(32, 3000, 600, "fft"), (64, 10240, 600, "fft"), (2, 777, 160, "fft"),
                                          (1, 500, 40, "fft"), (256, 5000, 1793, "fft"), (64, 3000, 600, "direct")])
def test_rangecompress_whitened_vs_oracle(bpmod, M, Ns, Nr, path, monkeypatch):
    """The composed single-pass K1 (filter conj(w) (x) r, start lag 1 - M/2) equals the oracle's
    cascade (whitening FIR, then the matched filter)."""
    if path == "direct":
        monkeypatch.setenv("SASBP_RC_DIRECT", "1")
    x = _coloured(Ns + M, nch=4, Ns=Ns)
    rng = np.random.default_rng(Nr)
    rep = ((rng.normal(size=Nr) + 1j * rng.normal(size=Nr)) / np.sqrt(2 * Nr)).astype(np.complex64)
    G, _ = oracle.whitening_gain(x, M, 0.05)
    got = bpmod.rangecompress_whitened(x, rep, G.astype(np.float32))
    ref = oracle.rangecompress_whitened(x, rep, G.astype(np.float32).astype(np.float64))
    assert np.max(np.abs(got - ref)) <= 2e-5 * np.max(np.abs(ref))


def test_whitening_device_chain(bpmod):
    """Device pipeline: gain estimated on the GPU feeds the whitened compression on the GPU."""
    import torch
    x = _coloured(9, nch=8, Ns=4096)
    rep = np.exp(1j * np.linspace(0, 20, 100) ** 2 / 20).astype(np.complex64) / np.float32(10)
    xd = torch.from_numpy(x).cuda()
    G = torch.empty(64, dtype=torch.float32, device="cuda")
    bpmod.whitening_gain_device(xd, 64, 0.0, G)
    out = torch.empty_like(xd)
    bpmod.rangecompress_whitened_device(xd, torch.from_numpy(rep).cuda(), G, out)
    torch.cuda.synchronize()
    Gh = G.cpu().numpy()
    ref = oracle.rangecompress_whitened(x, rep, Gh.astype(np.float64))
    got = out.cpu().numpy()
    assert np.max(np.abs(got - ref)) <= 2e-5 * np.max(np.abs(ref))


@pytest.mark.parametrize("cid,bistatic", [(2, False), (3, True)])
def test_weighted_gated_vs_oracle(bpmod, cid, bistatic):
    """Gate (R15) and weight (R18) together: reduced configs with the generator's beam."""
    s = synth.scenario(cid, reduced=True)
    e = s.echoes()
    az = 2 * float(np.arcsin(s.sin_half_beam))
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(e, s.tx, s.rx, s.t0)
        bp.set_weighting(True)
        bp.set_beam(az, 0.0, bistatic, True)
        got = bp.form()
    idx = _grid_idx(s.grid)
    pts = oracle.grid_points(s.grid, idx)
    ref = oracle.tdbp_points_gated_weighted(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, pts, az=az, bistatic=bistatic)
    _check(_at(got, idx), ref, label=f"weighted+gated {s.name}")


@pytest.mark.parametrize("how", ["odd_ns", "env"])
def test_weighted_cp_async_path(bpmod, how, monkeypatch):
    """The WEIGHT instantiation on the cp.async staging path (odd Ns, or SASBP_NO_TMA=1)."""
    s = synth.scenario(2, reduced=True)
    e = s.echoes()
    if how == "odd_ns":
        e = np.ascontiguousarray(e[:, :, :-1])
    else:
        monkeypatch.setenv("SASBP_NO_TMA", "1")
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(e, s.tx, s.rx, s.t0)
        bp.set_weighting(True)
        assert bp.plan()["tma"] is False
        got = bp.form()
    idx = _grid_idx(s.grid)
    pts = oracle.grid_points(s.grid, idx)
    ref = oracle.tdbp_points_weighted(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, pts)
    _check(_at(got, idx), ref, label=f"weighted cp.async {how}")


def test_weighted_streamed_matches_form(bpmod):
    """sas_bp_form_streamed (chunked H2D + accumulating launches) honours the weight."""
    s = synth.scenario(2, reduced=True)
    e = s.echoes()
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_weighting(True)
        a = bp.form_streamed(e, s.tx, s.rx, s.t0, chunks=3)
        bp.set_pings(e, s.tx, s.rx, s.t0)
        b = bp.form()
    assert np.max(np.abs(a - b)) <= 1e-5 * np.max(np.abs(b))


@pytest.mark.parametrize("Nin,Nh,Nout", [(4096, 63, 1024), (4096, 3, 1024), (4096, 5, 1000), (4096, 7, 1030),
                                         (8192, 1, 2048), (12, 9, 5), (4100, 201, 1025)])
def test_baseband_vec4_staging(bpmod, Nin, Nh, Nout, monkeypatch):
    """D = 4 with 16-byte aligned rows: the complex-tap kernel (default) and the mixed blocked
    kernel (SASBP_BB_LEGACY=1) stage the passband input with aligned float4 loads; the
    window start nlo = m0 D - (Nh - 1)/2 takes every residue mod 4 over these Nh (o = 0, 3, 2, 1),
    record edges (nlo < 0, the end past Nin) and Nout not a multiple of the CTA's run.  Against the
    fp64 oracle (R20) and the scalar staging path (SASBP_BB_VEC4=0)."""
    rng = np.random.default_rng(Nin + Nh + Nout)
    P, E = 3, 5
    x = rng.normal(size=(P, E, Nin)).astype(np.float32)
    h = (2.0 * _lowpass((Nh - 1) // 2, 0.1)) if Nh > 1 else np.array([1.0], dtype=np.float32)
    t0 = 0.0123 + 1e-4 * np.arange(P)
    fs, fc = 480e3, 120e3 + 17.0
    got = bpmod.baseband(x, fs, fc, t0, h, 4, Nout)
    ref = oracle.baseband(x, fs, fc, t0, h, 4, Nout)
    scale = max(np.max(np.abs(ref)), 1e-30)
    assert np.max(np.abs(got - ref)) <= TOL_FILT * scale
    monkeypatch.setenv("SASBP_BB_LEGACY", "1")        # the mixed blocked kernel, float4 staging
    mx = bpmod.baseband(x, fs, fc, t0, h, 4, Nout)
    assert np.max(np.abs(mx - ref)) <= TOL_FILT * scale
    monkeypatch.setenv("SASBP_BB_VEC4", "0")          # ... and its scalar staging
    sc = bpmod.baseband(x, fs, fc, t0, h, 4, Nout)
    assert np.max(np.abs(sc - ref)) <= TOL_FILT * scale
