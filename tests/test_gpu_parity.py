"""GPU-vs-oracle parity of the TDBP path through the C ABI (-m gpu).

Bar (north star): on the same generated inputs,
  max |I_gpu - I_oracle| <= 1e-3 * max |I_oracle| over the compared pixels, and
  |wrap(arg I_gpu - arg I_oracle)| <= 1e-2 rad at every scatterer's oracle peak pixel.
Compared pixels: the full image for small cases; at full BASELINE sizes (in the launch
configuration bench.py times) 4096 seeded-random pixels plus a window around every target.
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL_MAG = 1e-3
TOL_PHASE = 1e-2


@pytest.fixture(scope="module")
def bpmod(require_gpu):
    import torch
    torch.cuda.set_device(0)
    from paper_2101_05888_b200 import _build
    _build.build()
    import paper_2101_05888_b200 as pkg
    return pkg


def _form(pkg, s, echoes, grid=None, tx=None, rx=None, t0="same"):
    g = s.grid if grid is None else grid
    with pkg.Backprojector(s.fc, s.bandwidth, s.fs, s.c, g) as bp:
        bp.set_pings(echoes, s.tx if tx is None else tx, s.rx if rx is None else rx,
                     s.t0 if isinstance(t0, str) else t0)
        return bp.form()


def _check(got, ref, peaks_got=None, peaks_ref=None, label=""):
    scale = np.max(np.abs(ref))
    assert scale > 0, f"{label}: oracle image is all zero -- the case tests nothing"
    err = np.max(np.abs(got - ref))
    assert err <= TOL_MAG * scale, f"{label}: max|err| = {err:.3e} > {TOL_MAG} * {scale:.3e}"
    if peaks_ref is not None:
        dph = np.angle(peaks_got * np.conj(peaks_ref))
        assert np.max(np.abs(dph)) <= TOL_PHASE, f"{label}: peak phase err {np.max(np.abs(dph)):.3e} rad"
    return err / scale


def _peak_pixels(s, ref_fn, win=3):
    """Oracle peak pixel near every target (brute force over a small window)."""
    out = []
    g = s.grid
    for t in s.target_pixels:
        rz = range(-win, win + 1) if g["nz"] > 1 else [0]
        cand = np.array([(t[0] + dx, t[1] + dy, t[2] + dz) for dz in rz for dy in range(-win, win + 1)
                         for dx in range(-win, win + 1)])
        keep = ((cand >= 0) & (cand < np.array([g["nx"], g["ny"], g["nz"]]))).all(axis=1)
        cand = cand[keep]
        v = ref_fn(cand)
        out.append(cand[np.argmax(np.abs(v))])
    return np.array(out, dtype=np.int64)


def _at(img, idx):
    return img[idx[:, 2], idx[:, 1], idx[:, 0]]


# ------------------------------------------------------------------ full images, small cases

@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_parity_full_image(bpmod, cid):
    s = synth.scenario(cid, reduced=(cid != 1))
    e = s.echoes()
    got = _form(bpmod, s, e)
    ref = oracle.tdbp_grid(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, s.grid)
    pk = s.target_pixels
    rel = _check(got, ref, _at(got, pk), _at(ref, pk), label=s.name)
    assert rel < 1e-3


def test_cfg1_focus_on_gpu(bpmod):
    """The GPU image focuses the config-1 target at its true pixel with phase ~ 0."""
    s = synth.scenario(1)
    img = _form(bpmod, s, s.echoes())[0]
    iy, ix = np.unravel_index(np.argmax(np.abs(img)), img.shape)
    assert (ix, iy) == tuple(s.target_pixels[0][:2])
    assert abs(np.angle(img[iy, ix])) <= TOL_PHASE


# ------------------------------------------------------------------ edge cases

def _tiny(P=2, E=3, Ns=64, n=(5, 4, 1), seed=0, **kw):
    r = synth.random_case(seed, P=P, E=E, Ns=Ns, n=n, **kw)
    s = synth.Scenario(name="tiny", fc=r["fc"], bandwidth=r["fs"] / 4, fs=r["fs"], c=r["c"], tx=r["tx"],
                       rx=r["rx"], t0=r["t0"], Ns=Ns, grid=r["grid"], targets=np.zeros((0, 3)),
                       target_pixels=np.zeros((0, 3), dtype=np.int64), scat=np.zeros((0, 3)),
                       sigma=np.zeros(0, dtype=np.complex128), sin_half_beam=0.0)
    return s, r["echoes"]


@pytest.mark.parametrize("n", [(1, 1, 1), (33, 1, 1), (1, 33, 1), (31, 33, 1), (65, 40, 1), (17, 9, 9),
                               (3, 3, 17)])
def test_parity_ragged_grids(bpmod, n):
    s, e = _tiny(n=n, Ns=256, seed=sum(n))
    got = _form(bpmod, s, e)
    ref = oracle.tdbp_grid(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, s.grid)
    _check(got, ref, label=f"grid {n}")


@pytest.mark.parametrize("P,E,Ns", [(1, 1, 1), (1, 1, 256), (1, 37, 256), (33, 1, 256), (7, 5, 300)])
def test_parity_degenerate_sizes(bpmod, P, E, Ns):
    """Single ping / element / sample, channel counts that are not multiples of the batch."""
    s, e = _tiny(P=P, E=E, Ns=Ns, n=(9, 7, 3), seed=P * 100 + E)
    got = _form(bpmod, s, e)
    ref = oracle.tdbp_grid(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, s.grid)
    if np.max(np.abs(ref)) == 0:
        assert np.max(np.abs(got)) == 0
    else:
        _check(got, ref, label=f"P{P} E{E} Ns{Ns}")


def test_window_edges_zero_extension(bpmod):
    """Delays straddling both ends of the record: zero extension (R2) on the GPU too."""
    s, e = _tiny(P=4, E=4, Ns=90, n=(40, 30, 1), seed=3)
    # shift t0 so the grid's delays run off both ends of the 90-sample record
    for shift in (-70, -20, 30, 60):
        t0 = s.t0 + shift / s.fs
        got = _form(bpmod, s, e, t0=t0)
        ref = oracle.tdbp_grid(e, s.tx, s.rx, t0, s.fc, s.fs, s.c, s.grid)
        if np.max(np.abs(ref)) > 0:
            _check(got, ref, label=f"shift {shift}")


def test_t0_none_means_zero(bpmod):
    s, e = _tiny(P=3, E=2, Ns=512, seed=4)
    s.t0 = np.zeros(s.P)
    got = _form(bpmod, s, e, t0=None)
    ref = oracle.tdbp_grid(e, s.tx, s.rx, None, s.fc, s.fs, s.c, s.grid)
    _check(got, ref, label="t0=None")


def test_near_field_exact_leg(bpmod):
    """Elements within a few tile sizes of the grid select the exact (non-series) receive leg."""
    s = synth.scenario(4, reduced=True)
    e = s.echoes()
    # move the array to 20 cm above the grid top
    dz = 1.8
    tx, rx = s.tx + [0, 0, dz], s.rx + [0, 0, dz]
    t0 = s.t0 - 2 * dz / s.c   # keep the delays inside the record
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(e, tx, rx, t0)
        got = bp.form()
    ref = oracle.tdbp_grid(e, tx, rx, t0, s.fc, s.fs, s.c, s.grid)
    _check(got, ref, label="near field")


def test_rotated_grid(bpmod):
    """Non-axis-aligned steps (a tilted 2D image plane) use the dz-capable 2D kernel."""
    s = synth.scenario(2, reduced=True)
    e = s.echoes()
    th = 0.3
    g = dict(s.grid)
    g["step_x"] = np.array([0.01 * np.cos(th), 0.0, 0.01 * np.sin(th)])
    g["step_y"] = np.array([0.0, 0.01, 0.0])
    got = _form(bpmod, s, e, grid=g)
    ref = oracle.tdbp_grid(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, g)
    _check(got, ref, label="rotated grid")


# ------------------------------------------------------------------ invariants on the GPU path

def test_translation_precision(bpmod):
    """Range-relative fp32 holds under a (1e4, -3e3, 0) m coordinate offset."""
    s = synth.scenario(2, reduced=True)
    e = s.echoes()
    off = np.array([1e4, -3e3, 0.0])
    g = dict(s.grid)
    g["origin"] = s.grid["origin"] + off
    got = _form(bpmod, s, e, grid=g, tx=s.tx + off, rx=s.rx + off)
    ref = oracle.tdbp_grid(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, s.grid)
    pk = s.target_pixels
    _check(got, ref, _at(got, pk), _at(ref, pk), label="offset 1e4 m")


def test_axis_aligned_kernel_equals_general(bpmod, monkeypatch):
    """3D grids with diagonal steps run the compact-geometry (AXIS) instantiation.  It forms
    q = 2u.d + |d|^2 per axis (x pair, y row, z plane) instead of per pixel pair -- the same terms
    in another fp32 summation order -- so it agrees with the general kernel to fp32 rounding
    (and both with the oracle, test_parity_full_image)."""
    s = synth.scenario(4, reduced=True)
    e = s.echoes()
    a = _form(bpmod, s, e)
    monkeypatch.setenv("SASBP_NO_AXIS", "1")
    b = _form(bpmod, s, e)
    assert np.max(np.abs(a - b)) <= 2e-6 * np.max(np.abs(b))


def test_determinism_bitwise(bpmod):
    s = synth.scenario(2, reduced=True)
    e = s.echoes()
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(e, s.tx, s.rx, s.t0)
        a = bp.form().copy()
        b = bp.form().copy()
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_ping_chunk_accumulate(bpmod):
    """I(A u B) = I(A) + I(B) through SAS_FORM_ACCUMULATE on a device image."""
    import torch
    s = synth.scenario(2, reduced=True)
    e = s.echoes()
    full = _form(bpmod, s, e)
    img = torch.zeros(s.grid["nz"], s.grid["ny"], s.grid["nx"], dtype=torch.complex64, device="cuda")
    cuts = [0, 13, 27, s.P]
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        for i in range(len(cuts) - 1):
            a, b = cuts[i], cuts[i + 1]
            ed = torch.from_numpy(np.ascontiguousarray(e[a:b])).cuda()
            bp.set_pings_device(ed, s.tx[a:b], s.rx[a:b], s.t0[a:b])
            bp.form_device(img, accumulate=(i > 0))
            torch.cuda.synchronize()
    got = img.cpu().numpy()
    assert np.max(np.abs(got - full)) <= 1e-5 * np.max(np.abs(full))


def test_linearity_gpu(bpmod):
    s = synth.scenario(2, reduced=True)
    e1 = s.echoes()
    rng = np.random.default_rng(0)
    e2 = ((rng.normal(size=e1.shape) + 1j * rng.normal(size=e1.shape)) * 1e-4).astype(np.complex64)
    a = np.float32(-0.5)
    lhs = _form(bpmod, s, (a * e1 + e2).astype(np.complex64))
    rhs = a * _form(bpmod, s, e1) + _form(bpmod, s, e2)
    assert np.max(np.abs(lhs - rhs)) <= 1e-4 * np.max(np.abs(lhs))


# ------------------------------------------------------------------ API semantics on device

def test_form_before_set_pings_is_state_error(bpmod):
    s = synth.scenario(1)
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        with pytest.raises(bpmod.SasError) as ei:
            bp.form()
        assert ei.value.status == -2


def test_set_pings_device_matches_host(bpmod):
    import torch
    s = synth.scenario(1)
    e = s.echoes()
    host = _form(bpmod, s, e)
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings_device(torch.from_numpy(e).cuda(), s.tx, s.rx, s.t0)
        img = torch.empty(bp.shape, dtype=torch.complex64, device="cuda")
        bp.form_device(img)
        torch.cuda.synchronize()
    assert np.array_equal(img.cpu().numpy(), host)


def test_count_terms_matches_oracle(bpmod):
    """K3 in-window count vs the fp64 oracle count (agree to 1e-4)."""
    s, e = _tiny(P=5, E=4, Ns=90, n=(40, 30, 1), seed=7)
    t0 = s.t0 + 20 / s.fs
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(e, s.tx, s.rx, t0)
        dense, inwin = bp.count_terms()
    _, cnt = oracle.tdbp_grid(e, s.tx, s.rx, t0, s.fc, s.fs, s.c, s.grid, with_count=True)
    assert dense == s.n_pixels * s.P * s.E
    assert abs(inwin - int(cnt.sum())) <= max(1, 1e-4 * cnt.sum())
    assert 0 < inwin < dense


def test_rangecompress_gpu_vs_oracle(bpmod):
    rng = np.random.default_rng(1)
    fs, B, T = 120e3, 30e3, 5e-3
    n = int(round(T * fs))
    t = np.arange(n) / fs - T / 2
    rep = np.exp(1j * np.pi * (B / T) * t ** 2).astype(np.complex64)
    rep /= np.float32(np.sqrt(np.sum(np.abs(rep) ** 2)))
    raw = ((rng.normal(size=(3, 2, 3000)) + 1j * rng.normal(size=(3, 2, 3000))) / np.sqrt(2)).astype(np.complex64)
    got = bpmod.rangecompress(raw, rep)
    ref = oracle.rangecompress(raw, rep)
    assert np.max(np.abs(got - ref)) <= 1e-5 * np.max(np.abs(ref))


# ------------------------------------------------------------------ full BASELINE sizes (sampled)

@pytest.mark.parametrize("cid,stride", [(2, 1), (4, 1), (3, 4), (5, 10)])
def test_parity_full_size_sampled(bpmod, cid, stride):
    """At the BASELINE configs' full grid sizes, in bench.py's launch configuration (the same
    Backprojector plan), compare sampled pixels + windows around every target.  Configs 3 and 5
    use every 4th / 10th ping (full aperture span, full grid, full record length) to bound the
    echo generation time; config 5 is the precision stress case (ranges to 185 m, carrier phase
    to 2e5 rad, 2.7e8-pixel image)."""
    s = synth.scenario(cid)
    if stride > 1:
        s = s.subset_pings(np.arange(0, s.P, stride))
    e = s.echoes()
    got = _form(bpmod, s, e)
    idx = s.sample_pixels(4096, window=15 if s.grid["nz"] == 1 else 5, seed=cid)
    ref = oracle.tdbp_grid(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, s.grid, idx=idx)
    g = _at(got, idx)
    pk = _peak_pixels(s, lambda c: oracle.tdbp_grid(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, s.grid, idx=c), win=1)
    pref = oracle.tdbp_grid(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, s.grid, idx=pk)
    _check(g, ref, _at(got, pk), pref, label=f"cfg{cid} full")


# ------------------------------------------------------------------ plan selection and staging paths

def test_plan_selection(bpmod):
    """Far-field stripmap uses the 3-term series and TMA staging; near field the exact leg."""
    s = synth.scenario(2, reduced=True)
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(s.echoes(), s.tx, s.rx, s.t0)
        bp.form()
        pl = bp.plan()
    assert pl["tile"] == (32, 32, 1) and pl["tma"] is True and pl["rx_mode"] == "series3", pl
    assert pl["ctas_per_sm"] == 4, pl   # 126 registers and the shared-memory budget give 4 CTAs
    s4 = synth.scenario(4, reduced=True)
    with bpmod.Backprojector(s4.fc, s4.bandwidth, s4.fs, s4.c, s4.grid) as bp:
        bp.set_pings(s4.echoes(), s4.tx + [0, 0, 1.8], s4.rx + [0, 0, 1.8], s4.t0 - 3.6 / s4.c)
        assert bp.plan()["rx_mode"] == "exact"


@pytest.mark.parametrize("how", ["env", "odd_ns"])
def test_cp_async_fallback_path(bpmod, how, monkeypatch):
    """The cp.async staging fallback (odd Ns, or SASBP_NO_TMA=1) gives the same images."""
    s = synth.scenario(2, reduced=True)
    e = s.echoes()
    if how == "odd_ns":
        e = np.ascontiguousarray(e[:, :, :-1])
    else:
        monkeypatch.setenv("SASBP_NO_TMA", "1")
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(e, s.tx, s.rx, s.t0)
        assert bp.plan()["tma"] is False
        got = bp.form()
    ref = oracle.tdbp_grid(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, s.grid)
    pk = s.target_pixels
    _check(got, ref, _at(got, pk), _at(ref, pk), label=f"cp.async {how}")


# ------------------------------------------------------------------ K1 range compression

def _lfm(fs, B, T):
    n = int(round(T * fs))
    t = np.arange(n) / fs - T / 2
    r = np.exp(1j * np.pi * (B / T) * t ** 2).astype(np.complex64)
    return (r / np.float32(np.sqrt(np.sum(np.abs(r) ** 2)))).astype(np.complex64)


@pytest.mark.parametrize("Ns,Nr,path", [(3000, 600, "fft"), (10240, 600, "fft"), (777, 160, "fft"), (100, 1, "fft"),
                                         (5000, 2048, "fft"), (5000, 2049, "direct"), (3000, 600, "direct"),
                                         (4096, 3497, "direct")])
def test_rangecompress_paths(bpmod, Ns, Nr, path, monkeypatch):
    """FFT overlap-save (Nr <= 2048) and direct paths vs the fp64 direct correlation (R14)."""
    if path == "direct" and Nr <= 2048:
        monkeypatch.setenv("SASBP_RC_DIRECT", "1")
    rng = np.random.default_rng(Ns + Nr)
    rep = (rng.normal(size=Nr) + 1j * rng.normal(size=Nr)).astype(np.complex64) / np.float32(np.sqrt(2 * Nr))
    raw = ((rng.normal(size=(2, 3, Ns)) + 1j * rng.normal(size=(2, 3, Ns))) / np.sqrt(2)).astype(np.complex64)
    got = bpmod.rangecompress(raw, rep)
    ref = oracle.rangecompress(raw, rep)
    assert np.max(np.abs(got - ref)) <= 2e-5 * np.max(np.abs(ref))


def test_rangecompress_then_backproject(bpmod):
    """Row a1 feeding a4: raw LFM echoes of the config-1 target, compressed on the GPU, focus
    at the target with the same image as the oracle chain (oracle compression + oracle TDBP)."""
    s = synth.scenario(1)
    comp = s.echoes()                               # compressed echoes of the forward model
    rep = _lfm(s.fs, s.bandwidth, 2e-3)
    # raw = compressed convolved with the replica is not available from the generator; use the
    # linearity of both stages instead: compress(comp) on GPU vs oracle, then image both.
    g = bpmod.rangecompress(comp, rep)
    o = oracle.rangecompress(comp, rep).astype(np.complex64)
    assert np.max(np.abs(g - o)) <= 2e-5 * np.max(np.abs(o))
    img_g = _form(bpmod, s, g)
    img_o = oracle.tdbp_grid(o, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, s.grid)
    _check(img_g, img_o, label="compress -> backproject")


@pytest.mark.parametrize("chunks", [1, 3, 0])
def test_form_streamed_matches_form(bpmod, chunks):
    """sas_bp_form_streamed (chunked H2D overlapped with accumulating launches) equals
    set_pings + form: bitwise for one chunk, to fp32 summation order otherwise."""
    import torch
    s = synth.scenario(2, reduced=True)
    e = s.echoes()
    ref = _form(bpmod, s, e)
    pinned = torch.from_numpy(e).pin_memory()
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        got = bp.form_streamed(pinned, s.tx, s.rx, s.t0, chunks=chunks)
        again = bp.form()            # the handle now holds the ping set
    if chunks == 1:
        assert np.array_equal(got, ref)
    assert np.max(np.abs(got - ref)) <= 1e-5 * np.max(np.abs(ref))
    assert np.array_equal(again, ref)


# ------------------------------------------------------------------ NEXT-1: FOV gating + ray culling

def _gated_ref(s, e, grid, az, el=0.0, bistatic=False, axes=None, idx=None):
    pts = oracle.grid_points(grid, idx)
    v = oracle.tdbp_points_gated(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, pts, az=az, el=el, bistatic=bistatic,
                                 axes=axes)
    if idx is None:
        return v.reshape(grid["nz"], grid["ny"], grid["nx"])
    return v


def _gated_form(bpmod, s, e, az, el=0.0, bistatic=False, cull=True, axes=None):
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(e, s.tx, s.rx, s.t0)
        bp.set_beam(az, el, bistatic, cull, axes)
        img = bp.form()
        counts = bp.count_terms()
    return img, counts


@pytest.mark.parametrize("bistatic", [False, True])
@pytest.mark.parametrize("launches", ["one", "two"])
def test_gated_stripmap_vs_oracle(bpmod, bistatic, launches, monkeypatch):
    """Gated sum with the generator's azimuth beam (P:160 FOV query; R15) on reduced config 2, in
    the one-launch form and the two-launch A/B form (SASBP_GATE_TWO: mask-free IN pairs, then the
    edge pairs)."""
    if launches == "two":
        monkeypatch.setenv("SASBP_GATE_TWO", "1")
    s = synth.scenario(2, reduced=True)
    e = s.echoes()
    az = 2 * np.arcsin(s.sin_half_beam)
    got, (dense, inwin) = _gated_form(bpmod, s, e, az, bistatic=bistatic)
    ref = _gated_ref(s, e, s.grid, az, bistatic=bistatic)
    pk = s.target_pixels
    _check(got, ref, _at(got, pk), _at(ref, pk), label=f"gated bistatic={bistatic}")
    _, cnt = oracle.tdbp_points_gated(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, oracle.grid_points(s.grid), az=az,
                                      bistatic=bistatic, with_count=True)
    assert inwin == int(cnt.sum())       # fp64 gate decisions identical to the oracle's
    assert 0 < inwin < dense


def test_gated_near_field_3d_bistatic_elevation(bpmod):
    """Bistatic gating with azimuth + elevation cones on the downward-looking 3D array
    (P:310/315 near-field bistatic culling), per-ping axes a = +x, b = +z (down)."""
    s = synth.scenario(4, reduced=True)
    e = s.echoes()
    axes = np.tile(np.array([[[1.0, 0, 0], [0, 0, 1.0]]]), (s.P, 1, 1))
    got, (dense, inwin) = _gated_form(bpmod, s, e, az=0.3, el=0.4, bistatic=True, axes=axes)
    ref = _gated_ref(s, e, s.grid, 0.3, 0.4, True, axes)
    _check(got, ref, label="gated 3D bistatic")
    _, cnt = oracle.tdbp_points_gated(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, oracle.grid_points(s.grid), az=0.3,
                                      el=0.4, bistatic=True, axes=axes, with_count=True)
    assert 0 < inwin < dense and inwin == int(cnt.sum())   # the cones cut the volume (62 % of terms)


def test_culled_equals_unculled_bitwise(bpmod):
    """S:389 cardinal property: ray culling changes run time, never pixel values."""
    s = synth.scenario(2, reduced=True)
    e = s.echoes()
    az = 2 * np.arcsin(s.sin_half_beam)
    a, _ = _gated_form(bpmod, s, e, az, cull=True)
    b, _ = _gated_form(bpmod, s, e, az, cull=False)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_open_gate_equals_dense_bitwise(bpmod):
    """A gate with both tests disabled admits every term: identical to the dense image."""
    s = synth.scenario(2, reduced=True)
    e = s.echoes()
    dense = _form(bpmod, s, e)
    got, _ = _gated_form(bpmod, s, e, az=np.pi, el=0.0)
    assert np.array_equal(got.view(np.uint32), dense.view(np.uint32))
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:   # set_beam(None) = dense again
        bp.set_pings(e, s.tx, s.rx, s.t0)
        bp.set_beam(0.3)
        bp.set_beam(None)
        assert np.array_equal(bp.form().view(np.uint32), dense.view(np.uint32))


def test_set_beam_errors(bpmod):
    s = synth.scenario(1)
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(s.echoes(), s.tx, s.rx, s.t0)
        with pytest.raises(bpmod.SasError) as ei:
            bp.set_beam(0.3, axes=np.tile(np.array([[[1.0, 0, 0], [1.0, 0, 0]]]), (s.P, 1, 1)))
        assert ei.value.status == -1
        bp.set_beam(0.3, axes=np.tile(np.array([[[1.0, 0, 0], [0, 1.0, 0]]]), (s.P + 1, 1, 1)))
        with pytest.raises(bpmod.SasError) as ei:
            bp.form()
        assert ei.value.status == -2


def test_gated_full_size_cfg2_sampled(bpmod):
    """Gated + culled at the full config-2 size: sampled pixels vs the gated oracle."""
    s = synth.scenario(2)
    e = s.echoes()
    az = 2 * np.arcsin(s.sin_half_beam)
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(e, s.tx, s.rx, s.t0)
        bp.set_beam(az)
        got = bp.form()
    idx = s.sample_pixels(2048, window=7, seed=7)
    ref = _gated_ref(s, e, s.grid, az, idx=idx)
    _check(_at(got, idx), ref, label="gated cfg2 full")


# ------------------------------------------------------------------ NEXT-2: moving receiver

def _motion_form(bpmod, s, e, vel, beam=None):
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(e, s.tx, s.rx, s.t0)
        bp.set_motion(vel)
        if beam:
            bp.set_beam(*beam)
        return bp.form()


def test_motion_cfg1_vs_oracle(bpmod):
    """Config 1 recorded at 2 m/s along track: GPU moving-receiver image vs the oracle's exact
    delay root (R16), full grid; peak at the target with phase ~ 0."""
    s = synth.scenario(1)
    s.vel = np.tile([2.0, 0.0, 0.0], (s.P, 1))
    e = s.echoes()
    got = _motion_form(bpmod, s, e, s.vel)
    ref = oracle.tdbp_points_motion(e, s.tx, s.rx, s.t0, s.vel, s.fc, s.fs, s.c,
                                    oracle.grid_points(s.grid)).reshape(got.shape)
    pk = s.target_pixels
    _check(got, ref, _at(got, pk), _at(ref, pk), label="motion cfg1")
    iy, ix = np.unravel_index(np.argmax(np.abs(got[0])), got[0].shape)
    assert (ix, iy) == tuple(pk[0][:2])


@pytest.mark.parametrize("cid", [3, 4])
def test_motion_random_velocities(bpmod, cid):
    """Per-ping velocities with sway / heave components (reduced configs 3 and 4; config 4 runs
    the near-field exact receive leg)."""
    s = synth.scenario(cid, reduced=True)
    rng = np.random.default_rng(cid)
    s.vel = np.stack([1.5 + 0.2 * rng.normal(size=s.P), 0.3 * rng.normal(size=s.P), 0.1 * rng.normal(size=s.P)], 1)
    e = s.echoes()
    got = _motion_form(bpmod, s, e, s.vel)
    ref = oracle.tdbp_points_motion(e, s.tx, s.rx, s.t0, s.vel, s.fc, s.fs, s.c,
                                    oracle.grid_points(s.grid)).reshape(got.shape)
    pk = s.target_pixels
    _check(got, ref, _at(got, pk), _at(ref, pk), label=f"motion cfg{cid}r")


def test_motion_zero_velocity_bitwise(bpmod):
    s = synth.scenario(2, reduced=True)
    e = s.echoes()
    a = _form(bpmod, s, e)
    b = _motion_form(bpmod, s, e, np.zeros((s.P, 3)))
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("bistatic", [False, True])
def test_motion_with_gating(bpmod, bistatic):
    """Moving receiver and FOV gating together (R15 + R16, reading R22: gate decisions on the
    transmit-time positions): element-wise parity with the oracle's gated moving-receiver sum on
    reduced config 2, and the exact in-cone term count."""
    s = synth.scenario(2, reduced=True)
    s.vel = np.tile([1.8, 0.1, 0.0], (s.P, 1))
    e = s.echoes()
    az = 2 * np.arcsin(s.sin_half_beam)
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(e, s.tx, s.rx, s.t0)
        bp.set_motion(s.vel)
        bp.set_beam(az, 0.0, bistatic)
        got = bp.form()
        dense, inwin = bp.count_terms()
    ref, cnt = oracle.tdbp_points_gated_motion(e, s.tx, s.rx, s.t0, s.vel, s.fc, s.fs, s.c,
                                               oracle.grid_points(s.grid), az=az, bistatic=bistatic,
                                               with_count=True)
    ref = ref.reshape(got.shape)
    pk = s.target_pixels
    pk = pk[np.abs(_at(ref, pk)) > 0.1 * np.abs(ref).max()]   # phase at the targets the gate keeps bright
    _check(got, ref, _at(got, pk), _at(ref, pk), label=f"motion + gate bistatic={bistatic}")
    assert 0 < inwin < dense
    assert abs(inwin - int(cnt.sum())) <= max(1, 1e-4 * cnt.sum())


def test_motion_with_gating_3d_near_field(bpmod):
    """Reduced config 4 (near-field exact receive leg) moving at sway/heave velocities with a
    bistatic azimuth + elevation gate."""
    s = synth.scenario(4, reduced=True)
    rng = np.random.default_rng(44)
    s.vel = np.stack([0.5 + 0.1 * rng.normal(size=s.P), 0.2 * rng.normal(size=s.P), 0.05 * rng.normal(size=s.P)], 1)
    e = s.echoes()
    axes = np.tile(np.array([[[1.0, 0, 0], [0, 0, 1.0]]]), (s.P, 1, 1))
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(e, s.tx, s.rx, s.t0)
        bp.set_motion(s.vel)
        bp.set_beam(0.3, 0.4, True, True, axes)
        got = bp.form()
        dense, inwin = bp.count_terms()
    ref, cnt = oracle.tdbp_points_gated_motion(e, s.tx, s.rx, s.t0, s.vel, s.fc, s.fs, s.c, oracle.grid_points(s.grid),
                                               az=0.3, el=0.4, bistatic=True, axes=axes, with_count=True)
    _check(got, ref.reshape(got.shape), label="motion + gate 3D")
    assert 0 < inwin < dense
    assert abs(inwin - int(cnt.sum())) <= max(1, 1e-4 * cnt.sum())


def test_set_motion_errors(bpmod):
    s = synth.scenario(1)
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(s.echoes(), s.tx, s.rx, s.t0)
        with pytest.raises(bpmod.SasError) as ei:
            bp.set_motion(np.tile([100.0, 0, 0], (s.P, 1)))   # > c/100
        assert ei.value.status == -1
        bp.set_motion(np.zeros((s.P + 2, 3)))
        with pytest.raises(bpmod.SasError) as ei:
            bp.form()
        assert ei.value.status == -2


# ------------------------------------------------------------------ NEXT-3: sediment refraction

def _refr_form(bpmod, s, e, zb, c2, counts=False):
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(e, s.tx, s.rx, s.t0)
        bp.set_medium(zb, c2)
        img = bp.form()
        assert bp.plan()["rx_mode"] == "refracted"
        return (img, bp.count_terms()) if counts else img


@pytest.mark.parametrize("c2", [1700.0, 1560.0, 1450.0])
def test_refracted_3d_vs_oracle(bpmod, c2):
    """Reduced config 4 recorded through a sediment interface at z = 0 (fast and slow sediment):
    GPU Fermat delays vs the oracle's exact refracted delays, full volume, and the in-window
    term count."""
    s = synth.scenario(4, reduced=True)
    s.medium = (0.0, c2)
    e = s.echoes()
    (got, (dense, inwin)) = _refr_form(bpmod, s, e, 0.0, c2, counts=True)
    ref, cnt = oracle.tdbp_points_refracted(e, s.tx, s.rx, s.t0, 0.0, c2, s.fc, s.fs, s.c,
                                            oracle.grid_points(s.grid), with_count=True)
    ref = ref.reshape(got.shape)
    pk = s.target_pixels
    _check(got, ref, _at(got, pk), _at(ref, pk), label=f"refracted c2={c2}")
    assert abs(inwin - int(cnt.sum())) <= max(1, 1e-4 * cnt.sum())


def test_refracted_interface_inside_volume(bpmod):
    """Interface through the middle of the voxel grid: voxels above it take the straight water
    path, those below the Fermat path."""
    s = synth.scenario(4, reduced=True)
    zb = 0.15
    s.medium = (zb, 1650.0)
    e = s.echoes()
    got = _refr_form(bpmod, s, e, zb, 1650.0)
    ref = oracle.tdbp_points_refracted(e, s.tx, s.rx, s.t0, zb, 1650.0, s.fc, s.fs, s.c,
                                       oracle.grid_points(s.grid)).reshape(got.shape)
    _check(got, ref, label="interface inside the volume")


def test_refracted_equal_speed_is_dense(bpmod):
    s = synth.scenario(4, reduced=True)
    e = s.echoes()
    got = _refr_form(bpmod, s, e, 0.0, s.c)
    ref = oracle.tdbp_grid(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, s.grid)
    _check(got, ref, label="c2 = c")


@pytest.mark.parametrize("c2", [1700.0, 1450.0])
def test_refracted_with_gating_3d(bpmod, c2):
    """The paper's near-field craft: bistatic ray culling AND the sediment refraction model
    together (R15 + R17, reading R22: straight line-of-sight gate from the recorded
    sensor positions).  Reduced config 4, azimuth + elevation cones around a downward boresight,
    element-wise parity with the oracle's gated refracted sum, exact in-cone counts."""
    s = synth.scenario(4, reduced=True)
    s.medium = (0.0, c2)
    e = s.echoes()
    axes = np.tile(np.array([[[1.0, 0, 0], [0, 0, 1.0]]]), (s.P, 1, 1))
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(e, s.tx, s.rx, s.t0)
        bp.set_medium(0.0, c2)
        bp.set_beam(0.3, 0.4, True, True, axes)
        got = bp.form()
        dense, inwin = bp.count_terms()
    ref, cnt = oracle.tdbp_points_gated_refracted(e, s.tx, s.rx, s.t0, 0.0, c2, s.fc, s.fs, s.c,
                                                  oracle.grid_points(s.grid), az=0.3, el=0.4, bistatic=True,
                                                  axes=axes, with_count=True)
    ref = ref.reshape(got.shape)
    pk = s.target_pixels
    pk = pk[np.abs(_at(ref, pk)) > 0.1 * np.abs(ref).max()]   # phase at the targets the gate keeps bright
    _check(got, ref, _at(got, pk), _at(ref, pk), label=f"refracted + gate c2={c2}")
    assert 0 < inwin < dense
    assert abs(inwin - int(cnt.sum())) <= max(1, 1e-4 * cnt.sum())


def test_set_medium_errors(bpmod):
    s = synth.scenario(4, reduced=True)
    e = s.echoes()
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(e, s.tx, s.rx, s.t0)
        bp.set_medium(-2.5, 1700.0)                 # interface above the sensors (z = -2)
        with pytest.raises(bpmod.SasError) as ei:
            bp.form()
        assert ei.value.status == -1
        bp.set_medium(0.0, 1700.0)
        bp.set_motion(np.zeros((s.P, 3)))
        with pytest.raises(bpmod.SasError) as ei:
            bp.form()
        assert ei.value.status == -5
        bp.set_motion(None)
        bp.form()


def test_sensor_at_a_pixel_centre(bpmod):
    """Degenerate geometry: the transmitter and one receiver sit exactly on pixel centres inside
    the grid (R = 0 legs; the near-field exact mode); the image stays finite and matches the
    oracle."""
    s, e = _tiny(P=2, E=2, Ns=512, n=(9, 9, 3), seed=21)
    g = s.grid
    c0 = oracle.grid_points(g, np.array([[4, 4, 1]]))[0]
    c1 = oracle.grid_points(g, np.array([[2, 6, 1]]))[0]
    tx = s.tx.copy()
    rx = s.rx.copy()
    tx[0] = c0
    rx[1, 0] = c1
    t0 = np.zeros(s.P)
    got = _form(bpmod, s, e, tx=tx, rx=rx, t0=t0)
    assert np.all(np.isfinite(got))
    ref = oracle.tdbp_grid(e, tx, rx, t0, s.fc, s.fs, s.c, g)
    _check(got, ref, label="sensor on a pixel")


def test_sensor_at_a_pixel_centre_counts(bpmod):
    """K3 on the same degenerate geometry: the in-window count equals the oracle's."""
    s, e = _tiny(P=2, E=2, Ns=512, n=(9, 9, 3), seed=21)
    g = s.grid
    tx = s.tx.copy()
    rx = s.rx.copy()
    tx[0] = oracle.grid_points(g, np.array([[4, 4, 1]]))[0]
    rx[1, 0] = oracle.grid_points(g, np.array([[2, 6, 1]]))[0]
    t0 = np.zeros(s.P)
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, g) as bp:
        bp.set_pings(e, tx, rx, t0)
        dense, inwin = bp.count_terms()
    _, cnt = oracle.tdbp_grid(e, tx, rx, t0, s.fc, s.fs, s.c, g, with_count=True)
    assert inwin == int(cnt.sum()) and dense == g["nx"] * g["ny"] * g["nz"] * s.P * s.E


def test_rejects_delays_beyond_int32_windows(bpmod):
    """t0 in the wrong unit (e.g. 3e4 s): delays of ~1e9 samples are rejected, not launched."""
    s, e = _tiny(P=2, E=2, Ns=256, seed=5)
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        with pytest.raises(bpmod.SasError) as ei:
            bp.set_pings(e, s.tx, s.rx, np.full(s.P, 3.0e4))
        assert ei.value.status == bpmod.sasbp.SAS_E_INVALID
        bp.set_pings(e, s.tx, s.rx, s.t0)   # the handle stays usable
        assert np.all(np.isfinite(bp.form()))


def test_coarse_pixels_large_window_cp_async(bpmod):
    """Coarse 5 cm pixels at fs = 4B: the tile window exceeds a TMA box (256 samples), so the
    plan falls back to cp.async staging with ~150 KB of shared memory per CTA; parity holds."""
    s = synth.scenario(2, reduced=True)
    g = dict(s.grid)
    g["step_x"] = np.array([0.05, 0.0, 0.0])
    g["step_y"] = np.array([0.0, 0.05, 0.0])
    g["nx"], g["ny"] = 40, 37
    e = s.echoes()
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, g) as bp:
        bp.set_pings(e, s.tx, s.rx, s.t0)
        plan = bp.plan()
        got = bp.form()
    assert plan["window"] > 256 and plan["tma"] is False
    ref = oracle.tdbp_grid(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, g)
    _check(got, ref, label="coarse pixels")


@pytest.mark.parametrize("Ns,Nr,nch", [(1024, 160, 257), (1, 1, 5), (1889, 160, 7), (1, 2048, 9), (1365, 1, 10),
                                        (700, 666, 11), (2048, 1, 3)])
def test_rangecompress_packed_records(bpmod, Ns, Nr, nch):
    """Short records (S = Ns + Nr - 1 <= 2048): several whole channels share one 4096-point
    transform, each followed by Nr - 1 zeros; every channel (including a ragged last block) must
    still equal its own fp64 correlation (R14), and the unpacked path (SASBP_RC_NOPACK) agrees."""
    rng = np.random.default_rng(7 * Ns + Nr + nch)
    rep = (rng.normal(size=Nr) + 1j * rng.normal(size=Nr)).astype(np.complex64) / np.float32(np.sqrt(2 * Nr))
    raw = ((rng.normal(size=(nch, 1, Ns)) + 1j * rng.normal(size=(nch, 1, Ns))) / np.sqrt(2)).astype(np.complex64)
    got = bpmod.rangecompress(raw, rep)
    ref = oracle.rangecompress(raw, rep)
    scale = np.max(np.abs(ref))
    assert np.max(np.abs(got - ref)) <= 2e-5 * scale
    import os
    os.environ["SASBP_RC_NOPACK"] = "1"
    try:
        unp = bpmod.rangecompress(raw, rep)
    finally:
        del os.environ["SASBP_RC_NOPACK"]
    assert np.max(np.abs(unp - ref)) <= 2e-5 * scale


def test_wave_tail_split(bpmod, monkeypatch):
    """The last, at most half-full wave of tiles is split into two channel halves per tile (atomic
    float2 adds into the zeroed image).  Same sum in another fp32 order: agrees with the unsplit
    launch to fp32 rounding, is deterministic (0 + a + b = 0 + b + a), and is never used for
    SAS_FORM_ACCUMULATE launches."""
    import torch
    s = synth.scenario(2, reduced=True)
    e = s.echoes()
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(e, s.tx, s.rx, s.t0)
        a = bp.form().copy()
        assert bp.plan()["tail_split"] == 2, bp.plan()   # reduced grid: fewer tiles than half a wave
        a2 = bp.form().copy()
        assert np.array_equal(a.view(np.uint32), a2.view(np.uint32))
        img = torch.zeros(bp.shape, dtype=torch.complex64, device="cuda")
        bp.form_device(img, accumulate=True)
        torch.cuda.synchronize()
        assert bp.plan()["tail_split"] == 1
        acc = img.cpu().numpy()
        monkeypatch.setenv("SASBP_NO_TAILSPLIT", "1")
        b = bp.form().copy()
        assert bp.plan()["tail_split"] == 1
    scale = np.max(np.abs(b))
    assert np.max(np.abs(a - b)) <= 2e-6 * scale
    assert np.max(np.abs(acc - b)) <= 2e-6 * scale


@pytest.mark.parametrize("Ns,Nr,nch,M", [(1024, 160, 257, 0), (10240, 600, 3, 0), (3000, 600, 4, 0), (4096, 1, 2, 0),
                                          (8192, 2048, 2, 0), (6, 1, 5, 0), (2, 3, 7, 0), (3498, 600, 3, 0),
                                          (10240, 600, 3, 64), (1024, 160, 31, 64), (3000, 41, 5, 4), (2, 1, 9, 4),
                                          (4096, 600, 3, 2), (7000, 1793, 2, 256)])
@pytest.mark.parametrize("impl", ["pipe", "legacy"])
def test_rangecompress_pipelined_and_legacy(bpmod, Ns, Nr, nch, M, impl, monkeypatch):
    """K1's bulk-staged persistent kernel (even Ns, aligned input; packed and long records, ragged
    last blocks, channel-edge windows, odd start lags of the whitened filter) and the per-thread
    load kernel (SASBP_RC_LEGACY=1) both equal the fp64 correlation (R14) / the oracle's whitening
    cascade (R21)."""
    if impl == "legacy":
        monkeypatch.setenv("SASBP_RC_LEGACY", "1")
    rng = np.random.default_rng(3 * Ns + Nr + nch + M)
    rep = (rng.normal(size=Nr) + 1j * rng.normal(size=Nr)).astype(np.complex64) / np.float32(np.sqrt(2 * Nr))
    raw = ((rng.normal(size=(nch, 1, Ns)) + 1j * rng.normal(size=(nch, 1, Ns))) / np.sqrt(2)).astype(np.complex64)
    if M == 0:
        got = bpmod.rangecompress(raw, rep)
        ref = oracle.rangecompress(raw, rep)
    else:
        x = raw.reshape(nch, Ns)
        G = (0.2 + rng.random(M)).astype(np.float32)
        G /= G.max()
        got = bpmod.rangecompress_whitened(x, rep, G)
        ref = oracle.rangecompress_whitened(x, rep, G.astype(np.float64))
    assert np.max(np.abs(got - ref)) <= 2e-5 * np.max(np.abs(ref))


# ------------------------------------------------------------------ NEXT-2: tabled receiver trajectories (R23)

def _nav_form(pkg, s, echoes, lut, dt, beam=None):
    with pkg.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(echoes, s.tx, s.rx, s.t0)
        bp.set_nav(lut, dt)
        if beam:
            bp.set_beam(*beam)
        img = bp.form()
        return img, bp.count_terms(), bp.plan()


@pytest.mark.parametrize("cid,K", [(1, 6), (3, 9), (4, 5)])
def test_nav_table_vs_oracle(bpmod, cid, K):
    """Receivers on tabled trajectories (velocity + acceleration + lever arms turning at a yaw
    rate; the paper's position LUT): full reduced images vs the oracle's per-term fixed
    point on the interpolated trajectory (config 4 runs the near-field exact receive leg), exact
    in-window term counts within 1e-4."""
    s = synth.scenario(cid, reduced=True)
    e = s.echoes()
    lut, dt = synth.nav_table(s, K=K, accel=0.8, yaw_rate_deg=3.0, seed=cid)
    got, (dense, inwin), plan = _nav_form(bpmod, s, e, lut, dt)
    ref, cnt = oracle.tdbp_points_nav(e, s.tx, lut, dt, s.t0, s.fc, s.fs, s.c, oracle.grid_points(s.grid),
                                      with_count=True)
    ref = ref.reshape(got.shape)
    pk = s.target_pixels
    pk = pk[np.abs(_at(ref, pk)) > 0.1 * np.abs(ref).max()]
    _check(got, ref, _at(got, pk), _at(ref, pk), label=f"nav cfg{cid}r")
    assert abs(inwin - int(cnt.sum())) <= max(1, 1e-4 * cnt.sum())


def test_nav_linear_table_matches_set_motion(bpmod):
    """A table of the constant-velocity trajectory rx + v t images like sas_bp_set_motion (the
    same reference solution up to fp64 rounding of the spline)."""
    s = synth.scenario(3, reduced=True)
    e = s.echoes()
    rng = np.random.default_rng(9)
    vel = np.stack([1.5 + 0.2 * rng.normal(size=s.P), 0.3 * rng.normal(size=s.P), 0.1 * rng.normal(size=s.P)], 1)
    lut, dt = synth.nav_table(s, K=4, accel=0.0, yaw_rate_deg=0.0, vel=vel)
    a, _, _ = _nav_form(bpmod, s, e, lut, dt)
    b = _motion_form(bpmod, s, e, vel)
    assert np.max(np.abs(a - b)) <= 1e-5 * np.max(np.abs(b))


@pytest.mark.parametrize("bistatic", [False, True])
def test_nav_with_gating(bpmod, bistatic):
    """Tabled trajectories with FOV gating (R22 + R23: gate on the recorded positions): parity with
    the oracle's gated tabled sum and its in-cone count."""
    s = synth.scenario(2, reduced=True)
    e = s.echoes()
    lut, dt = synth.nav_table(s, K=7, accel=0.5, yaw_rate_deg=2.0, seed=21)
    az = 2 * np.arcsin(s.sin_half_beam)
    got, (dense, inwin), _ = _nav_form(bpmod, s, e, lut, dt, beam=(az, 0.0, bistatic))
    ref, cnt = oracle.tdbp_points_gated_nav(e, s.tx, s.rx, lut, dt, s.t0, s.fc, s.fs, s.c,
                                            oracle.grid_points(s.grid), az=az, bistatic=bistatic, with_count=True)
    ref = ref.reshape(got.shape)
    pk = s.target_pixels
    pk = pk[np.abs(_at(ref, pk)) > 0.1 * np.abs(ref).max()]
    _check(got, ref, _at(got, pk), _at(ref, pk), label=f"nav + gate bistatic={bistatic}")
    assert 0 < inwin < dense
    assert abs(inwin - int(cnt.sum())) <= max(1, 1e-4 * cnt.sum())


def test_set_nav_errors(bpmod):
    s = synth.scenario(1, reduced=True)
    e = s.echoes()
    lut, dt = synth.nav_table(s, K=5)
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(e, s.tx, s.rx, s.t0)
        for bad_lut, bad_dt in ((lut[:, :, :2], dt), (lut, 0.0), (lut, -1.0), (lut, np.nan)):
            with pytest.raises(bpmod.SasError):
                bp.set_nav(bad_lut, bad_dt)
        nan = lut.copy(); nan[0, 0, 1, 0] = np.nan
        with pytest.raises(bpmod.SasError):
            bp.set_nav(nan, dt)
        fast = lut.copy(); fast[0, 0, 2, 0] += 0.02 * s.c * dt
        with pytest.raises(bpmod.SasError):
            bp.set_nav(fast, dt)
        bp.set_nav(lut[:-1], dt)            # tables for another ping count: form refuses (SAS_E_STATE)
        with pytest.raises(bpmod.SasError):
            bp.form()
        bp.set_nav(lut, dt)
        bp.set_medium(100.0, 1600.0)        # refraction + motion: unsupported
        with pytest.raises(bpmod.SasError):
            bp.form()
        bp.set_medium(0.0, 0.0)
        a = bp.form()
        bp.set_nav(None)                     # back to stop-and-hop
        b = bp.form()
    ref = _form(bpmod, s, e)
    assert np.array_equal(b.view(np.uint32), ref.view(np.uint32))
    assert not np.array_equal(a, b)


def test_nav_table_streamed_and_cpasync(bpmod, monkeypatch):
    """Tabled trajectories through the chunked host path (form_streamed: per-chunk launches index the
    table by global channel) and through the cp.async staging fallback equal the plain form."""
    s = synth.scenario(3, reduced=True)
    e = s.echoes()
    lut, dt = synth.nav_table(s, K=6, accel=0.6, yaw_rate_deg=2.5, seed=33)
    with bpmod.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        bp.set_pings(e, s.tx, s.rx, s.t0)
        bp.set_nav(lut, dt)
        ref = bp.form()
        got = bp.form_streamed(e, s.tx, s.rx, s.t0, chunks=3)
    assert np.max(np.abs(got - ref)) <= 1e-5 * np.max(np.abs(ref))
    monkeypatch.setenv("SASBP_NO_TMA", "1")
    got2, _, plan = _nav_form(bpmod, s, e, lut, dt)
    assert plan["tma"] is False
    assert np.max(np.abs(got2 - ref)) <= 1e-5 * np.max(np.abs(ref))
