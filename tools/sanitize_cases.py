"""Small representative launches of every kernel and mode, for compute-sanitizer:
    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py
(racecheck / initcheck likewise).  Prints one line per case; no parity checks (the tests do that)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2101_05888_b200 as pkg  # noqa: E402


def run(name, fn):
    fn()
    torch.cuda.synchronize()
    print("ok", name, flush=True)


def tdbp(s, e, **opt):
    with pkg.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
        if opt.get("weight"):
            bp.set_weighting(True)
        if "beam" in opt:
            bp.set_beam(*opt["beam"])
        if "vel" in opt:
            bp.set_motion(opt["vel"])
        if "nav" in opt:
            bp.set_nav(*opt["nav"])
        if "medium" in opt:
            bp.set_medium(*opt["medium"])
        bp.set_pings(e, s.tx, s.rx, s.t0)
        bp.form()
        bp.count_terms()


for cid in (1, 2, 3, 4):
    s = synth.scenario(cid, reduced=(cid != 1))
    s = s.subset_pings(np.arange(min(s.P, 12)))
    e = s.echoes()
    run(f"dense cfg{cid}", lambda: tdbp(s, e))
    run(f"weighted cfg{cid}", lambda: tdbp(s, e, weight=True))
    if s.sin_half_beam > 0:
        az = 2 * float(np.arcsin(s.sin_half_beam))
        run(f"gated cfg{cid}", lambda: tdbp(s, e, beam=(az, 0.0, True, True)))
    run(f"motion cfg{cid}", lambda: tdbp(s, e, vel=np.tile([1.5, 0.2, 0.05], (s.P, 1))))
s4 = synth.scenario(4, reduced=True).subset_pings(np.arange(6))
e4 = s4.echoes()
run("refracted cfg4", lambda: tdbp(s4, e4, medium=(float(s4.grid["origin"][2]) + 0.2, 1700.0)))
os.environ["SASBP_NO_TMA"] = "1"
s2 = synth.scenario(2, reduced=True).subset_pings(np.arange(8))
e2 = s2.echoes()
run("cp.async dense cfg2", lambda: tdbp(s2, e2))
del os.environ["SASBP_NO_TMA"]
rng = np.random.default_rng(1)
x = (rng.normal(size=(3, 2, 3001)) + 1j * rng.normal(size=(3, 2, 3001))).astype(np.complex64)
rep = (rng.normal(size=600) + 1j * rng.normal(size=600)).astype(np.complex64)
run("rangecompress fft", lambda: pkg.rangecompress(x, rep))
os.environ["SASBP_RC_DIRECT"] = "1"
run("rangecompress direct", lambda: pkg.rangecompress(x, rep))
del os.environ["SASBP_RC_DIRECT"]
for U in (1, 3, 4, 8):
    run(f"upsample U={U}", lambda: pkg.upsample(x, U))
xr = rng.normal(size=(2, 3, 5000)).astype(np.float32)
h = np.hanning(65).astype(np.float32)
for D in (1, 4, 37):
    run(f"baseband D={D}", lambda: pkg.baseband(xr, 480e3, 120e3, np.array([0.01, 0.02]), h, D, 5000 // D))
os.environ["SASBP_BB_SIMPLE"] = "1"
run("baseband simple", lambda: pkg.baseband(xr, 480e3, 120e3, None, h, 4, 1250))
del os.environ["SASBP_BB_SIMPLE"]
for M in (2, 48, 64, 256):
    run(f"whitening gain M={M}", lambda: pkg.whitening_gain(x, M, 0.1))
G = pkg.whitening_gain(x, 64, 0.1)
run("whitened compression", lambda: pkg.rangecompress_whitened(x, rep, G))
# round 2: K1 bulk-staged persistent kernel (packed ragged / long records / whitened odd start lag), the legacy K1
# kernel on even Ns, K0 complex-tap kernel and its legacy mixed form, tabled receiver trajectories, two-launch gating
xe = (rng.normal(size=(7, 1, 1024)) + 1j * rng.normal(size=(7, 1, 1024))).astype(np.complex64)
rep160 = (rng.normal(size=160) + 1j * rng.normal(size=160)).astype(np.complex64)
run("rangecompress pipe packed", lambda: pkg.rangecompress(xe, rep160))
xl = (rng.normal(size=(2, 2, 3000)) + 1j * rng.normal(size=(2, 2, 3000))).astype(np.complex64)
run("rangecompress pipe long", lambda: pkg.rangecompress(xl, rep))
Gl = pkg.whitening_gain(xl, 64, 0.1)
run("whitened compression pipe (odd lag)", lambda: pkg.rangecompress_whitened(xl.reshape(4, 3000), rep, Gl))
run("whitened compression pipe packed", lambda: pkg.rangecompress_whitened(xe.reshape(7, 1024), rep160, G))
os.environ["SASBP_RC_LEGACY"] = "1"
run("rangecompress legacy even Ns", lambda: pkg.rangecompress(xl, rep))
del os.environ["SASBP_RC_LEGACY"]
xb = rng.normal(size=(2, 3, 4096)).astype(np.float32)
run("baseband ctap", lambda: pkg.baseband(xb, 480e3, 120e3, np.array([0.01, 0.02]), h, 4, 1024))
os.environ["SASBP_BB_LEGACY"] = "1"
run("baseband mixed (legacy)", lambda: pkg.baseband(xb, 480e3, 120e3, np.array([0.01, 0.02]), h, 4, 1024))
del os.environ["SASBP_BB_LEGACY"]
for cid in (1, 4):
    sn = synth.scenario(cid, reduced=(cid != 1))
    sn = sn.subset_pings(np.arange(min(sn.P, 8)))
    en = sn.echoes()
    lut, dtn = synth.nav_table(sn, K=5, accel=0.8, yaw_rate_deg=3.0, seed=cid)
    run(f"nav table cfg{cid}", lambda: tdbp(sn, en, nav=(lut, dtn)))
s2g = synth.scenario(2, reduced=True).subset_pings(np.arange(12))
e2g = s2g.echoes()
azg = 2 * float(np.arcsin(s2g.sin_half_beam))
os.environ["SASBP_GATE_TWO"] = "1"
run("gated two-launch cfg2", lambda: tdbp(s2g, e2g, beam=(azg, 0.0, True, True)))
del os.environ["SASBP_GATE_TWO"]
print("all cases ran")
# degenerate geometry: sensors on a pixel centre and on a tile centre (with receiver motion)
import oracle  # noqa: E402  (positions only: grid_points)
r = synth.random_case(21, P=2, E=2, Ns=512, n=(17, 9, 9))
g = r["grid"]
tx, rx = r["tx"].copy(), r["rx"].copy()
tx[0] = oracle.grid_points(g, np.array([[4, 4, 1]]))[0]
rx[1, 0] = oracle.grid_points(g, np.array([[2, 6, 1]]))[0]
ctr = np.asarray(g["origin"]) + 7.5 * np.asarray(g["step_x"]) + 3.5 * np.asarray(g["step_y"]) + 3.5 * np.asarray(g["step_z"])
rx[0, 1] = ctr
sd = synth.Scenario(name="degenerate", fc=r["fc"], bandwidth=r["fs"] / 4, fs=r["fs"], c=r["c"], tx=tx, rx=rx,
                    t0=np.zeros(2), Ns=512, grid=g, targets=np.zeros((0, 3)), target_pixels=np.zeros((0, 3), dtype=np.int64),
                    scat=np.zeros((0, 3)), sigma=np.zeros(0, dtype=np.complex128), sin_half_beam=0.0)
run("degenerate dense", lambda: tdbp(sd, r["echoes"]))
run("degenerate motion", lambda: tdbp(sd, r["echoes"], vel=np.tile([2.0, 0.5, 0.1], (2, 1))))
print("degenerate cases ran")
