"""Device-resident K2 timing on every BASELINE config at full size (timing only: the echoes are
seeded device-random complex64 of the config's shape -- the TDBP work is data independent;
parity at these sizes is tests/test_gpu_parity.py's job).  One JSON line per config.
    python tools/bench_configs.py [--configs 2 3 4 5] [--steps 2] [--gated]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2101_05888_b200 as pkg  # noqa: E402


def roof(E, sms=148, f=1.965e9):
    F, S = 20 + 6 / E, 3 + 1 / E
    return sms * f * min(128 / F, 16 / S)


ap = argparse.ArgumentParser()
ap.add_argument("--configs", type=int, nargs="+", default=[2, 3, 4, 5])
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--gated", action="store_true")
a = ap.parse_args()
torch.cuda.set_device(0)
for cid in a.configs:
    s = synth.scenario(cid)
    g = s.grid
    P, E, Ns = s.P, s.E, s.Ns
    gen = torch.Generator(device="cuda").manual_seed(1000 + cid)
    e = torch.randn((P, E, Ns), dtype=torch.complex64, device="cuda", generator=gen)
    bp = pkg.Backprojector(s.fc, s.bandwidth, s.fs, s.c, g)
    bp.set_pings_device(e, s.tx, s.rx, s.t0)
    dense, inwin = bp.count_terms()
    img = torch.empty(bp.shape, dtype=torch.complex64, device="cuda")
    res = {}
    for mode in (["dense", "gated"] if a.gated and s.sin_half_beam > 0 else ["dense"]):
        if mode == "gated":
            bp.set_beam(2 * float(np.arcsin(s.sin_half_beam)), 0.0, False, True)
            _, terms = bp.count_terms()
        else:
            terms = dense
        bp.form_device(img)
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(a.steps):
            bp.form_device(img)
        t1.record()
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1) / a.steps
        res[mode] = {"ms_per_step": ms, "terms": terms, "Gterm_per_s": terms / (ms * 1e-3) / 1e9,
                     "dense_equivalent_Gterm_per_s": dense / (ms * 1e-3) / 1e9}
    plan = bp.plan()
    out = {"config": cid, "name": s.name, "grid": [g["nx"], g["ny"], g["nz"]], "P": P, "E": E, "Ns": Ns,
           "echo_GB": P * E * Ns * 8 / 1e9, "dense_terms": dense, "in_window_terms": inwin, "plan": plan,
           "roof_Gterm_per_s": roof(E) / 1e9, "frac": res["dense"]["Gterm_per_s"] / (roof(E) / 1e9), **res,
           "data": "device-random complex64 echoes (timing only)"}
    print(json.dumps(out), flush=True)
    bp.close()
    del e, img
    torch.cuda.empty_cache()
