"""One TDBP launch on a BASELINE config for ncu (device-resident inputs, 1 warm-up form + N profiled).
    python tools/prof_tdbp.py [--config 2] [--forms 2] [--pings P'] [--random] [--gated]

--pings P' keeps the first P' pings of the config (same grid, elements, samples and plan), so an
`ncu --set full` replay of a config whose full launch takes seconds (config 4: 6.7 s) finishes;
--random uses seeded device-random echoes of the config's shape (the TDBP work is data
independent) instead of generating the synthetic scene."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2101_05888_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--forms", type=int, default=2)
ap.add_argument("--reduced", action="store_true")
ap.add_argument("--pings", type=int, default=0)
ap.add_argument("--random", action="store_true")
ap.add_argument("--gated", action="store_true")
a = ap.parse_args()
s = synth.scenario(a.config, reduced=a.reduced)
P = a.pings if a.pings > 0 else s.P
if a.random:
    gen = torch.Generator(device="cuda").manual_seed(1000 + a.config)
    e = torch.randn((P, s.E, s.Ns), dtype=torch.complex64, device="cuda", generator=gen)
else:
    e = torch.from_numpy(np.ascontiguousarray(s.echoes()[:P])).cuda()
bp = pkg.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid)
bp.set_pings_device(e, s.tx[:P], s.rx[:P], s.t0[:P])
if a.gated and s.sin_half_beam > 0:
    bp.set_beam(2 * float(np.arcsin(s.sin_half_beam)), 0.0, False, True)
img = torch.empty(bp.shape, dtype=torch.complex64, device="cuda")
for _ in range(a.forms):
    bp.form_device(img)
torch.cuda.synchronize()
print("done", s.name, bp.shape, "P", P, bp.plan(), float(img.abs().max()))
