"""One TDBP launch on a BASELINE config for ncu (device-resident inputs, 1 warm-up form + N profiled).
    python tools/prof_tdbp.py [--config 2] [--forms 2]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_2101_05888_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--forms", type=int, default=2)
ap.add_argument("--reduced", action="store_true")
a = ap.parse_args()
s = synth.scenario(a.config, reduced=a.reduced)
e = torch.from_numpy(s.echoes()).cuda()
bp = pkg.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid)
bp.set_pings_device(e, s.tx, s.rx, s.t0)
img = torch.empty(bp.shape, dtype=torch.complex64, device="cuda")
for _ in range(a.forms):
    bp.form_device(img)
torch.cuda.synchronize()
print("done", s.name, bp.shape, float(img.abs().max()))
