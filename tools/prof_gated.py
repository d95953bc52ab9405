"""One gated (NEXT-1) TDBP launch on config 2 with the generator's beam, for ncu."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2101_05888_b200 as pkg  # noqa: E402

s = synth.scenario(2)
e = torch.randn((s.P, s.E, s.Ns), dtype=torch.complex64, device="cuda")
bp = pkg.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid)
bp.set_pings_device(e, s.tx, s.rx, s.t0)
bp.set_beam(2 * float(np.arcsin(s.sin_half_beam)), 0.0, False, True)
img = torch.empty(bp.shape, dtype=torch.complex64, device="cuda")
bp.form_device(img)
torch.cuda.synchronize()
print("done")
