"""K1 range-compression timing on a BASELINE config's channel layout (A/B builds via SASBP_LIB).
    python tools/k1_bench.py [--config 2|4] [--reps 50]
The replica is the bench's (T_p = 5 ms for 2D configs, 2 ms for the 3D config)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2101_05888_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--reps", type=int, default=50)
a = ap.parse_args()
s = synth.scenario(a.config)
P, E, Ns, fs, B = s.P, s.E, s.Ns, s.fs, s.bandwidth
Tp = 2e-3 if s.grid["nz"] > 1 else 5e-3
nr = int(round(Tp * fs))
t = np.arange(nr) / fs - Tp / 2
rep = torch.from_numpy((np.exp(1j * np.pi * (B / Tp) * t ** 2) / np.sqrt(nr)).astype(np.complex64)).cuda()
x = torch.randn(P, E, Ns, dtype=torch.complex64, device="cuda")
y = torch.empty_like(x)
for _ in range(a.reps):   # warm the clocks up
    pkg.rangecompress_device(x, rep, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    pkg.rangecompress_device(x, rep, y)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
print(os.environ.get("SASBP_LIB", "default"), f"cfg {a.config} Nr {nr} nopack={os.environ.get('SASBP_RC_NOPACK', '0')}",
      f"{ms:.3f} ms", f"{16 * P * E * Ns / ms / 1e6:.0f} GB/s", flush=True)
