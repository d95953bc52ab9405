"""K0 basebanding timing on a BASELINE config's channel layout (the bench's K0 leg: real passband at
4 fs, D = 4, 63-tap windowed-sinc low-pass), for A/B via SASBP_LIB / SASBP_BB_VEC4.
    python tools/k0_bench.py [--config 4] [--reps 20]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2101_05888_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
s = synth.scenario(a.config)
P, E, Ns = s.P, s.E, s.Ns
nin = 4 * Ns
pb = torch.randn((P, E, nin), dtype=torch.float32, device="cuda")
out = torch.empty((P, E, Ns), dtype=torch.complex64, device="cuda")
kk = np.arange(-31, 32)
h = (2 * 0.1 * np.sinc(2 * 0.1 * kk) * (0.5 + 0.5 * np.cos(np.pi * kk / 32))).astype(np.float32)
h *= np.float32(2.0 / h.sum())
t0 = torch.from_numpy(np.ascontiguousarray(s.t0, dtype=np.float64)).cuda()
hd = torch.from_numpy(h).cuda()
fn = lambda: pkg.baseband_device(pb, 4 * s.fs, s.fc, t0, hd, 4, out)  # noqa: E731
for _ in range(a.reps):
    fn()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    fn()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
nbytes = 4 * P * E * nin + 8 * P * E * Ns
print(os.environ.get("SASBP_LIB", "default"), f"cfg {a.config} vec4={os.environ.get('SASBP_BB_VEC4', '1')}",
      f"{ms:.3f} ms", f"{nbytes / ms / 1e6:.0f} GB/s", flush=True)
