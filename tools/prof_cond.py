"""One launch each of the conditioning kernels (K1b upsample x4, K0 baseband) at the bench's
config-2 channel layout, for ncu captures:
    ncu --set full -k regex:"upsample|baseband|wh_periodogram|rc_fft" -o gpurun_out/ncu_cond python tools/prof_cond.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_05888_b200 as pkg  # noqa: E402

P, E, Ns, fs, fc = 1000, 32, 10240, 120e3, 120e3
nch = P * E
x = torch.randn((nch, Ns // 4), dtype=torch.complex64, device="cuda")
y = torch.empty((nch, Ns), dtype=torch.complex64, device="cuda")
pkg.upsample_device(x, 4, y)
del x, y
pb = torch.randn((P, E, 4 * Ns), dtype=torch.float32, device="cuda")
out = torch.empty((P, E, Ns), dtype=torch.complex64, device="cuda")
kk = np.arange(-31, 32)
h = (2 * 0.1 * np.sinc(2 * 0.1 * kk) * (0.5 + 0.5 * np.cos(np.pi * kk / 32))).astype(np.float32)
h *= np.float32(2.0 / h.sum())
pkg.baseband_device(pb, 4 * fs, fc, torch.full((P,), 0.02667, dtype=torch.float64, device="cuda"),
                    torch.from_numpy(h).cuda(), 4, out)
torch.cuda.synchronize()
print("ok")
del pb, out
# whitening gain (M = 64) and K1 range compression on the same layout
x = torch.randn((P, E, Ns), dtype=torch.complex64, device="cuda")
G = torch.empty(64, dtype=torch.float32, device="cuda")
pkg.whitening_gain_device(x, 64, 0.0, G)
t = np.arange(600) / fs - 2.5e-3
rep = torch.from_numpy((np.exp(1j * np.pi * (30e3 / 5e-3) * t ** 2) / np.sqrt(600)).astype(np.complex64)).cuda()
y = torch.empty_like(x)
pkg.rangecompress_device(x, rep, y)
torch.cuda.synchronize()
print("ok2")
