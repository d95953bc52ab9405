"""K1 range-compression timing on the cfg-2 channel layout (for A/B builds via SASBP_LIB)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_05888_b200 as pkg  # noqa: E402

P, E, Ns, fs, B, Tp = 1000, 32, 10240, 120e3, 30e3, 5e-3
nr = int(round(Tp * fs))
t = np.arange(nr) / fs - Tp / 2
rep = torch.from_numpy((np.exp(1j * np.pi * (B / Tp) * t ** 2) / np.sqrt(nr)).astype(np.complex64)).cuda()
x = torch.randn(P, E, Ns, dtype=torch.complex64, device="cuda")
y = torch.empty_like(x)
for _ in range(50):   # warm the clocks up
    pkg.rangecompress_device(x, rep, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    pkg.rangecompress_device(x, rep, y)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 50
print(os.environ.get("SASBP_LIB", "default"), f"{ms:.3f} ms", f"{16 * P * E * Ns / ms / 1e6:.0f} GB/s")
