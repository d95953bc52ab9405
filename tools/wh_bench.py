"""Whitening-gain (periodogram) timing on the cfg-2 channel layout, M = 64 (A/B via SASBP_LIB)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_05888_b200 as pkg  # noqa: E402

x = torch.randn(1000, 32, 10240, dtype=torch.complex64, device="cuda")
G = torch.empty(64, dtype=torch.float32, device="cuda")
for _ in range(20):
    pkg.whitening_gain_device(x, 64, 0.0, G)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    pkg.whitening_gain_device(x, 64, 0.0, G)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(os.environ.get("SASBP_LIB", "default"), f"{ms:.3f} ms", f"{x.numel() * 8 / ms / 1e6:.0f} GB/s")
