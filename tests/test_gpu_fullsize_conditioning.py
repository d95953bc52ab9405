"""Full-size parity of the conditioning kernels in the launch configuration bench.py times
(-m gpu): the whole config-2 channel layout (32 000 channels) goes through K1, K1b, K0 and the
whitening kernels on the device; sampled channels are compared with the oracle element by element
(bars as in tests/test_gpu_next4.py), and the full-batch whitening gain against an exactly known
spectrum."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
P, E, Ns = 1000, 32, 10240
NCH = P * E
SAMPLE = [0, 1, 12345, 20000, NCH - 1]
TOL = 2e-5


@pytest.fixture(scope="module")
def pk(require_gpu):
    import torch
    torch.cuda.set_device(0)
    from paper_2101_05888_b200 import _build
    _build.build()
    import paper_2101_05888_b200 as pkg
    return pkg


def _lfm(n, fs=120e3, B=30e3):
    t = np.arange(n) / fs - n / (2 * fs)
    Tp = n / fs
    return (np.exp(1j * np.pi * (B / Tp) * t ** 2) / np.sqrt(n)).astype(np.complex64)


def _dev_randn(shape, seed, complex_=True):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(shape, dtype=torch.complex64 if complex_ else torch.float32, device="cuda", generator=g)


def test_rangecompress_full_layout(pk):
    import torch
    x = _dev_randn((P, E, Ns), 11)
    rep = _lfm(600)
    y = torch.empty_like(x)
    pk.rangecompress_device(x, torch.from_numpy(rep).cuda(), y)
    torch.cuda.synchronize()
    xf, yf = x.view(NCH, Ns), y.view(NCH, Ns)
    for c in SAMPLE:
        ref = oracle.rangecompress(xf[c].cpu().numpy(), rep)
        assert np.max(np.abs(yf[c].cpu().numpy() - ref)) <= TOL * np.max(np.abs(ref)), c


def test_upsample_full_layout(pk):
    import torch
    x = _dev_randn((NCH, Ns // 4), 12)
    y = torch.empty((NCH, Ns), dtype=torch.complex64, device="cuda")
    pk.upsample_device(x, 4, y)
    torch.cuda.synchronize()
    for c in SAMPLE:
        ref = oracle.upsample(x[c].cpu().numpy(), 4)
        assert np.max(np.abs(y[c].cpu().numpy() - ref)) <= TOL * np.max(np.abs(ref)), c


def test_baseband_full_layout(pk):
    import torch
    x = _dev_randn((P, E, 4 * Ns), 13, complex_=False)
    k = np.arange(-31, 32)
    h = (2 * 0.1 * np.sinc(2 * 0.1 * k) * (0.5 + 0.5 * np.cos(np.pi * k / 32))).astype(np.float32)
    h *= np.float32(2.0 / h.sum())
    t0 = np.full(P, 0.02667) + 1e-5 * np.arange(P)
    out = torch.empty((P, E, Ns), dtype=torch.complex64, device="cuda")
    pk.baseband_device(x, 480e3, 120e3, torch.from_numpy(t0).cuda(), torch.from_numpy(h).cuda(), 4, out)
    torch.cuda.synchronize()
    for c in SAMPLE:
        p, e = divmod(c, E)
        ref = oracle.baseband(x[p, e].cpu().numpy().reshape(1, 1, -1), 480e3, 120e3, t0[p:p + 1], h, 4, Ns)[0, 0]
        assert np.max(np.abs(out[p, e].cpu().numpy() - ref)) <= TOL * np.max(np.abs(ref)), c


def test_whitening_gain_full_batch_known_spectrum(pk):
    """Every 64-sample block of all 32 000 channels is the same sequence b, so the batch-mean
    periodogram is exactly |DFT(b)|^2: the full-size GPU gain equals the oracle's on one block."""
    import torch
    rng = np.random.default_rng(14)
    b = ((rng.normal(size=64) + 1j * rng.normal(size=64)) * (1 + np.arange(64) / 16)).astype(np.complex64)
    x = torch.from_numpy(np.tile(b, Ns // 64)).cuda().view(1, 1, Ns).expand(P, E, Ns).contiguous()
    G = torch.empty(64, dtype=torch.float32, device="cuda")
    pk.whitening_gain_device(x, 64, 0.1, G)
    torch.cuda.synchronize()
    ref, _ = oracle.whitening_gain(b.reshape(1, -1), 64, 0.1)
    assert np.max(np.abs(G.cpu().numpy() - ref)) <= 2e-5


def test_whitened_compression_full_layout(pk):
    import torch
    x = _dev_randn((P, E, Ns), 15)
    rep = _lfm(600)
    G = torch.empty(64, dtype=torch.float32, device="cuda")
    pk.whitening_gain_device(x, 64, 0.05, G)
    y = torch.empty_like(x)
    pk.rangecompress_whitened_device(x, torch.from_numpy(rep).cuda(), G, y)
    torch.cuda.synchronize()
    Gh = G.cpu().numpy().astype(np.float64)
    xf, yf = x.view(NCH, Ns), y.view(NCH, Ns)
    for c in (0, NCH - 1):
        ref = oracle.rangecompress_whitened(xf[c].cpu().numpy(), rep, Gh)
        assert np.max(np.abs(yf[c].cpu().numpy() - ref)) <= TOL * np.max(np.abs(ref)), c
