"""Multi-GPU TDBP over torch.distributed (one process per GPU; NCCL on B200s, gloo in CPU tests).

The method shards two ways; both are exact re-partitionings of the sum of
Eq. (eqn:backprojection)'s inversion ("Any pair of pixel locations ... can be computed
independently"; images add over pings):

* image-shard (default): rank r owns a contiguous band of grid rows (iy for 2D, iz for 3D) and
  forms it from ALL pings; the echoes are broadcast once from rank 0 over NVLink (the
  north star's "ping data broadcast once"), the bands are gathered to rank 0.  Every pixel
  sees the same channels in the same order as on one GPU; the only difference is the fp64
  rounding of the shifted band origin (~1e-13 m), i.e. ~1e-7 relative in the image.
* ping-shard: rank r forms the full grid from pings r::G; the partial images are summed to
  rank 0 with an NCCL reduce.  Output differs from one GPU only by fp32 summation order.

The per-rank compute is pluggable (`former`) so the host-side partitioning / collective logic
is testable on CPU with gloo; the product former is the CUDA library (make_cuda_former).
"""
from __future__ import annotations

from typing import Callable, Dict, Tuple

import numpy as np


def row_bands(n: int, world: int, align: int = 1):
    """Split n rows into `world` contiguous bands [lo, hi), sizes differing by at most `align`
    (bands start on multiples of `align` so CUDA tiles are not split)."""
    blocks = (n + align - 1) // align
    out = []
    for r in range(world):
        lo = (blocks * r) // world * align
        hi = min(n, (blocks * (r + 1)) // world * align)
        out.append((min(lo, n), hi))
    return out


def sub_grid(grid: Dict, lo: int, hi: int) -> Dict:
    """The band [lo, hi) of the slowest varying grid axis (y for 2D, z for 3D) as its own grid."""
    g = dict(grid)
    if grid["nz"] > 1:
        g["origin"] = np.asarray(grid["origin"], dtype=np.float64) + lo * np.asarray(grid["step_z"], dtype=np.float64)
        g["nz"] = hi - lo
    else:
        g["origin"] = np.asarray(grid["origin"], dtype=np.float64) + lo * np.asarray(grid["step_y"], dtype=np.float64)
        g["ny"] = hi - lo
    return g


def band_axis_len(grid: Dict) -> int:
    return grid["nz"] if grid["nz"] > 1 else grid["ny"]


def ping_shard(P: int, world: int, rank: int) -> np.ndarray:
    """Interleaved ping assignment r::G (balances pings with different window positions)."""
    return np.arange(rank, P, world)


Former = Callable[[Dict, object, np.ndarray, np.ndarray, np.ndarray, object], object]


def form_image_sharded(grid: Dict, echoes, tx, rx, t0, former: Former, dist, device=None, align: int = 32):
    """Image-shard TDBP.  `echoes` must be present on every rank (same tensor shape); call
    broadcast_echoes first if only rank 0 holds them.  Returns the full image on rank 0
    (a tensor [nz][ny][nx] complex64) and None elsewhere."""
    import torch
    world, rank = dist.get_world_size(), dist.get_rank()
    n = band_axis_len(grid)
    bands = row_bands(n, world, align if grid["nz"] == 1 else 8)
    lo, hi = bands[rank]
    hmax = max(b - a for a, b in bands)
    nz, ny, nx = grid["nz"], grid["ny"], grid["nx"]
    if nz > 1:
        part_shape, full_shape = (hmax, ny, nx), (nz, ny, nx)
    else:
        part_shape, full_shape = (1, hmax, nx), (1, ny, nx)
    part = torch.zeros(part_shape, dtype=torch.complex64, device=device)
    if hi > lo:
        img = former(sub_grid(grid, lo, hi), echoes, tx, rx, t0, device)
        if nz > 1:
            part[: hi - lo] = img
        else:
            part[:, : hi - lo] = img
    # all_gather is supported by both NCCL and gloo; only rank 0 keeps the result
    bufs = [torch.empty_like(part) for _ in range(world)]
    dist.all_gather([torch.view_as_real(b) for b in bufs], torch.view_as_real(part))
    if rank != 0:
        return None
    gathered = bufs
    out = torch.empty(full_shape, dtype=torch.complex64, device=device)
    for r, (a, b) in enumerate(bands):
        if b <= a:
            continue
        if nz > 1:
            out[a:b] = gathered[r][: b - a]
        else:
            out[:, a:b] = gathered[r][:, : b - a]
    return out


def form_ping_sharded(grid: Dict, echoes, tx, rx, t0, former: Former, dist, device=None):
    """Ping-shard TDBP: each rank holds only ITS pings (echoes[i] = ping ping_shard(P, G, r)[i])
    and forms the full grid; an NCCL reduce sums the partial images to rank 0."""
    img = former(grid, echoes, tx, rx, t0, device)
    view = img.view(-1) if img.is_contiguous() else img.reshape(-1)
    import torch
    flat = torch.view_as_real(view)
    dist.reduce(flat, dst=0, op=dist.ReduceOp.SUM)
    return img if dist.get_rank() == 0 else None


def broadcast_echoes(echoes, dist, src: int = 0):
    """Broadcast the device-resident echoes from `src` to every rank (NCCL over NVLink)."""
    import torch
    flat = torch.view_as_real(echoes.view(-1))
    dist.broadcast(flat, src=src)
    return echoes


def make_cuda_former(fc: float, bandwidth: float, fs: float, c: float, cache: Dict = None):
    """Per-rank former backed by libsasbp (plans cached per sub-grid)."""
    import torch
    from .sasbp import Backprojector
    plans = {} if cache is None else cache

    def former(g, echoes, tx, rx, t0, device):
        key = (tuple(np.asarray(g["origin"]).tolist()), g["nx"], g["ny"], g["nz"])
        bp = plans.get(key)
        if bp is None:
            bp = plans[key] = Backprojector(fc, bandwidth, fs, c, g)
        bp.set_pings_device(echoes, tx, rx, t0)
        img = torch.empty((g["nz"], g["ny"], g["nx"]), dtype=torch.complex64, device=echoes.device)
        bp.form_device(img)
        return img

    return former
