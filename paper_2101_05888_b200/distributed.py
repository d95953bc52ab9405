"""Multi-GPU TDBP over torch.distributed (one process per GPU; NCCL on B200s, gloo in CPU tests).

The method shards two ways; both are exact re-partitionings of the sum of
Eq. (eqn:backprojection)'s inversion ("Any pair of pixel locations ... can be computed
independently"; images add over pings):

* image-shard: rank r owns a contiguous band of grid rows (iy for 2D, iz for 3D, aligned to the
  CUDA tile height) and forms it from ALL pings.  Echoes: every rank copies its 1/G slice of the
  pings host -> device and an NCCL all-gather assembles the full ping set on every rank over
  NVLink (each byte crosses PCIe once, the north star's "ping data broadcast once").  The bands
  are gathered to rank 0 only.  Every pixel sees the same channels in the same order as on one
  GPU; each band's plan (series order or exact receive leg) is chosen for the band by the same
  truncation bound, so a band equals the single-GPU image to the fp32 rounding of its own plan
  (within the parity tolerance; bitwise when the plans coincide).
* ping-shard: rank r holds and forms pings r::G over the full grid; the partial images are summed
  to rank 0 with an NCCL reduce.  Output differs from one GPU only by fp32 summation order.

The per-rank compute is pluggable (`former`) so the host-side partitioning / collective logic
is testable on CPU with gloo; the product former is the CUDA library (make_cuda_former).
"""
from __future__ import annotations

from typing import Callable, Dict

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


def band_align(grid: Dict) -> int:
    """Rows per CUDA tile along the band axis (2D: 32 rows of y, 3D: 8 planes of z)."""
    return 8 if grid["nz"] > 1 else 32


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


def ping_slices(P: int, world: int):
    """Contiguous, equal-size ping slices [lo, hi) for the echo all-gather (the last may be padded:
    slice size = ceil(P / world))."""
    per = (P + world - 1) // world
    return [(min(P, r * per), min(P, (r + 1) * per)) for r in range(world)], per


Former = Callable[[Dict, object, np.ndarray, np.ndarray, np.ndarray, object], object]


def gather_echoes(local, full_padded, dist):
    """All-gather equal-size ping slices `local` [per][E][Ns] into `full_padded` [world*per][E][Ns]
    (NCCL all_gather_into_tensor over NVLink; gloo in CPU tests).  Returns full_padded."""
    import torch
    if hasattr(dist, "all_gather_into_tensor") and dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(torch.view_as_real(full_padded).view(-1), torch.view_as_real(local).view(-1))
    else:
        world = dist.get_world_size()
        per = local.shape[0]
        parts = [torch.view_as_real(full_padded[r * per:(r + 1) * per]) for r in range(world)]
        dist.all_gather(parts, torch.view_as_real(local))
    return full_padded


def gather_bands(part, grid: Dict, bands, dist, out=None):
    """Gather the per-rank band images (each padded to the largest band) to rank 0 and assemble the
    full image there (returned on rank 0, None elsewhere).  `part` is [hmax][ny][nx] (3D) or
    [1][hmax][nx] (2D)."""
    import torch
    world, rank = dist.get_world_size(), dist.get_rank()
    nz, ny, nx = grid["nz"], grid["ny"], grid["nx"]
    bufs = [torch.empty_like(part) for _ in range(world)] if rank == 0 else None
    dist.gather(torch.view_as_real(part), [torch.view_as_real(b) for b in bufs] if bufs else None, dst=0)
    if rank != 0:
        return None
    if out is None:
        out = torch.empty((nz, ny, nx), dtype=torch.complex64, device=part.device)
    for r, (a, b) in enumerate(bands):
        if b <= a:
            continue
        if nz > 1:
            out[a:b] = bufs[r][: b - a]
        else:
            out[:, a:b] = bufs[r][:, : b - a]
    return out


def band_part_shape(grid: Dict, bands):
    hmax = max(b - a for a, b in bands)
    return (hmax, grid["ny"], grid["nx"]) if grid["nz"] > 1 else (1, hmax, grid["nx"])


def form_image_sharded(grid: Dict, echoes, tx, rx, t0, former: Former, dist, device=None, align: int = None):
    """Image-shard TDBP.  `echoes` must be present on every rank (gather_echoes first if each rank
    holds only its slice).  Returns the full image on rank 0 (a tensor [nz][ny][nx] complex64) and
    None elsewhere; the bands travel to rank 0 only."""
    import torch
    world, rank = dist.get_world_size(), dist.get_rank()
    bands = row_bands(band_axis_len(grid), world, align or band_align(grid))
    lo, hi = bands[rank]
    part = torch.zeros(band_part_shape(grid, bands), dtype=torch.complex64, device=device)
    if hi > lo:
        img = former(sub_grid(grid, lo, hi), echoes, tx, rx, t0, device)
        if grid["nz"] > 1:
            part[: hi - lo] = img
        else:
            part[:, : hi - lo] = img
    return gather_bands(part, grid, bands, dist)


def form_ping_sharded(grid: Dict, echoes, tx, rx, t0, former: Former, dist, device=None):
    """Ping-shard TDBP: each rank holds only ITS pings (echoes[i] = ping ping_shard(P, G, r)[i])
    and forms the full grid; an NCCL reduce sums the partial images to rank 0."""
    import torch
    img = former(grid, echoes, tx, rx, t0, device)
    view = img.view(-1) if img.is_contiguous() else img.reshape(-1)
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
    """Per-rank former backed by libsasbp (plans cached per sub-grid: origin, steps and sizes, and
    the former's own fc, bandwidth, fs, c, so a shared cache never returns another grid's plan)."""
    import torch
    from .sasbp import Backprojector
    plans = {} if cache is None else cache

    def former(g, echoes, tx, rx, t0, device):
        key = (float(fc), float(bandwidth), float(fs), float(c),
               *(tuple(np.asarray(g[k], dtype=np.float64).reshape(3).tolist()) for k in
                 ("origin", "step_x", "step_y", "step_z")),
               int(g["nx"]), int(g["ny"]), int(g["nz"]))
        bp = plans.get(key)
        if bp is None:
            bp = plans[key] = Backprojector(fc, bandwidth, fs, c, g)
        bp.set_pings_device(echoes, tx, rx, t0)
        img = torch.empty((g["nz"], g["ny"], g["nx"]), dtype=torch.complex64, device=echoes.device)
        bp.form_device(img)
        return img

    return former
