"""Multi-process (world_size 2, gloo, CPU) tests of the multi-GPU partitioning and collective
logic (paper_2101_05888_b200/distributed.py).  The per-rank compute is the fp64 oracle here
(injected by the test); on B200s the same code calls the CUDA former over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2101_05888_b200 import distributed as pdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_former(g, echoes, tx, rx, t0, device):
    sc = _SC
    e = echoes.numpy() if isinstance(echoes, torch.Tensor) else echoes
    img = oracle.tdbp_grid(e, tx, rx, t0, sc.fc, sc.fs, sc.c, g)
    return torch.from_numpy(img.astype(np.complex64))


_SC = None


def _worker(rank, world, port, mode, cid, out_q):
    global _SC
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = synth.scenario(cid, reduced=True)
        _SC = s
        e = torch.from_numpy(s.echoes())
        if mode == "image":
            # each rank holds only its contiguous ping slice; the all-gather assembles the set
            sl, per = pdist.ping_slices(s.P, world)
            lo, hi = sl[rank]
            local = torch.zeros((per,) + tuple(e.shape[1:]), dtype=e.dtype)
            local[: hi - lo] = e[lo:hi]
            full_e = torch.empty((per * world,) + tuple(e.shape[1:]), dtype=e.dtype)
            pdist.gather_echoes(local, full_e, dist)
            e = full_e[: s.P].contiguous()
            full = pdist.form_image_sharded(s.grid, e, s.tx, s.rx, s.t0, oracle_former, dist)
        else:
            sel = pdist.ping_shard(s.P, world, rank)
            full = pdist.form_ping_sharded(s.grid, e[sel].contiguous(), s.tx[sel], s.rx[sel], s.t0[sel],
                                           oracle_former, dist)
        if rank == 0:
            out_q.put(full.numpy())
    finally:
        dist.destroy_process_group()


def _run(mode, cid, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, cid, q)) for r in range(world)]
    for p in procs:
        p.start()
    img = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return img


@pytest.mark.parametrize("cid", [2, 4])
def test_image_shard_equals_single(cid):
    """Image-shard: bands formed on different ranks reassemble to the single-process image
    (per-pixel independence) -- equal up to the fp64 rounding of the shifted
    band origin."""
    s = synth.scenario(cid, reduced=True)
    ref = oracle.tdbp_grid(s.echoes(), s.tx, s.rx, s.t0, s.fc, s.fs, s.c, s.grid).astype(np.complex64)
    got = _run("image", cid)
    assert got.shape == ref.shape
    assert np.max(np.abs(got - ref)) <= 1e-6 * np.max(np.abs(ref))


def test_ping_shard_sums_to_single():
    """Ping-shard: partial images over disjoint ping sets reduce to the full image."""
    s = synth.scenario(2, reduced=True)
    ref = oracle.tdbp_grid(s.echoes(), s.tx, s.rx, s.t0, s.fc, s.fs, s.c, s.grid)
    got = _run("ping", 2)
    assert np.max(np.abs(got - ref)) <= 1e-5 * np.max(np.abs(ref))


def test_three_ranks_ragged_bands():
    s = synth.scenario(2, reduced=True)
    ref = oracle.tdbp_grid(s.echoes(), s.tx, s.rx, s.t0, s.fc, s.fs, s.c, s.grid).astype(np.complex64)
    got = _run("image", 2, world=3)
    assert np.max(np.abs(got - ref)) <= 1e-6 * np.max(np.abs(ref))


def test_row_bands_cover_and_align():
    for n in [1, 31, 32, 33, 150, 4096, 4097]:
        for world in [1, 2, 3, 8]:
            b = pdist.row_bands(n, world, 32)
            assert b[0][0] == 0 and b[-1][1] == n
            for (a0, a1), (c0, c1) in zip(b, b[1:]):
                assert a1 == c0
            for a, _ in b:
                assert a % 32 == 0 or a == n
            sizes = [hi - lo for lo, hi in b]
            assert max(sizes) - min(sizes) <= 32


def test_sub_grid_origin():
    g = synth.grid_dict((1.0, 2.0, 3.0), (0.1, 0.2, 0.3), (10, 20, 1))
    sg = pdist.sub_grid(g, 5, 12)
    assert sg["ny"] == 7 and np.allclose(sg["origin"], [1.0, 3.0, 3.0])
    g3 = synth.grid_dict((1.0, 2.0, 3.0), (0.1, 0.2, 0.3), (10, 20, 16))
    sg3 = pdist.sub_grid(g3, 8, 16)
    assert sg3["nz"] == 8 and np.allclose(sg3["origin"], [1.0, 2.0, 3.0 + 2.4])


def test_ping_slices_cover():
    for P in (1, 7, 1000, 1001):
        for world in (1, 2, 3, 8):
            sl, per = pdist.ping_slices(P, world)
            assert sl[0][0] == 0 and sl[-1][1] == P and per * world >= P
            assert all(a1 == c0 for (a0, a1), (c0, c1) in zip(sl, sl[1:]))
            assert all(hi - lo <= per for lo, hi in sl)


def test_ping_shard_partition():
    P = 1001
    parts = [pdist.ping_shard(P, 8, r) for r in range(8)]
    allp = np.sort(np.concatenate(parts))
    assert np.array_equal(allp, np.arange(P))
