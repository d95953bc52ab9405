"""Predict multi-GPU scaling of both partitionings from 1-GPU timings.

Only one B200 is reachable from this environment, so N > 1 cannot be timed directly.  This tool
times, on one GPU, exactly the launch each rank of an N-GPU run would make, one after the other:

* image-shard: rank r forms its band of grid rows (`distributed.row_bands`, the bench's bands)
  from all pings;
* ping-shard: rank r forms the full grid from pings r::N.

and predicts the step time of the N-GPU run as  max_r T_r + T_combine(N), where T_combine is
the bench step's exchange (image-shard: gather of the bands to rank 0; ping-shard: NCCL reduce
of the complex image to rank 0) modelled as bytes / BW with BW an ASSUMED effective NVLink-5
collective bandwidth (--bw-gbs, default 400 GB/s; nominal 900 GB/s per direction per GPU).
Efficiency  eta(N) = T_1 / (N * T_pred(N)).  The work is data independent, so the echoes are
seeded device-random arrays of the config's shape.  One JSON line per (config, scheme, N).

    python tools/predict_scaling.py [--configs 4,2,5] [--ns 2,4,8] [--bw-gbs 400]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2101_05888_b200 as pkg  # noqa: E402
from paper_2101_05888_b200 import distributed as pdist  # noqa: E402


def timed_form(s, grid, echoes, tx, rx, t0, reps):
    bp = pkg.Backprojector(s.fc, s.bandwidth, s.fs, s.c, grid)
    bp.set_pings_device(echoes, tx, rx, t0)
    img = torch.empty(bp.shape, dtype=torch.complex64, device="cuda")
    bp.form_device(img)   # warm
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        bp.form_device(img)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    _, nu = bp.count_terms()
    bp.close()
    return min(ms), nu


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="4,2")
    ap.add_argument("--ns", default="2,4,8")
    ap.add_argument("--bw-gbs", type=float, default=400.0)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    for cfg in [int(c) for c in a.configs.split(",")]:
        s = synth.scenario(cfg)
        g = s.grid
        gen = torch.Generator(device="cuda").manual_seed(4242 + cfg)
        e = torch.randn((s.P, s.E, s.Ns), dtype=torch.complex64, device="cuda", generator=gen)
        t1, nu1 = timed_form(s, g, e, s.tx, s.rx, s.t0, a.reps)
        img_bytes = g["nx"] * g["ny"] * g["nz"] * 8
        print(json.dumps({"config": cfg, "scheme": "single", "N": 1, "ms": t1, "Gterm_per_s": nu1 / t1 / 1e6}),
              flush=True)
        for n in [int(x) for x in a.ns.split(",")]:
            bands = pdist.row_bands(pdist.band_axis_len(g), n, pdist.band_align(g))
            t_img = []
            for lo, hi in bands:
                t_img.append(timed_form(s, pdist.sub_grid(g, lo, hi), e, s.tx, s.rx, s.t0, a.reps)[0] if hi > lo else 0.0)
            # bands gathered to rank 0: it receives (N-1)/N of the image (padded to the largest band)
            hmax = max(hi - lo for lo, hi in bands)
            gather_bytes = (n - 1) * hmax * img_bytes / pdist.band_axis_len(g)
            t_comm = gather_bytes / (a.bw_gbs * 1e9) * 1e3
            pred = max(t_img) + t_comm
            print(json.dumps({"config": cfg, "scheme": "image", "N": n, "rank_ms": t_img, "max_rank_ms": max(t_img),
                              "combine_ms_model": t_comm, "combine_bytes": gather_bytes, "pred_step_ms": pred,
                              "eta_pred": t1 / (n * pred), "bw_gbs_assumed": a.bw_gbs}), flush=True)
            t_png = []
            for r in range(n):
                sel = pdist.ping_shard(s.P, n, r)
                er = e.index_select(0, torch.from_numpy(sel).cuda())
                t_png.append(timed_form(s, g, er, s.tx[sel], s.rx[sel], s.t0[sel], a.reps)[0])
                del er
            # reduce of the full complex image to rank 0 (ring/tree: ~ image bytes per link)
            t_comm = img_bytes / (a.bw_gbs * 1e9) * 1e3
            pred = max(t_png) + t_comm
            print(json.dumps({"config": cfg, "scheme": "ping", "N": n, "rank_ms": t_png, "max_rank_ms": max(t_png),
                              "combine_ms_model": t_comm, "combine_bytes": img_bytes, "pred_step_ms": pred,
                              "eta_pred": t1 / (n * pred), "bw_gbs_assumed": a.bw_gbs}), flush=True)
        del e
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
