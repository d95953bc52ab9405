#!/usr/bin/env python
"""Benchmark of the TDBP hot path (BASELINE.json metric: giga pixel.ping.element backprojections/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl sasbp|reference] [--config 4]
                    [--shard image|ping]

A step = one whole TDBP image formation (all §8(a) rows: reference geometry, delays,
interpolation, phase ramp, accumulation, image write, and for N > 1 the combine collective)
over config 4 of BASELINE.json by default -- the 3D volumetric config the north star's targets
name (near-field, 1000 pings x 256 elements x 1024 samples, 512 x 512 x 128 voxels; synthetic,
seeded inputs from synth/).  N = 1 times one GPU; under torchrun (N > 1) the work is sharded
across ranks, strong scaling: --shard ping (default; pings r::G, NCCL reduce of the image) or
--shard image (bands of the grid, echoes all-gathered over NVLink, bands gathered to rank 0).
The default is the scheme DESIGN.md §6 predicts to scale better from 1-GPU timings of every
rank's launch (tools/predict_scaling.py: config 4 at N = 8, eta 0.999 ping vs 0.973 image).

value  : N_u (terms whose interpolation support meets the record, K3; = dense for configs 1-4)
         / device time of the timed steps (CUDA events on the launching stream, max over
         ranks), inputs resident.
e2e    : the same metric through the public API with HOST buffers (pinned echoes -> H2D ->
         form -> D2H image), wall time per step, max over ranks.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "giga pixel·ping·element backprojections/s"
UNIT = "Gterm/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="sasbp", choices=["sasbp", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--shard", default="ping", choices=["image", "ping"],
                    help="N > 1 partitioning (SURVEY §8(e)): interleaved pings + NCCL reduce (default: the "
                         "scheme predicted to scale better, profiles/scaling_pred_r02.jsonl) or image bands")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-k1", action="store_true")
    ap.add_argument("--no-gated", action="store_true")
    ap.add_argument("--no-next4", action="store_true")
    return ap.parse_args()


# ------------------------------------------------------------------ roofline

def roof_terms_per_s(E: int, sms: int, f_hz: float) -> float:
    """FP32/SFU roofline of the canonical per-term instruction mix:
    F = 20 + 6/E FP32-pipe ops, S = 3 + 1/E MUFU ops per term; 128 FP32 lanes and 16 MUFU per SM
    per clock (B200, measured in profiles/ubench_r01.jsonl)."""
    F = 20.0 + 6.0 / E
    S = 3.0 + 1.0 / E
    return sms * f_hz * min(128.0 / F, 16.0 / S)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        pw = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "power_w_max": max(pw) if pw else None}


# ------------------------------------------------------------------ CPU oracle baseline

def cpu_oracle_rate(s, echoes, seconds: float, seed: int = 123):
    """Time the fp64 oracle (as it stands) on a bounded random-pixel sample of the workload."""
    import oracle
    rng = np.random.default_rng(seed)
    g = s.grid

    def sample(n):
        return np.stack([rng.integers(0, g["nx"], n), rng.integers(0, g["ny"], n), rng.integers(0, g["nz"], n)], 1)

    oracle.tdbp_grid(echoes, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, g, idx=sample(16))  # load + thread pool
    probe = sample(512)
    t = time.perf_counter()
    oracle.tdbp_grid(echoes, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, g, idx=probe)
    dt = max(time.perf_counter() - t, 1e-6)
    n = int(max(512, min(1 << 21, 512 * seconds / dt)))
    idx = sample(n)
    t = time.perf_counter()
    oracle.tdbp_grid(echoes, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, g, idx=idx)
    dt = time.perf_counter() - t
    terms = n * s.P * s.E
    return {"value": terms / dt / 1e9, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"{n} seeded-random pixels of config {s.name} x all {s.P} pings x {s.E} elements "
                      f"({terms:.3e} terms, {dt:.1f} s, fp64 C + OpenMP)"}


def _profile_traffic(name, config):
    """dram bytes per launch from a committed ncu summary (profiles/), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            pj = json.load(f)
        if config is not None and pj.get("config") != config:
            return None
        return pj.get("dram_bytes_per_launch")
    except Exception:
        return None


def _measured_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def host_cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


# ------------------------------------------------------------------ arms

def time_short_kernel(fn, stream, warm_s: float = 1.0, min_ms: float = 250.0, groups: int = 5) -> float:
    """ms per call of a short (few-ms) launch sequence: warm up for warm_s of wall time (clocks
    and memory state settle after the host-side gaps between bench phases), then time `groups`
    back-to-back groups of >= min_ms/groups each with CUDA events on `stream` and return the
    median group mean (a single short window was seen to vary 1.7-4 ms on an idle-to-busy box)."""
    import torch
    t_end = time.perf_counter() + warm_s
    n_warm = 0
    while time.perf_counter() < t_end or n_warm < 3:
        fn()
        n_warm += 1
        if n_warm % 8 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(3):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    est = max(a.elapsed_time(b) / 3, 1e-3)
    per = max(3, int(np.ceil(min_ms / groups / est)))
    means = []
    for _ in range(groups):
        a.record(stream)
        for _ in range(per):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        means.append(a.elapsed_time(b) / per)
    return float(np.median(means))


def workload_name(cid, s):
    g = s.grid
    kind = "3D volumetric" if g["nz"] > 1 else "2D stripmap"
    return (f"BASELINE config {cid}: {s.name} {kind} {g['nx']}x{g['ny']}x{g['nz']} pixels, "
            f"P={s.P} pings x E={s.E} elements x Ns={s.Ns} samples")


def run_reference(args):
    """Reference arm: the fp64 CPU oracle (this tier has no reference implementation)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import synth
    s = synth.scenario(args.config)
    echoes = s.echoes()
    per_step = max(2.0, 60.0 / max(1, args.steps + args.warmup))
    rates = []
    last = None
    for i in range(args.warmup + args.steps):
        last = cpu_oracle_rate(s, echoes, per_step, seed=1000 + i)
        if i >= args.warmup:
            rates.append(last["value"])
    v = float(np.mean(rates))
    terms_per_step = s.dense_terms
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": terms_per_step / (v * 1e9) * 1e3, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": workload_name(args.config, s), "terms_per_step": terms_per_step,
                      "parallelism": "host cores (oracle)", "sampled": True},
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": last["cores"], "kind": "oracle",
                            "sample": "per step: " + last["sample"], "cpu_model": host_cpu_model()},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "note": "reference arm = the fp64 C oracle on the host cores, timed on bounded random-pixel samples; "
                   "ms_per_step is extrapolated to the full image"}
    print(json.dumps(out), flush=True)
    return 0


def _collective_ok(dist, t):
    """gloo (test plumbing on one GPU) runs gather / reduce on host copies."""
    return dist.get_backend() == "nccl" or not t.is_cuda


def run_sasbp(args):
    import torch
    import torch.distributed as dist

    import synth
    import paper_2101_05888_b200 as pkg
    from paper_2101_05888_b200 import distributed as pdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test plumbing only (never used for a reported number): run the multi-rank path with every
    # rank on cuda:0 and gloo collectives, to exercise N > 1 on a one-GPU box
    if os.environ.get("SASBP_SAME_DEVICE") == "1":
        local = 0
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("SASBP_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    pkg.load_library()
    shard = args.shard if world > 1 else "none"

    s = synth.scenario(args.config)
    g = s.grid
    P, E, Ns = s.P, s.E, s.Ns
    dense = s.dense_terms
    # every rank generates the seeded scene itself (its "disk"); only its share goes to the device
    echoes_h = s.echoes()

    # ---- device-resident inputs and this rank's plan
    bands = pdist.row_bands(pdist.band_axis_len(g), world, pdist.band_align(g))
    if shard == "ping":
        sel = pdist.ping_shard(P, world, rank)
        my_h = np.ascontiguousarray(echoes_h[sel])
        tx, rx, t0 = s.tx[sel], s.rx[sel], s.t0[sel]
        echoes_d = torch.from_numpy(my_h).to(dev)
        sg = g
    else:
        # image-shard / one GPU: the full ping set on every rank, in the padded buffer the
        # echo all-gather of the e2e path fills (the plan borrows its first P pings)
        sl, per = pdist.ping_slices(P, world)
        full_pad = torch.empty((per * world, E, Ns), dtype=torch.complex64, device=dev)
        full_pad[:P].copy_(torch.from_numpy(echoes_h))
        echoes_d = full_pad[:P]
        tx, rx, t0 = s.tx, s.rx, s.t0
        lo, hi = bands[rank]
        sg = pdist.sub_grid(g, lo, hi) if world > 1 else g
    bp = pkg.Backprojector(s.fc, s.bandwidth, s.fs, s.c, sg)
    bp.set_pings_device(echoes_d, tx, rx, t0)
    stream = torch.cuda.current_stream()

    # combine-step buffers (row a6): image-shard gathers bands to rank 0, ping-shard reduces
    if shard == "image":
        part = torch.zeros(pdist.band_part_shape(g, bands), dtype=torch.complex64, device=dev)
        hb = bands[rank][1] - bands[rank][0]
        img = part[:hb] if g["nz"] > 1 else part[:, :hb]
        full_img = torch.empty((g["nz"], g["ny"], g["nx"]), dtype=torch.complex64, device=dev) if rank == 0 else None
    else:
        img = torch.empty(bp.shape, dtype=torch.complex64, device=dev)

    def combine():
        if shard == "image":
            if _collective_ok(dist, part):
                pdist.gather_bands(part, g, bands, dist, out=full_img)
            else:
                pc = part.cpu()
                out = pdist.gather_bands(pc, g, bands, dist)
                if rank == 0:
                    full_img.copy_(out)
        elif shard == "ping":
            if _collective_ok(dist, img):
                dist.reduce(torch.view_as_real(img.view(-1)), dst=0, op=dist.ReduceOp.SUM)
            else:
                ic = img.cpu()
                dist.reduce(torch.view_as_real(ic.view(-1)), dst=0, op=dist.ReduceOp.SUM)
                if rank == 0:
                    img.copy_(ic)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # metric denominator: N_u from K3, off the clock; summed over the ranks' shares
    _, nu_local = bp.count_terms()
    nu_t = torch.tensor([float(nu_local)], dtype=torch.float64, device=dev)
    if world > 1:
        if _collective_ok(dist, nu_t):
            dist.all_reduce(nu_t)
        else:
            c = nu_t.cpu(); dist.all_reduce(c); nu_t.copy_(c)
    n_u = int(round(float(nu_t[0])))

    for _ in range(args.warmup):
        bp.form_device(img, stream=stream)
        combine()
    barrier()

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    steps_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local) as clk:
        barrier()
        steps_ev[0].record(stream)
        for i in range(args.steps):
            evs[i][0].record(stream)
            bp.form_device(img, stream=stream)
            evs[i][1].record(stream)
            combine()                       # the step's exchange (N > 1): part of the timed step
            steps_ev[i + 1].record(stream)
        barrier()
    step_ms = [steps_ev[i].elapsed_time(steps_ev[i + 1]) for i in range(args.steps)]
    per_launch = [a.elapsed_time(b) for a, b in evs]
    tm = torch.tensor([sum(step_ms), statistics.mean(per_launch)] + step_ms, dtype=torch.float64, device=dev)
    if world > 1:
        if _collective_ok(dist, tm):
            dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        else:
            c = tm.cpu(); dist.all_reduce(c, op=dist.ReduceOp.MAX); tm.copy_(c)
    total_ms, launch_ms = float(tm[0]), float(tm[1])
    step_ms = [float(x) for x in tm[2:]]
    value = n_u * args.steps / (total_ms * 1e-3) / 1e9

    # dominant kernel = the TDBP launch: algorithmic terms per launch / its average duration
    props = torch.cuda.get_device_properties(dev)
    sms = props.multi_processor_count
    peak = roof_terms_per_s(E, sms, 1.965e9) / 1e9
    terms_per_launch = nu_local                                       # this rank's launch
    achieved = terms_per_launch / (launch_ms * 1e-3) / 1e9            # per GPU, vs the per-GPU peak

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        img_bytes = g["nx"] * g["ny"] * g["nz"] * 8
        nav_bytes = (P * 3 + P * E * 3 + P) * 8
        if world == 1:
            pinned = torch.from_numpy(echoes_h).pin_memory()
            host_img = torch.empty(bp.shape, dtype=torch.complex64).pin_memory()
            bp_h = pkg.Backprojector(s.fc, s.bandwidth, s.fs, s.c, g)
            bp_h.form_streamed(pinned, s.tx, s.rx, s.t0, out=host_img)  # warm
            ts = []
            for _ in range(max(1, min(args.steps, 3))):
                t0w = time.perf_counter()
                bp_h.form_streamed(pinned, s.tx, s.rx, s.t0, out=host_img)
                ts.append(time.perf_counter() - t0w)
            bp_h.close()
            e2e_s = statistics.mean(ts)
            e2e = {"value": n_u / e2e_s / 1e9, "unit": UNIT, "h2d_bytes_per_step": P * E * Ns * 8 + nav_bytes,
                   "d2h_bytes_per_step": img_bytes, "ms_per_step": e2e_s * 1e3,
                   "api": "sas_bp_form_streamed(pinned host echoes -> chunked H2D overlapped with "
                          "accumulating TDBP launches -> image to pinned host)"}
        else:
            host_img = torch.empty((g["nz"], g["ny"], g["nx"]), dtype=torch.complex64).pin_memory() if rank == 0 else None
            if shard == "image":
                lo_p, hi_p = sl[rank]
                local_h = torch.zeros((per, E, Ns), dtype=torch.complex64)
                local_h[: hi_p - lo_p] = torch.from_numpy(echoes_h[lo_p:hi_p])
                local_h = local_h.pin_memory()
                local_d = torch.empty((per, E, Ns), dtype=torch.complex64, device=dev)
            else:
                local_h = torch.from_numpy(my_h).pin_memory()
            ts = []
            for it in range(max(1, min(args.steps, 3)) + 1):
                barrier()
                t0w = time.perf_counter()
                if shard == "image":
                    # rank-local 1/G H2D, NCCL all-gather of the ping set, band, gather to rank 0
                    local_d.copy_(local_h, non_blocking=True)
                    if _collective_ok(dist, local_d):
                        pdist.gather_echoes(local_d, full_pad, dist)
                    else:
                        fp = torch.empty(full_pad.shape, dtype=full_pad.dtype)
                        pdist.gather_echoes(local_d.cpu(), fp, dist)
                        full_pad.copy_(fp)
                    bp.form_device(img, stream=stream)
                    combine()
                    if rank == 0:
                        host_img.copy_(full_img, non_blocking=True)
                else:
                    # rank-local H2D of its own pings, full grid, NCCL reduce to rank 0
                    echoes_d.copy_(local_h, non_blocking=True)
                    bp.form_device(img, stream=stream)
                    combine()
                    if rank == 0:
                        host_img.copy_(img, non_blocking=True)
                torch.cuda.synchronize()
                dt = torch.tensor([time.perf_counter() - t0w], dtype=torch.float64, device=dev)
                if _collective_ok(dist, dt):
                    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
                else:
                    c = dt.cpu(); dist.all_reduce(c, op=dist.ReduceOp.MAX); dt.copy_(c)
                if it > 0:
                    ts.append(float(dt[0]))
            e2e_s = statistics.mean(ts)
            e2e = {"value": n_u / e2e_s / 1e9, "unit": UNIT, "h2d_bytes_per_step": P * E * Ns * 8,
                   "d2h_bytes_per_step": img_bytes, "ms_per_step": e2e_s * 1e3,
                   "api": ("per rank: pinned H2D of its 1/G ping slice + NCCL all-gather + sas_bp_form_device "
                           "on its band + NCCL gather to rank 0 + D2H" if shard == "image" else
                           "per rank: pinned H2D of its pings r::G + sas_bp_form_device (full grid) + "
                           "NCCL reduce to rank 0 + D2H")}

    # ---- NEXT-1: the same workload gated to the transmit beam (generator's FWHM), ray culling on
    gated = None
    if not args.no_gated and world == 1 and s.sin_half_beam > 0:
        az = 2 * float(np.arcsin(s.sin_half_beam))
        bp.set_beam(az, 0.0, False, True)
        _, g_terms = bp.count_terms()
        for _ in range(2):
            bp.form_device(img, stream=stream)
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            bp.form_device(img, stream=stream)
        g1.record(stream)
        torch.cuda.synchronize()
        g_ms = g0.elapsed_time(g1) / args.steps
        bp.set_beam(None)
        gated = {"beam": f"azimuth FWHM {az:.4f} rad at tx (monostatic), ray culling on", "ms_per_step": g_ms,
                 "speedup_vs_dense": (total_ms / args.steps) / g_ms, "in_cone_terms": g_terms,
                 "in_cone_fraction": g_terms / dense, "in_cone_Gterm_per_s": g_terms / (g_ms * 1e-3) / 1e9,
                 "dense_equivalent_Gterm_per_s": dense / (g_ms * 1e-3) / 1e9}

    # ---- K1 range compression on the same channel layout (row a1), reported separately
    k1 = None
    if not args.no_k1 and rank == 0:
        fsr, Br, Tp = s.fs, s.bandwidth, (2e-3 if g["nz"] > 1 else 5e-3)   # SURVEY §8(a) a1 replicas
        nr = int(round(Tp * fsr))
        tt = np.arange(nr) / fsr - Tp / 2
        rep = np.exp(1j * np.pi * (Br / Tp) * tt ** 2).astype(np.complex64)
        rep_d = torch.from_numpy(rep / np.float32(np.sqrt(nr))).to(dev)
        out_d = torch.empty_like(echoes_d)
        k1_ms = time_short_kernel(lambda: pkg.rangecompress_device(echoes_d, rep_d, out_d, stream=stream), stream)
        k1_bytes = 16 * P * E * Ns
        hbm = _measured_hbm()
        k1 = {"kernel": ("rc_pipe_kernel<PACK> (bulk-staged persistent overlap-save, L=4096, %d records per transform)"
                         % (4096 // (Ns + nr - 1)) if Ns + nr - 1 <= 2048 else
                         "rc_pipe_kernel (bulk-staged persistent overlap-save, L=4096)"), "Nr": nr, "ms": k1_ms,
              "achieved": k1_bytes / (k1_ms * 1e-3) / 1e9, "unit": "GB/s", "bound": "hbm", "peak": hbm[0],
              "peak_source": hbm[1], "frac": k1_bytes / (k1_ms * 1e-3) / 1e9 / hbm[0],
              "algorithmic_bytes": k1_bytes, "note": "16 B per sample: read raw + write compressed once",
              "traffic": _profile_traffic(f"ncu_k1_cfg{args.config}.json", args.config)}
        del out_d

    # ---- NEXT-4: spreading-weighted K2 on the same workload; K1b x4 upsampling and K0 basebanding
    # on the same channel layout (cfg-2 channels recorded at fs/4, resp. real passband at 4 fs)
    next4 = None
    if not args.no_next4 and rank == 0 and world == 1:
        def _time(fn, nrep, long_launch=False):
            if long_launch:   # the weighted K2 step: long launches, plain event timing
                for _ in range(2):
                    fn()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                for _ in range(nrep):
                    fn()
                b.record(stream)
                torch.cuda.synchronize()
                return a.elapsed_time(b) / nrep
            return time_short_kernel(fn, stream)
        hbm = _measured_hbm()
        bp.set_weighting(True)
        w_ms = _time(lambda: bp.form_device(img, stream=stream), min(args.steps, 2), long_launch=True)
        bp.set_weighting(False)
        nch = P * E
        ns_in = Ns // 4
        up_in = echoes_d.view(-1)[: nch * ns_in].view(nch, ns_in)
        up_out = torch.empty((nch, 4 * ns_in), dtype=torch.complex64, device=dev)
        up_ms = _time(lambda: pkg.upsample_device(up_in, 4, up_out, stream=stream), 5)
        up_bytes = 8 * nch * ns_in * (1 + 4)
        del up_out
        nin = 4 * Ns
        pb = torch.randn((P, E, nin), dtype=torch.float32, device=dev)
        bb_out = torch.empty((P, E, Ns), dtype=torch.complex64, device=dev)
        kk = np.arange(-31, 32)
        hbb = (2 * 0.1 * np.sinc(2 * 0.1 * kk) * (0.5 + 0.5 * np.cos(np.pi * kk / 32))).astype(np.float32)
        hbb *= np.float32(2.0 / hbb.sum())
        t0_d = torch.from_numpy(np.ascontiguousarray(s.t0, dtype=np.float64)).to(dev)
        hbb_d = torch.from_numpy(hbb).to(dev)
        bb_ms = _time(lambda: pkg.baseband_device(pb, 4 * s.fs, s.fc, t0_d, hbb_d, 4, bb_out, stream=stream), 5)
        bb_bytes = 4 * nch * nin + 8 * nch * Ns
        del pb, bb_out
        # whitening (R21): gain estimate (M = 64 periodogram over the whole batch) and the
        # whitened compression (one K1 pass with the composed Nr + 63-tap filter)
        Mw = 64
        Gw = torch.empty(Mw, dtype=torch.float32, device=dev)
        wg_ms = _time(lambda: pkg.whitening_gain_device(echoes_d, Mw, 0.0, Gw, stream=stream), 3)
        tt = np.arange(600) / s.fs - 2.5e-3
        rep_w = torch.from_numpy((np.exp(1j * np.pi * (s.bandwidth / 5e-3) * tt ** 2) / np.sqrt(600)).astype(np.complex64)).to(dev)
        wout = torch.empty_like(echoes_d)
        wc_ms = _time(lambda: pkg.rangecompress_whitened_device(echoes_d, rep_w, Gw, wout, stream=stream), 5)
        del wout
        next4 = {
            "weighted_k2": {"what": "TDBP with the spreading weight R_tx R_rx (R18), same workload",
                            "ms_per_step": w_ms, "Gterm_per_s": dense / (w_ms * 1e-3) / 1e9,
                            "frac": dense / (w_ms * 1e-3) / 1e9 / peak,
                            "slowdown_vs_unweighted": w_ms / (total_ms / args.steps)},
            "k1b_upsample": {"kernel": "upsample_kernel<4> (8-tap Lanczos, x4)",
                             "shape": f"{nch} channels x {ns_in} -> {4 * ns_in} samples", "ms": up_ms,
                             "algorithmic_bytes": up_bytes, "achieved": up_bytes / (up_ms * 1e-3) / 1e9,
                             "unit": "GB/s", "bound": "hbm", "peak": hbm[0], "peak_source": hbm[1],
                             "frac": up_bytes / (up_ms * 1e-3) / 1e9 / hbm[0],
                             "note": "8 B read + 32 B written per input sample"},
            "whitening": {"gain_kernel": "wh_periodogram_reg_kernel<4> (M = 64: 16-point register DFT x radix-4 across "
                                         "4 lanes per block) + wh_gain_kernel",
                          "gain_ms": wg_ms, "gain_GB_per_s": 8 * nch * Ns / (wg_ms * 1e-3) / 1e9,
                          "gain_frac_hbm": 8 * nch * Ns / (wg_ms * 1e-3) / 1e9 / hbm[0],
                          "whitened_k1_ms": wc_ms,
                          "whitened_k1_GB_per_s": 16 * nch * Ns / (wc_ms * 1e-3) / 1e9,
                          "note": "gain: 8 B read per sample; whitened K1: 16 B per sample, Nr + M - 1 = 663 taps"},
            "k0_baseband": {"kernel": "baseband_ctap_kernel (complex taps on the real samples, polyphase, fp64 phase reduction)",
                            "shape": f"{nch} channels x {nin} real @ {4 * s.fs / 1e3:.0f} kHz -> {Ns} complex, D=4, "
                                     f"Nh={hbb.size}", "ms": bb_ms, "algorithmic_bytes": bb_bytes,
                            "achieved": bb_bytes / (bb_ms * 1e-3) / 1e9, "unit": "GB/s", "bound": "hbm",
                            "peak": hbm[0], "peak_source": hbm[1], "frac": bb_bytes / (bb_ms * 1e-3) / 1e9 / hbm[0],
                            "note": "4 B read per passband sample + 8 B written per baseband sample"},
        }

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_oracle_rate(s, echoes_h, args.cpu_seconds)
        cpu["cpu_model"] = host_cpu_model()

    if rank == 0:
        traffic = _profile_traffic(f"ncu_tdbp_cfg{args.config}.json", args.config)
        last3 = step_ms[-3:]
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded synth/ forward model)",
            "config": {"workload": workload_name(args.config, s),
                       "terms_per_step": n_u, "dense_terms_per_step": dense,
                       "denominator": "N_u = terms whose interpolation support meets the record (K3, SURVEY §8(d))",
                       "parallelism": f"{shard}-shard x{world}" if world > 1 else "single GPU",
                       "l2": (f"inputs larger than L2 ({P * E * Ns * 8 / 1e9:.2f} GB echoes, 126 MB L2), no flush"
                              if P * E * Ns * 8 > 126e6 else
                              f"inputs SMALLER than L2 ({P * E * Ns * 8 / 1e6:.1f} MB): not a timing config")},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": UNIT, "frac": achieved / peak,
                         "traffic": traffic,
                         "algorithmic_bytes": P * E * Ns * 8 + g["nx"] * g["ny"] * g["nz"] * 8,
                         "peak_basis": f"{sms} SMs x 1965 MHz x min(128/F, 16/S), F=20+6/E, S=3+1/E, E={E} "
                                       "(FP32/SFU roofline of the direct per-term formula, BASELINE.md)",
                         "peak_sfu_2mufu": sms * 1.965e9 * 8 / 1e9,
                         "frac_sfu_2mufu": achieved / (sms * 1.965e9 * 8 / 1e9)},
            "clocks": clk.summary(),
            "gpu_launches": args.steps,   # one tdbp_kernel launch per timed step
            "step_ms": step_ms,
            "paper_protocol": {"what": "process three times and report the last (P:338)", "runs_ms": last3,
                               "value_last": n_u / (last3[-1] * 1e-3) / 1e9,
                               "median_of_steps": n_u / (statistics.median(step_ms) * 1e-3) / 1e9},
            "e2e": e2e,
            "cpu_baseline": cpu,
            "k1_rangecompress": k1,
            "next1_gated": gated,
            "next4": next4,
        }
        if cpu:
            out["gpu_over_cpu"] = value / cpu["value"]
        print(json.dumps(out), flush=True)
    bp.close()
    if world > 1:
        dist.destroy_process_group()
    return 0




def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_sasbp(args)


if __name__ == "__main__":
    sys.exit(main())
