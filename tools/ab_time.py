"""A/B timing of libsasbp.so variants on BASELINE configs (same box, interleaved).

    python tools/ab_time.py --libs build_ab/a.so build_ab/b.so --configs 4:200 2:250 [--reps 2] [--forms 3]
    python tools/ab_time.py --child LIB CFG PINGS FORMS      (one measurement, internal)

A config "C:P" keeps the first P pings of BASELINE config C (same grid, elements, samples and
plan) with seeded device-random echoes (the TDBP work is data independent).  Prints one line per
(rep, config, lib): ms per form (mean of FORMS CUDA-event-timed launches after one warm-up) and
Gterm/s.  Timing only; never a bench value."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(lib, cfg, pings, forms, env_extra=None):
    sys.path.insert(0, ROOT)
    import torch
    import synth
    import paper_2101_05888_b200 as pkg
    pkg.load_library(lib)
    s = synth.scenario(cfg)
    P = pings if pings > 0 else s.P
    gen = torch.Generator(device="cuda").manual_seed(1000 + cfg)
    e = torch.randn((P, s.E, s.Ns), dtype=torch.complex64, device="cuda", generator=gen)
    bp = pkg.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid)
    bp.set_pings_device(e, s.tx[:P], s.rx[:P], s.t0[:P])
    img = torch.empty(bp.shape, dtype=torch.complex64, device="cuda")
    bp.form_device(img)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(forms):
        bp.form_device(img)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / forms
    try:   # clocks / power right after the timed forms (a throttled box shows here)
        q = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                            "--format=csv,noheader"], capture_output=True, text=True, timeout=20).stdout.strip()
    except Exception:
        q = ""
    terms = bp.shape[0] * bp.shape[1] * bp.shape[2] * P * s.E
    print(json.dumps({"lib": lib, "config": cfg, "pings": P, "ms": ms, "Gterm_per_s": terms / ms / 1e6,
                      "plan": bp.plan(), "smi": q}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", nargs="+", default=[])
    ap.add_argument("--configs", nargs="+", default=["4:200"])
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--forms", type=int, default=3)
    ap.add_argument("--child", nargs=4)
    a = ap.parse_args()
    if a.child:
        lib, cfg, pings, forms = a.child
        child(lib, int(cfg), int(pings), int(forms))
        return
    for rep in range(a.reps):
        for c in a.configs:
            cfg, pings = (int(x) for x in c.split(":"))
            for spec in a.libs:
                # "path.so" or "path.so,VAR=value,..." (environment of that variant's run)
                lib, *envs = spec.split(",")
                env = dict(os.environ, **dict(e.split("=", 1) for e in envs))
                r = subprocess.run([sys.executable, __file__, "--child", lib, str(cfg), str(pings), str(a.forms)],
                                   capture_output=True, text=True, timeout=900, env=env)
                line = [l for l in r.stdout.splitlines() if l.startswith("{")]
                if not line:
                    print(f"rep {rep} cfg {c} {spec}: FAILED {r.stderr[-400:]}", flush=True)
                    continue
                d = json.loads(line[0])
                print(f"rep {rep} cfg {c} {os.path.basename(spec):36s} {d['ms']:9.2f} ms  {d['Gterm_per_s']:8.1f} Gterm/s  "
                      f"occ {d['plan']['ctas_per_sm']}  [{d.get('smi', '')}]", flush=True)


if __name__ == "__main__":
    main()
