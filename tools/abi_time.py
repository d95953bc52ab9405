"""K2 timing of historical libsasbp.so builds through the C ABI only (sas_bp_create /
sas_bp_set_pings_device / sas_bp_form_device, unchanged since round 1), so builds of older commits
can be compared with the current one on the same box.  Seeded device-random echoes of config C's
first P pings.  Timing only; never a bench value.
    python tools/abi_time.py --libs a.so b.so --configs 2:250 4:100 [--reps 2] [--forms 3]"""
import argparse
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(lib, cfg, pings, forms):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import synth
    from paper_2101_05888_b200.sasbp import make_grid
    L = ctypes.CDLL(lib)
    s = synth.scenario(cfg)
    P = pings if pings > 0 else s.P
    gen = torch.Generator(device="cuda").manual_seed(1000 + cfg)
    e = torch.randn((P, s.E, s.Ns), dtype=torch.complex64, device="cuda", generator=gen)
    g = make_grid(s.grid)
    h = ctypes.c_void_p()
    f64 = lambda a: np.ascontiguousarray(a, dtype=np.float64)
    tx, rx, t0 = f64(s.tx[:P]), f64(s.rx[:P]), f64(s.t0[:P])
    dp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    L.sas_bp_create.argtypes = [ctypes.c_double] * 4 + [ctypes.c_void_p, ctypes.c_void_p]
    assert L.sas_bp_create(s.fc, s.bandwidth, s.fs, s.c, ctypes.byref(g), ctypes.byref(h)) == 0
    L.sas_bp_set_pings_device.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.c_int32] + [ctypes.POINTER(ctypes.c_double)] * 3 + [ctypes.c_void_p]
    st = torch.cuda.current_stream()
    assert L.sas_bp_set_pings_device(h, ctypes.c_void_p(e.data_ptr()), P, s.E, s.Ns, dp(tx), dp(rx), dp(t0),
                                     ctypes.c_void_p(st.cuda_stream)) == 0
    img = torch.empty((s.grid["nz"], s.grid["ny"], s.grid["nx"]), dtype=torch.complex64, device="cuda")
    L.sas_bp_form_device.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
    form = lambda: L.sas_bp_form_device(h, ctypes.c_void_p(img.data_ptr()), ctypes.c_void_p(st.cuda_stream), 0)
    assert form() == 0
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(forms):
        form()
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / forms
    terms = s.grid["nx"] * s.grid["ny"] * s.grid["nz"] * P * s.E
    print(f"{ms:.2f} {terms / (ms * 1e-3) / 1e9:.1f}")


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]))
        return
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", nargs="+", required=True)
    ap.add_argument("--configs", nargs="+", default=["2:250"])
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--forms", type=int, default=3)
    a = ap.parse_args()
    for rep in range(a.reps):
        for cp in a.configs:
            cfg, pings = (int(v) for v in cp.split(":"))
            for lib in a.libs:
                out = subprocess.run([sys.executable, __file__, "--child", lib, str(cfg), str(pings), str(a.forms)],
                                     capture_output=True, text=True)
                res = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else "FAILED " + out.stderr[-300:]
                print(f"rep {rep} cfg {cfg}:{pings} {lib:40s} {res}", flush=True)


if __name__ == "__main__":
    main()
