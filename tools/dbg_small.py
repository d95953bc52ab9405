import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import synth, oracle
import paper_2101_05888_b200 as pkg
s = synth.scenario(1)
e = s.echoes()
with pkg.Backprojector(s.fc, s.bandwidth, s.fs, s.c, s.grid) as bp:
    bp.set_pings(e, s.tx, s.rx, s.t0)
    print(bp.plan())
    img = bp.form()
ref = oracle.tdbp_grid(e, s.tx, s.rx, s.t0, s.fc, s.fs, s.c, s.grid)
print("err", np.abs(img-ref).max()/np.abs(ref).max())
