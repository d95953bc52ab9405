import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import oracle, synth
import paper_2101_05888_b200 as pkg
r = synth.random_case(21, P=2, E=2, Ns=512, n=(9, 9, 3))
g = r["grid"]
tx = r["tx"].copy(); rx = r["rx"].copy()
tx[0] = oracle.grid_points(g, np.array([[4, 4, 1]]))[0]
rx[1, 0] = oracle.grid_points(g, np.array([[2, 6, 1]]))[0]
bp = pkg.Backprojector(r["fc"], r["fs"] / 4, r["fs"], r["c"], g)
bp.set_pings(r["echoes"], tx, rx, np.zeros(2))
print(bp.plan())
img = bp.form()
print(np.isfinite(img).all())
