"""cfg4 at 2^18: where do the device and oracle bases diverge at step 1?"""
import sys, os
sys.path.insert(0, "."); sys.path.insert(0, "oracle"); sys.path.insert(0, "tests")
import numpy as np
import pyoracle as po
from harness import sin_angle
from paper_2603_19439_b200 import TrackerSession, streams

s = streams.config4(n=1 << 18, steps=2)
rp, col, val = s.csr0()
n = len(rp) - 1
k = 64
g = TrackerSession.tracker_init(rp, col, val, k, kind="grest-rsvd", seed=0)
v0, x0 = g.embedding()
print("init values head/tail", v0[:3], v0[-3:])
o = po.Session(po.Csr(n, rp, col, val), kind="grest-rsvd", k=k, seed=0, values=v0, vectors=x0)
u0, u1 = s.updates
g.step(u0); o.step(u0)
gv, gx = g.embedding(); ov, ox = o.embedding()
print("step0 vals err", np.abs(gv - ov).max(), "sin", sin_angle(gx, ox))
print("step0 values", gv[60:64], "gaps", np.diff(np.abs(gv))[58:63])
n1 = n + u0.n_new
seed = po.mix_seed(po.mix_seed(0, 0x6b7a), 1)
zg = g.probe_basis(u1, "grest-rsvd", seed)
zo = o.probe_basis(u1, "grest-rsvd", seed)
print("D gpu", zg.shape, "D oracle", zo.shape)
m = min(zg.shape[1], zo.shape[1])
for c0 in range(0, m, 8):
    print("cols", c0, c0 + 8, "sin", sin_angle(zg[:, :c0 + 8], zo[:, :c0 + 8]))
print("full sin", sin_angle(zg, zo), sin_angle(zo, zg))
# rr on the same basis
vg, xg = g.probe_rr(u1, zo)
vo, xo = o.probe_rr(u1, zo)
print("rr on oracle basis: val err", np.abs(vg - vo).max() / np.abs(vo).max(), "sin", sin_angle(xg, xo))
g.step(u1); o.step(u1)
gv, gx = g.embedding(); ov, ox = o.embedding()
print("step1 per-value err", np.max(np.abs(gv - ov) / np.abs(ov)), "sin", sin_angle(gx, ox))
print("values gpu", gv[-4:], "oracle", ov[-4:])
