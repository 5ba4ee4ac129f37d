import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2603_19439_b200 import TrackerSession, streams
s = streams.config1(n=3000, steps=0)
rp, col, val = s.csr0()
x = np.linalg.qr(np.random.default_rng(0).standard_normal((len(rp) - 1, 8)))[0]
g = TrackerSession(rp, col, val, np.arange(8.0, 0, -1), x, kind="grest-rsvd", k=8)
N = 20000
tot = 0
for m1, m2 in [(148, 76), (128, 76), (150, 100), (200, 100), (148, 65), (64, 76), (100, 100), (164, 164)]:
    d = g.determinism(1, N, m1, m2, 20)
    tot += d > 0
    print(m1, m2, "rerun diff", d, flush=True)
for m1, m2 in [(148, 148), (76, 76), (200, 200), (32, 200), (64, 100)]:
    d = g.determinism(0, N, m1, m2, 20)
    tot += d > 0
    print("gram", m1, m2, "rerun diff", d, flush=True)
print("nondeterministic shapes:", tot)
