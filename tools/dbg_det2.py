import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2603_19439_b200 import TrackerSession, streams
s = streams.config1(n=3000, steps=0)
rp, col, val = s.csr0()
x = np.linalg.qr(np.random.default_rng(0).standard_normal((len(rp) - 1, 8)))[0]
g = TrackerSession(rp, col, val, np.arange(8.0, 0, -1), x, kind="grest-rsvd", k=8)
for m1, m2 in [(148, 76), (148, 65), (128, 76)]:
    print(m1, m2, g.determinism(1, 20000, m1, m2, 30), flush=True)
