import sys, hashlib
sys.path.insert(0, "."); sys.path.insert(0, "oracle"); sys.path.insert(0, "tests")
import numpy as np
import pyoracle as po
from harness import sin_angle
from paper_2603_19439_b200 import TrackerSession, streams
s = streams.config4(n=1 << 18, steps=2)
rp, col, val = s.csr0()
print("md5", hashlib.md5(rp.tobytes() + col.tobytes() + val.tobytes()).hexdigest(), rp.dtype, col.dtype, val.dtype, flush=True)
for rep in range(2):
    try:
        g = TrackerSession.tracker_init(rp, col, val, 64, kind="grest-rsvd", seed=0, max_restarts=int(sys.argv[1]))
        print(rep, "ok", g.init_stats(), flush=True)
    except Exception as e:
        print(rep, "ERR", e, flush=True)
