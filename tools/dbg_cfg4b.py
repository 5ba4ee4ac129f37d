import sys
sys.path.insert(0, "."); sys.path.insert(0, "oracle"); sys.path.insert(0, "tests")
import numpy as np
from harness import sin_angle  # noqa  (same imports as dbg_cfg4)
from paper_2603_19439_b200 import TrackerSession, streams
s = streams.config4(n=1 << 18, steps=2)
rp, col, val = s.csr0()
for rep in range(2):
    for cus in (False, True):
        try:
            g = TrackerSession.tracker_init(rp, col, val, 64, kind="grest-rsvd", seed=0, max_restarts=40, cusolver_eig=cus)
            print(rep, "cusolver" if cus else "device", g.init_stats(), g.residual_norms().max(), flush=True)
            g.close()
        except Exception as e:
            print(rep, "cusolver" if cus else "device", "ERR", str(e)[:120], flush=True)
