"""Determinism of the device tracker_init: the same graph twice in one process."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 0
if len(sys.argv) > 4:
    import pyoracle  # noqa
import numpy as np
from paper_2603_19439_b200 import TrackerSession, streams

s = streams.config4(n=n, steps=steps)
rp, col, val = s.csr0()
print("graph", len(rp) - 1, rp[-1], hash(col.tobytes()), flush=True)
for r in range(reps):
    try:
        g = TrackerSession.tracker_init(rp, col, val, 64, kind="grest-rsvd", seed=0, max_restarts=60)
        v, x = g.embedding()
        print(r, "restarts/products", g.init_stats(), "vals", v[:2], v[-2:], "res", g.residual_norms().max(), flush=True)
        g.close()
    except Exception as e:
        print(r, "ERR", e, flush=True)
