"""Runs a few G-REST steps of config 3 for profiling (ncu launch lists and
per-kernel deep dives). X0 is a random orthonormal basis: the step's kernels
and shapes do not depend on its quality, and no torch kernels pollute the list."""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2603_19439_b200 import TrackerSession, streams  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=20)
ap.add_argument("--config", default="cfg3", choices=["cfg3", "cfg4"])
ap.add_argument("--n", type=int, default=1 << 22, help="cfg4 node count")
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--k", type=int, default=32)
ap.add_argument("--real-x0", action="store_true", help="leading eigenpairs (as bench.py) instead of a random basis")
ap.add_argument("--device-edits", action="store_true", help="edit lists resident in HBM (st_step_device, as bench.py)")
args = ap.parse_args()

if args.config == "cfg4":
    s = streams.config4(n=args.n, steps=args.warmup + args.steps)
else:
    s = streams.config3(scale=args.scale, steps=args.warmup + args.steps)
rp, col, val = s.csr0()
n = len(rp) - 1
if args.real_x0:
    g0 = TrackerSession.tracker_init(rp, col, val, args.k, kind="grest-rsvd", seed=0)  # device Lanczos
    vals, x = g0.embedding()
    g0.close()
else:
    x, _ = np.linalg.qr(np.random.default_rng(0).standard_normal((n, args.k)))
    vals = np.linspace(100.0, 10.0, args.k)
g = TrackerSession(rp, col, val, vals, x, kind="grest-rsvd", k=args.k, seed=0, timing=True,
                   kernel_timing=bool(os.environ.get("STG_KLOG")), cusolver_eig=bool(os.environ.get("STG_CUSOLVER")))
if args.device_edits:
    from paper_2603_19439_b200 import DeviceUpdate  # noqa: E402
    dev = [DeviceUpdate(u, device="cuda:0") for u in s.updates]
for t, u in enumerate(s.updates):
    t0 = time.perf_counter()
    if args.device_edits:
        g.step_device(dev[t])
    else:
        g.step(u)
    print(f"step {t}: {1e3 * (time.perf_counter() - t0):.2f} ms wall, phases {np.round(g.timings(), 3).tolist()}, "
          f"launches {g.launches()}", flush=True)
