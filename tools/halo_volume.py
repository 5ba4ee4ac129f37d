"""Boundary-row halo volume of the row-sharded step (VERDICT r01
item 5): for R ranks, the rows of P each rank's owned Delta rows reference on
other ranks (what the alltoallv halo moves) against the rows the former
allgather moved (every rank's rows of P). Host arithmetic on the first update
of the stream, with the library's ownership map (shard_bounds + round-robin
chunks of appended ids)."""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_19439_b200 import streams  # noqa: E402
from paper_2603_19439_b200.shard import shard_bounds  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg5")
ap.add_argument("--scale", type=int, default=25)
ap.add_argument("--ranks", type=int, nargs="+", default=[2, 4, 8])
ap.add_argument("--chunk", type=int, default=1024)
ap.add_argument("--k", type=int, default=32)
args = ap.parse_args()

if args.config == "cfg5":
    s = streams.config5(scale=args.scale, steps=1, device="cuda:0")
else:
    s = streams.config3(scale=args.scale, steps=1)
rp, col, val = s.csr0()
n = len(rp) - 1
u = s.updates[0]
ai, aj = (np.asarray(x, np.int64) for x in u.added[:2])
ri, rj = (np.asarray(x, np.int64) for x in u.removed)
ni, nj = (np.asarray(x, np.int64) for x in u.new_edges[:2])
rows = np.concatenate([ai, aj, ri, rj, ni, nj])
cols = np.concatenate([aj, ai, rj, ri, nj, ni])
S = int(u.n_new)
n_total = n + S
P = np.unique(np.concatenate([rows, np.arange(n, n_total)]))
nnz = len(rows)
out = {"config": args.config, "scale": args.scale, "n": n, "nnz_delta": int(nnz), "P": int(len(P)), "S": S, "ranks": {}}
for R in args.ranks:
    b = shard_bounds(rp, R)

    def owner(g):
        o = np.searchsorted(b, g, side="right") - 1
        app = g >= n
        o[app] = ((g[app] - n) // args.chunk) % R
        return o

    orow, ocol = owner(rows), owner(cols)
    halo_rows = []
    for r in range(R):
        m = (orow == r) & (ocol != r)
        halo_rows.append(len(np.unique(cols[m])))
    p_own = np.bincount(owner(P), minlength=R)
    per = {"halo_rows_max": int(max(halo_rows)), "halo_rows_mean": float(np.mean(halo_rows)),
           "allgather_rows": int(len(P)), "p_rows_max": int(p_own.max()),
           "bound_nnz_over_R": int(nnz // R)}
    for m_ in (args.k, 164, 200):
        per[f"halo_MB_m{m_}_max"] = 8 * m_ * per["halo_rows_max"] / 1e6
        per[f"allgather_MB_m{m_}"] = 8 * m_ * len(P) / 1e6
    out["ranks"][R] = per
print(json.dumps(out, indent=1))
