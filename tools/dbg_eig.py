"""Device sym_eig_dense on a clustered spectrum (SBM-like: one outlier, a
63-fold near-degenerate cluster, a bulk): residuals, orthogonality and
run-to-run determinism."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2603_19439_b200 import sym_eig_dense

rng = np.random.default_rng(0)
for n, want in ((148, 76), (164, 32), (228, 64)):
    lam = np.concatenate([[33.0], rng.uniform(26.47, 27.16, 63), rng.uniform(-11, 11, n - 64)])
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    m = (q * lam) @ q.T
    m = 0.5 * (m + m.T)
    ref = np.sort(np.abs(lam))[::-1]
    outs = []
    for rep in range(5):
        w, v = sym_eig_dense(m, "abs_desc", want)
        res = np.abs(m @ v - v * w[:want]).max()
        orth = np.abs(v.T @ v - np.eye(want)).max()
        outs.append((w.copy(), v.copy()))
        print(n, want, rep, "res", res, "orth", orth, "val err", np.abs(np.abs(w) - ref).max(), flush=True)
    same = all(np.array_equal(outs[0][1], o[1]) for o in outs[1:])
    print(n, "deterministic:", same)
