import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["STG_EIG_PROF"] = "1"
import paper_2603_19439_b200 as m
rng = np.random.default_rng(0)
for n, want in ((164, 32), (200, 100), (228, 64)):
    g = rng.standard_normal((n, n)); s = g + g.T
    for _ in range(2):
        m.sym_eig_dense(s, "abs_desc", want)
    b = rng.standard_normal((n, 3 * n)) * np.logspace(0, -8, n)[:, None]
    for _ in range(2):
        m.sym_eig_dense(b @ b.T, "alg_desc", want)
