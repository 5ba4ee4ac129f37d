"""CPU checks of the config-5 stream generator (torch, run here on the CPU
device): the batches are valid edit lists for assemble_update
(proj/src/graph.cpp:45-100) and follow the config's rules."""
import numpy as np

import pyoracle as po
from paper_2603_19439_b200 import streams


def _keys(i, j):
    lo, hi = np.minimum(i, j), np.maximum(i, j)
    return lo.astype(np.int64) * (1 << 32) + hi


def test_config5_generator_rules_and_oracle_accepts():
    s = streams.config5(scale=12, steps=3, device="cpu")
    rp, col, val = s.csr0()
    n = s.n0
    assert n == 4096 and rp[-1] == len(col) == s.nnz0
    rows = np.repeat(np.arange(n), np.diff(rp))
    present = set(_keys(rows, col).tolist())
    assert np.all(rows != col)  # no self-loops
    k_csr = rows.astype(np.int64) * (1 << 32) + col
    assert np.all(np.diff(k_csr) > 0)  # sorted, deduplicated
    assert len(present) * 2 == len(col)  # symmetric
    m = len(present)
    cur = n
    a = po.Csr(n, rp, col, val)
    for u in s.updates:
        ai, aj, aw = u.added
        ka = _keys(ai, aj)
        assert len(ka) == m // 1000 and len(np.unique(ka)) == len(ka)
        assert not any(x in present for x in ka.tolist())
        assert np.all(ai < aj) and np.all(aj < cur) and np.all(aw == 1.0)
        assert len(u.removed[0]) == 0 and u.n_new == cur // 1000
        ni, nj, _ = u.new_edges
        assert np.all(nj >= cur) and np.all(ni < cur)  # old <-> new, preferential attachment to pre-step nodes
        assert np.all(np.bincount(nj - cur, minlength=u.n_new) == 16)
        kn = _keys(ni, nj)
        assert len(np.unique(kn)) == len(kn)
        a = po.apply_update(a, u)  # assemble_update + apply_update (the reference validation) accept the batch
        present.update(ka.tolist())
        present.update(kn.tolist())
        m = len(present)
        cur += u.n_new
    assert a.n == cur and a.nnz == 2 * m
