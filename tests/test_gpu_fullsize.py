"""BASELINE config 3 at its full size (R-MAT s20: 1,048,576 nodes, 31.4M stored
entries, k = 32, grest-rsvd L = P = 100; per step 1% new nodes with 10
preferential-attachment edges and 0.5% deletions). One oracle step takes ~25 s
on 16 threads, so instead of the oracle these tests check size-independent
properties of the reference's algebra at the full size:

* apply_update (proj/src/graph.cpp:102-115): the device CSR equals, bit for
  bit, the CSR built on the host from the edge set with the step's edits
  applied (set algebra on sorted keys);
* rayleigh_ritz_step (proj/src/trackers.cpp:282-308) on the projected
  operator of Eq. (14), A~ = X-bar Lambda X-bar' + Delta: the new vectors are
  orthonormal, each Ritz value is the Rayleigh quotient x' A~ x, the
  Rayleigh-Ritz residual A~ X - X Theta is orthogonal to span(X) (it is
  orthogonal to the whole basis Z), and the values are in spectral order
  (abs_desc, types.hpp:26-40).
"""
import numpy as np
import pytest

from paper_2603_19439_b200 import TrackerSession, init_eig, streams


def _delta(upd, n_total, device):
    import torch

    ai, aj, aw = (np.asarray(x) for x in upd.added)
    ri, rj = (np.asarray(x) for x in upd.removed)
    ni, nj, nw = (np.asarray(x) for x in upd.new_edges)
    i = np.concatenate([ai, aj, ri, rj, ni, nj]).astype(np.int64)
    j = np.concatenate([aj, ai, rj, ri, nj, ni]).astype(np.int64)
    v = np.concatenate([aw, aw, -np.ones(len(ri)), -np.ones(len(ri)), nw, nw]).astype(np.float64)
    return torch.sparse_coo_tensor(torch.as_tensor(np.stack([i, j])), torch.as_tensor(v),
                                   (n_total, n_total)).coalesce().to(device)


@pytest.mark.gpu
def test_config3_full_size_properties():
    import torch

    dev = "cuda:0"
    s = streams.config3(steps=2)
    rp, col, val = s.csr0()
    n = len(rp) - 1
    k = 32
    vals, vecs = init_eig.leading_eigenpairs(rp, col, val, k, "abs_desc", device=dev)
    gpu = TrackerSession(rp, col, val, vals, vecs, kind="grest-rsvd", k=k, seed=3)
    keys = np.sort(s.keys0)
    for t, upd in enumerate(s.updates):
        lam_old, x_old = gpu.embedding()
        gpu.step(upd)
        n_total = n + upd.n_new
        # -- apply_update, bit-exact against host set algebra
        ri, rj = (np.asarray(x, np.int64) for x in upd.removed)
        keys = np.setdiff1d(keys, streams._keys(ri, rj), assume_unique=True)
        add = streams._keys(np.asarray(upd.added[0]), np.asarray(upd.added[1]))
        new = streams._keys(np.asarray(upd.new_edges[0]), np.asarray(upd.new_edges[1]))
        keys = np.sort(np.concatenate([keys, add, new]))
        erp, ecol, evals = streams.csr_from_keys(n_total, keys)
        grp, gcol, gval = gpu.csr(0)
        assert np.array_equal(grp, erp) and np.array_equal(gcol, ecol) and np.array_equal(gval, evals), f"CSR step {t}"
        # -- Rayleigh-Ritz on A~ = X-bar Lambda X-bar' + Delta (Eq. (14))
        lam, x = gpu.embedding()
        X = torch.as_tensor(np.ascontiguousarray(x), device=dev)
        Xb = torch.zeros(n_total, k, dtype=torch.float64, device=dev)
        Xb[:n] = torch.as_tensor(np.ascontiguousarray(x_old), device=dev)
        L = torch.as_tensor(lam_old, device=dev)
        D = _delta(upd, n_total, dev)
        AX = Xb @ (L[:, None] * (Xb.T @ X)) + torch.sparse.mm(D, X)
        th = torch.as_tensor(lam, device=dev)
        scale = float(th.abs().max())
        orth = float((X.T @ X - torch.eye(k, dtype=torch.float64, device=dev)).abs().max())
        rq = float(((X * AX).sum(0) - th).abs().max()) / scale
        res = float((X.T @ (AX - X * th)).abs().max()) / scale
        print(f"cfg3 full size step {t}: n={n_total} nnz={len(gcol)} |X'X-I|={orth:.1e} "
              f"Rayleigh quotients {rq:.1e} residual'X {res:.1e}")
        assert orth <= 1e-12, orth
        assert rq <= 1e-10, rq
        assert res <= 1e-10, res
        a = np.abs(lam)
        assert np.all(a[:-1] >= a[1:]), "abs_desc order"
        n = n_total
