"""Device replacements of two reference kernels checked against the oracle:
sym_eig_dense (eig.hpp:37-50, test_linalg.cpp:30-96) and the GaussianSampler
stream (rng.hpp:27-75) that feeds the RSVD sketch."""
import numpy as np
import pytest

import pyoracle as po
from harness import sin_angle

pytestmark = pytest.mark.gpu


def dev():
    import paper_2603_19439_b200 as m
    return m


def test_sym_eig_reference_cases():
    m = dev()
    w, v = m.sym_eig_dense(np.diag([3.0, 1.0, 2.0]), "abs_desc")
    assert np.allclose(w, [3, 2, 1], rtol=0, atol=1e-14)
    assert abs(v[0, 0]) == pytest.approx(1) and abs(v[2, 1]) == pytest.approx(1) and abs(v[1, 2]) == pytest.approx(1)
    w, v = m.sym_eig_dense(np.array([[-7.5]]), "alg_desc")
    assert w[0] == pytest.approx(-7.5) and abs(v[0, 0]) == pytest.approx(1.0)
    w, _ = m.sym_eig_dense(np.diag([-3.0, 1.0, 2.0]), "abs_desc")
    assert np.allclose(w[:2], [-3, 2])
    w, _ = m.sym_eig_dense(np.diag([-3.0, 1.0, 2.0]), "alg_desc")
    assert np.allclose(w[[0, 2]], [2, -3])
    w, _ = m.sym_eig_dense(np.array([[0.0, 2.0], [2.0, 0.0]]), "abs_desc")
    # spectrum {2, -2}: bisection resolves each value to within an ulp, so the
    # exact magnitude tie of test_linalg.cpp:62-69 may break either way here
    assert np.allclose(sorted(w), [-2, 2], rtol=0, atol=1e-15)
    nan2 = np.zeros((2, 2))
    nan2[0, 0] = np.nan
    with pytest.raises(m.TrackerError, match="non-finite"):
        m.sym_eig_dense(nan2)


@pytest.mark.parametrize("n", [2, 8, 33, 64, 164, 200, 228])
@pytest.mark.parametrize("order", ["abs_desc", "alg_desc"])
def test_sym_eig_random_matches_oracle(n, order):
    m = dev()
    g = po.gaussian_matrix(100 + n, n, n)
    s = 0.5 * (g + g.T)
    s[0, 1] += 1e-13  # slightly asymmetric input is symmetrized (test_linalg.cpp:80-88)
    w, v = m.sym_eig_dense(s, order, want=min(n, 40))
    wo, vo = po.sym_eig(s, {"abs_desc": 0, "alg_desc": 1}[order])
    scale = np.abs(wo).max()
    assert np.abs(w - wo).max() <= 1e-12 * scale
    sym = 0.5 * (s + s.T)
    resid = np.abs(sym @ v - v * w[: v.shape[1]]).max()
    assert resid <= 1e-11 * scale
    assert np.abs(v.T @ v - np.eye(v.shape[1])).max() <= 1e-12
    # compare spans over groups of separated eigenvalues
    k = v.shape[1]
    if k < n and abs(abs(wo[k - 1]) - abs(wo[k])) > 1e-6 * scale:
        assert sin_angle(v, vo[:, :k]) <= 1e-9


def test_sym_eig_clustered_and_repeated():
    m = dev()
    rng = np.random.default_rng(4)
    n = 120
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    d = np.concatenate([np.full(5, 7.0), np.full(3, -7.0 + 1e-13), np.linspace(-3, 3, n - 8)])
    s = (q * d) @ q.T
    w, v = m.sym_eig_dense(s, "abs_desc", want=8)
    assert np.abs(np.abs(w[:8]) - 7.0).max() <= 1e-12 * 7
    assert np.abs(v.T @ v - np.eye(8)).max() <= 1e-11
    top = q[:, :8]
    assert sin_angle(v, top) <= 1e-9


@pytest.mark.parametrize("seed,rows,cols", [(0, 10, 3), (5489, 1000, 7), (12345, 10485, 200), (7, 3, 3)])
def test_gaussian_stream_matches_reference_sampler(seed, rows, cols):
    m = dev()
    g = m.gaussian_matrix(seed, rows, cols)
    o = po.gaussian_matrix(seed, rows, cols)
    # identical mt19937_64 words and uniforms; log/sincos may differ by an ulp
    rel = np.abs(g - o) / np.maximum(1.0, np.abs(o))
    assert rel.max() <= 4e-16 * 8
    assert (g == o).mean() > 0.5


@pytest.mark.gpu
def test_residual_norms_match_host():
    """st_residual_norms (one full-operator SpMM on the device) equals the
    per-pair residual ||A x_i - theta_i x_i|| of the reference's Lanczos test
    (lanczos.hpp:85-95) computed on the host from the session's own CSR and
    embedding, for the adjacency and the normalized-Laplacian operator."""
    import scipy.sparse as sp

    from paper_2603_19439_b200 import TrackerSession, streams

    s = streams.config1(n=3000, steps=2)
    rp, col, val = s.csr0()
    rng = np.random.default_rng(0)
    x, _ = np.linalg.qr(rng.standard_normal((len(rp) - 1, 8)))
    for op, order in (("adjacency", "abs_desc"), ("normalized-laplacian", "alg_desc")):
        g = TrackerSession(rp, col, val, np.linspace(8.0, 1.0, 8), x, kind="grest-rsvd", k=8, seed=1,
                           operator=op, order=order)
        for upd in s.updates:
            g.step(upd)
        lam, X = g.embedding()
        which = 1 if op != "adjacency" else 0
        crp, ccol, cval = g.csr(which)
        n = len(crp) - 1
        A = sp.csr_matrix((cval, ccol, crp), shape=(n, n))
        ref = np.linalg.norm(A @ X - X * lam, axis=0)
        got = g.residual_norms()
        assert np.allclose(got, ref, rtol=1e-10, atol=1e-12 * np.abs(lam).max()), (op, got, ref)


@pytest.mark.gpu
def test_dmma_and_sparse_kernels_are_deterministic():
    """Repeated runs of the DMMA Gram / row-local GEMM (TMA pipelines) and the
    full-operator SpMV / SpMM on the same pseudo-random operands give the same
    bits (a lane-divergent mbarrier wait ahead of mma.sync.aligned once made
    partial column tiles sporadically wrong)."""
    from paper_2603_19439_b200 import TrackerSession, streams

    s = streams.config1(n=3000, steps=0)
    rp, col, val = s.csr0()
    x = np.linalg.qr(np.random.default_rng(0).standard_normal((len(rp) - 1, 8)))[0]
    g = TrackerSession(rp, col, val, np.arange(8.0, 0, -1), x, kind="grest-rsvd", k=8)
    bad = []
    for m1, m2 in [(148, 76), (128, 76), (148, 65), (100, 100), (200, 100), (164, 164), (64, 76), (32, 20)]:
        d = g.determinism(1, 20000, m1, m2, 12)
        if d != 0.0:
            bad.append(("nn", m1, m2, d))
    for m1, m2 in [(148, 148), (76, 76), (200, 200), (32, 200), (64, 100), (32, 32)]:
        d = g.determinism(0, 20000, m1, m2, 12)
        if d != 0.0:
            bad.append(("gram", m1, m2, d))
    for which, m in [(2, 1), (3, 32), (3, 100)]:
        d = g.determinism(which, 0, m, m, 8)
        if d != 0.0:
            bad.append(("sparse", which, m, d))
    assert not bad, bad
