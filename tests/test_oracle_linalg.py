"""Pins the CPU restatement against proj/tests/test_linalg.cpp and
proj/tests/test_lanczos_rsvd.cpp (ordering, eig, orthonormalize, RNG, RSVD)."""
import json
import os

import numpy as np
import pytest

import pyoracle as po
from support import col_angle, orthonormality_error

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_known_answers.json")))


def test_mt19937_64_standard_known_answer():
    g = GOLD["mt19937_64"]
    raw = po.mt_raw(g["seed"], g["index"])
    assert int(raw[-1]) == int(g["value"])


def test_spectral_sort_known_answer():
    # test_linalg.cpp:17-28
    g = GOLD["spectral_sort"]
    assert po.spectral_sort(g["values"], 0).tolist() == g["abs_desc"]
    assert po.spectral_sort(g["values"], 1).tolist() == g["alg_desc"]
    assert po.spectral_sort([1.0, 1.0, 1.0], 0).tolist() == g["ties"]


def random_symmetric(n, seed):
    m = po.gaussian_matrix(seed, n, n)
    return 0.5 * (m + m.T)


def test_sym_eig_cases():
    # test_linalg.cpp:30-96
    w, v = po.sym_eig(np.diag([3.0, 1.0, 2.0]), 0)
    assert np.allclose(w, [3, 2, 1])
    assert abs(v[0, 0]) == pytest.approx(1) and abs(v[2, 1]) == pytest.approx(1)
    w, v = po.sym_eig(np.array([[-7.5]]), 1)
    assert w[0] == -7.5 and abs(v[0, 0]) == 1
    w, _ = po.sym_eig(np.diag([-3.0, 1.0, 2.0]), 0)
    assert np.allclose(w[:2], [-3, 2])
    w, _ = po.sym_eig(np.diag([-3.0, 1.0, 2.0]), 1)
    assert np.allclose(w[[0, 2]], [2, -3])
    w, _ = po.sym_eig(np.array([[0.0, 2.0], [2.0, 0.0]]), 0)
    assert np.allclose(w, [2, -2])
    s = random_symmetric(8, 17)
    w, v = po.sym_eig(s, 0)
    assert np.abs(v @ np.diag(w) @ v.T - s).max() <= 1e-10 * np.abs(s).max()
    assert orthonormality_error(v) <= 1e-10
    nan2 = np.zeros((2, 2)); nan2[0, 0] = np.nan
    with pytest.raises(po.OracleError, match="non-finite"):
        po.sym_eig(nan2, 0)


def test_orthonormalize_cases():
    # test_linalg.cpp:98-154
    m = po.gaussian_matrix(5, 50, 8)
    q = po.orthonormalize(m)
    assert q.shape[1] == 8 and orthonormality_error(q) <= 1e-12
    for c in range(8):
        assert np.linalg.norm(m[:, c] - q @ (q.T @ m[:, c])) <= 1e-10 * np.linalg.norm(m[:, c])
    m = po.gaussian_matrix(9, 30, 4)
    m[:, 3] = 2 * m[:, 0] - m[:, 1]
    assert po.orthonormalize(m).shape[1] == 3
    wz = m.copy(); wz[:, 2] = 0
    assert po.orthonormalize(wz).shape[1] == 2
    assert po.orthonormalize(np.zeros((10, 3))).shape[1] == 0
    # against an existing basis: uses two successive draws of one sampler (seed 11)
    g = po.gaussian_matrix(11, 40, 5 + 6 + 2)
    q1 = po.orthonormalize(g[:, :5])
    q2 = po.orthonormalize(g[:, 5:11], q1)
    assert q2.shape[1] == 6 and np.abs(q1.T @ q2).max() <= 1e-10 and orthonormality_error(q2) <= 1e-10
    assert po.orthonormalize(q1 @ po.gaussian_matrix(3, 5, 2), q1).shape[1] == 0
    q = po.orthonormalize(po.gaussian_matrix(13, 25, 6))
    q2 = po.orthonormalize(q)
    assert q2.shape[1] == 6 and np.abs(q2 - q @ (q.T @ q2)).max() <= 1e-10
    with pytest.raises(po.OracleError, match="row count mismatch"):
        po.orthonormalize(np.ones((4, 2)), np.ones((5, 1)))
    bad = np.ones((4, 2)); bad[1, 1] = np.inf
    with pytest.raises(po.OracleError, match="non-finite"):
        po.orthonormalize(bad)


def test_gaussian_sampler_statistics_and_determinism():
    # test_linalg.cpp:206-233
    a = po.gaussian_matrix(42, 64, 1)
    assert np.array_equal(a, po.gaussian_matrix(42, 64, 1))
    assert np.abs(a - po.gaussian_matrix(43, 64, 1)).max() > 0
    big = po.gaussian_matrix(7, 50000, 1).ravel()
    assert abs(big.mean()) < 0.02 and 0.95 < big.var() < 1.05
    assert po.mix_seed(0, 1) != po.mix_seed(0, 2)
    assert po.mix_seed(1, 1) != po.mix_seed(2, 1)
    assert po.mix_seed(5, 1, 2) != po.mix_seed(5, 2, 1)


def test_rsvd_exact_range_truncation_clamp_reproducible():
    # test_lanczos_rsvd.cpp:151-205
    g = po.gaussian_matrix(71, 120, 3)
    u = po.orthonormalize(g)
    v = po.orthonormalize(po.gaussian_matrix(1071, 20, 3))
    b = u @ np.diag([5.0, 2.0, 0.5]) @ v.T
    r = po.rsvd_dense(b, 3, 5, 9)
    assert r.shape[1] == 3 and orthonormality_error(r) <= 1e-12
    assert np.linalg.norm(u - r @ (r.T @ u)) <= 1e-10
    col = po.gaussian_matrix(72, 50, 1).ravel()
    row = po.gaussian_matrix(172, 8, 1).ravel()
    r = po.rsvd_dense(np.outer(col, row), 4, 2, 13)
    assert r.shape[1] == 1 and col_angle(r[:, 0], col) <= 1e-10
    assert po.rsvd_dense(np.zeros((12, 5)), 3, 3, 1).shape == (12, 0)
    b = po.gaussian_matrix(73, 40, 5)
    r = po.rsvd_dense(b, 10, 10, 3)
    assert r.shape[1] == 5 and np.linalg.norm(b - r @ (r.T @ b)) <= 1e-10 * np.linalg.norm(b)
    b = po.gaussian_matrix(74, 30, 10)
    r1, r2, r3 = po.rsvd_dense(b, 4, 3, 17), po.rsvd_dense(b, 4, 3, 17), po.rsvd_dense(b, 4, 3, 18)
    assert np.array_equal(r1, r2) and not np.array_equal(r1, r3)
    with pytest.raises(po.OracleError):
        po.rsvd_dense(b, 0, 3, 1)
    with pytest.raises(po.OracleError):
        po.rsvd_dense(b, 3, -1, 1)


def test_lanczos_known_spectra():
    # test_lanczos_rsvd.cpp:61-86 (triangle, 4-cycle)
    k3 = po.from_edges(3, [(0, 1), (1, 2), (0, 2)])
    w, v = po.lanczos(k3, 1)
    assert w[0] == pytest.approx(2.0, rel=1e-12) and col_angle(v[:, 0], np.ones(3)) <= 1e-8
    c4 = po.from_edges(4, [(0, 1), (1, 2), (2, 3), (3, 0)])
    w, _ = po.lanczos(c4, 2)
    assert abs(w[0]) == pytest.approx(2.0, rel=1e-10) and w[0] * w[1] < 0
