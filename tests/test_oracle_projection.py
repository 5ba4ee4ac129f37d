"""Pins the CPU restatement against proj/tests/test_projection.cpp and
proj/tests/test_trackers.cpp:73-98 (projection basis, Rayleigh-Ritz, empty
updates)."""
import numpy as np
import pytest

import pyoracle as po
from support import col_angle, orthonormality_error, random_graph, span_residual


def session(a, kind, k, seed=0, **kw):
    return po.Session(a, kind=kind, k=k, seed=seed, **kw)


def mixed_update(n_old):
    # test_projection.cpp:35-39
    return po.Update.make([(0, 4, 1.0), (1, 5, 1.0)], [], 3,
                          [(2, n_old, 1.0), (3, n_old + 1, 1.0), (6, n_old + 2, 1.0), (n_old, n_old + 1, 1.0)])


def test_iasc_basis_is_padded_identity():
    a = random_graph(12, 0.3, 7)
    s = session(a, "iasc", 3)
    _, x = s.embedding()
    z = s.probe_basis(mixed_update(12), "iasc", 1)
    assert z.shape == (15, 6)
    assert np.array_equal(z[:12, :3], x)
    assert np.array_equal(z[12:, 3:], np.eye(3))
    assert np.abs(z[:12, 3:]).max() == 0 and np.abs(z[12:, :3]).max() == 0
    assert orthonormality_error(z) <= 1e-12


def test_grest2_keeps_old_basis_and_captures_perturbation():
    a = random_graph(12, 0.3, 8)
    s = session(a, "grest2", 3)
    _, x = s.embedding()
    up = mixed_update(12)
    z = s.probe_basis(up, "grest2", 1)
    assert z.shape[0] == 15 and z.shape[1] <= 6
    xb = np.zeros((15, 3)); xb[:12] = x
    assert np.array_equal(z[:, :3], xb)
    assert orthonormality_error(z) <= 1e-10
    dx = po.update_delta(12, up).dense() @ xb
    assert span_residual(z, dx) <= 1e-8 * max(1.0, np.linalg.norm(dx))


def test_empty_perturbation_basis_is_padded_old_basis():
    a = random_graph(10, 0.3, 9)
    s = session(a, "grest2", 4)
    _, x = s.embedding()
    z = s.probe_basis(po.Update.make(), "grest2", 1)
    assert z.shape == (10, 4) and np.array_equal(z, x)


def test_grest3_extends_grest2():
    a = random_graph(12, 0.3, 10)
    s = session(a, "grest3", 3)
    up = mixed_update(12)
    z2 = s.probe_basis(up, "grest2", 1)
    z3 = s.probe_basis(up, "grest3", 1)
    assert z2.shape[1] <= z3.shape[1] <= z2.shape[1] + 3
    assert span_residual(z3, z2) <= 1e-8
    d2 = po.update_delta(12, up).dense()[:, 12:]
    assert span_residual(z3, d2) <= 1e-8 * max(1.0, np.linalg.norm(d2))
    assert orthonormality_error(z3) <= 1e-10


def test_rsvd_bypass_is_bitwise_grest3():
    a = random_graph(12, 0.3, 12)
    s = session(a, "grest-rsvd", 3, rsvd_l=8)
    up = mixed_update(12)
    assert np.array_equal(s.probe_basis(up, "grest3", 5), s.probe_basis(up, "grest-rsvd", 5))


def test_rsvd_recovers_full_span_for_small_rank():
    a = random_graph(14, 0.3, 13)
    s = session(a, "grest-rsvd", 3, rsvd_l=2, rsvd_p=2)
    up = po.Update.make(n_new=3, new_edges=[(1, 14, 1.0), (6, 14, 1.0), (1, 15, 1.0), (6, 15, 1.0), (1, 16, 1.0),
                                            (6, 16, 1.0)])
    z3 = s.probe_basis(up, "grest3", 5)
    zr = s.probe_basis(up, "grest-rsvd", 5)
    assert orthonormality_error(zr) <= 1e-10
    assert span_residual(z3, zr) <= 1e-8 and span_residual(zr, z3) <= 1e-8


def test_rayleigh_ritz_exact_on_invariant_subspace():
    a = random_graph(8, 0.5, 14)
    up = po.Update.make([(0, 5, 1.0)], [], 2, [(3, 8, 1.0), (6, 9, 1.0), (8, 9, 1.0)])
    a_next = po.apply_update(a, up)
    w, v = po.sym_eig(a_next.dense(), 0)
    s = session(a, "grest2", 8)
    vals, vecs = s.probe_rr(up, v[:, :8])
    for j in range(8):
        assert vals[j] == pytest.approx(w[j], rel=1e-9)
        assert col_angle(vecs[:, j], v[:, j]) <= 1e-7


def test_rayleigh_ritz_validates_subspace():
    a = random_graph(10, 0.3, 16)
    s = session(a, "grest2", 4)
    up = po.Update.make([(0, 3, 1.0)])
    with pytest.raises(po.OracleError, match="projection subspace too small"):
        s.probe_rr(up, np.eye(10, 3))
    skew = np.eye(10, 5); skew[0, 1] = 0.5
    with pytest.raises(po.OracleError, match="column-orthonormal"):
        s.probe_rr(up, skew)
    with pytest.raises(po.OracleError, match="row count"):
        s.probe_rr(up, np.eye(9, 5))


def test_empty_update_leaves_tracker_untouched():
    # test_trackers.cpp:73-87 (projection kinds)
    a = random_graph(24, 0.2, 3)
    for kind in ("iasc", "grest2", "grest3", "grest-rsvd"):
        s = session(a, kind, 4)
        v0, x0 = s.embedding()
        s.step(po.Update.make())
        v1, x1 = s.embedding()
        n, k, steps, _ = s.info()
        assert np.array_equal(v0, v1) and np.array_equal(x0, x1) and n == 24 and steps == 1
