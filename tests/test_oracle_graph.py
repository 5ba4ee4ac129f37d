"""Pins the CPU restatement (oracle/) against the reference's own known-answer
tests for the ingestion half of the hot path: proj/tests/test_sparse_graph.cpp
and proj/tests/test_laplacian.cpp, plus tests/golden/reference_known_answers.json."""
import json
import os

import numpy as np
import pytest

import pyoracle as po
from support import random_edges, random_graph, uniforms

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_known_answers.json")))


def path3():
    return po.from_edges(3, [(0, 1), (1, 2)])


def triangle():
    return po.from_edges(3, [(0, 1), (1, 2), (0, 2)])


def golden_csr(g):
    return po.Csr(g["n"], np.array(g["rowptr"], np.int32), np.array(g["col"], np.int32), np.array(g["val"]))


def fig1_update():
    u = GOLD["fig1"]["update"]
    return po.Update.make(u["added"], u["removed"], u["n_new"], u["new_edges"])


def test_compressed_storage_invariants():
    # test_sparse_graph.cpp:52-64
    edges = random_edges(25, 0.2, 3)
    a = po.from_edges(25, edges)
    assert a.nnz == 2 * len(edges)
    assert np.all(np.diff(a.rowptr) >= 0)
    for r in range(a.n):
        assert np.all(np.diff(a.col[a.rowptr[r]:a.rowptr[r + 1]]) > 0)
    assert np.all(a.val != 0)
    d = a.dense()
    assert np.array_equal(d, d.T)


def test_builders_reject_malformed_edges():
    # test_sparse_graph.cpp:66-73
    for bad in ([(0, 0)], [(0, 1), (1, 0)], [(0, 5)]):
        with pytest.raises(po.OracleError) as e:
            po.from_edges(3, bad)
        assert e.value.kind == "invalid_argument"
    with pytest.raises(po.OracleError, match="not symmetric"):
        po.from_triplets(2, [(0, 1, 1.0)])


def test_from_triplets_sums_duplicates_and_prunes():
    a = po.from_triplets(3, [(0, 1, 1.0), (1, 0, 1.0), (0, 1, 2.0), (1, 0, 2.0), (1, 2, 1.0), (2, 1, 1.0),
                             (1, 2, -1.0), (2, 1, -1.0)])
    assert a.nnz == 2 and a.coeff(0, 1) == 3.0 and a.coeff(1, 2) == 0.0


def test_assemble_update_places_edits():
    # test_sparse_graph.cpp:128-144 via the delta it produces
    d = po.update_delta(6, fig1_update())
    assert d.equal(golden_csr(GOLD["fig1"]["delta"]))
    assert d.nnz == GOLD["fig1"]["k_block_nnz"] + 2 * GOLD["fig1"]["g_block_nnz"] + GOLD["fig1"]["c_block_nnz"]


@pytest.mark.parametrize("n_old,upd,msg", [
    (4, po.Update.make([(0, 1, 1.0)], [(0, 1)]), "duplicate edge"),
    (4, po.Update.make([(2, 2, 1.0)]), "self-loop"),
    (4, po.Update.make([(0, 9, 1.0)]), "existing nodes"),
    (4, po.Update.make(n_new=1, new_edges=[(0, 1, 1.0)]), "only existing"),
    (4, po.Update.make(n_new=1, new_edges=[(0, 4, -1.0)]), "positive weight"),
    (4, po.Update.make([(0, 1, 0.0)]), "zero-weight"),
])
def test_assemble_update_validates(n_old, upd, msg):
    # test_sparse_graph.cpp:146-153 (messages from graph.cpp:50-90)
    with pytest.raises(po.OracleError, match=msg) as e:
        po.update_delta(n_old, upd)
    assert e.value.kind == "invalid_argument"


def test_apply_update_fig1_known_answer():
    # test_sparse_graph.cpp:174-185: the cycle with chord evolves into the 8-node target, bitwise
    a0 = po.from_edges(6, GOLD["fig1"]["a0_edges"])
    a1 = po.apply_update(a0, fig1_update())
    assert a1.equal(golden_csr(GOLD["fig1"]["a1"]))
    assert a1.coeff(1, 4) == 0.0
    assert np.all(a1.val != 0)


def test_apply_update_rejects_bad_deletions():
    # test_sparse_graph.cpp:187-199
    with pytest.raises(po.OracleError, match="invalid deletion") as e:
        po.apply_update(path3(), po.Update.make(removed=[(0, 2)]))
    assert e.value.kind == "invalid_argument"
    weighted = po.from_edges(2, [(0, 1, 0.5)])
    with pytest.raises(po.OracleError, match="negative"):
        po.apply_update(weighted, po.Update.make(removed=[(0, 1)]))
    with pytest.raises(po.OracleError, match="d.n_old"):
        po.apply_update(path3(), po.Update.make(), n_old=7)


def test_apply_update_triangle_deletion_and_expansions():
    # test_sparse_graph.cpp:201-229
    after = po.apply_update(triangle(), po.Update.make(removed=[(0, 1)]))
    assert after.equal(po.from_edges(3, [(0, 2), (1, 2)]))
    grown = po.apply_update(triangle(), po.Update.make(n_new=1))
    assert grown.n == 4 and grown.rowptr[-1] == grown.rowptr[-2]
    same = po.apply_update(triangle(), po.Update.make())
    assert same.equal(triangle())
    bigger = po.apply_update(triangle(), po.Update.make(n_new=2, new_edges=[(0, 3, 1.0), (3, 4, 1.0)]))
    assert bigger.n == 5 and bigger.coeff(0, 3) == 1.0 and bigger.coeff(4, 3) == 1.0


def test_shifted_laplacians_of_the_triangle():
    # test_sparse_graph.cpp:231-266
    t, warned = po.shifted_laplacian(triangle(), 0, 4.0)
    assert np.array_equal(t.dense(), np.array(GOLD["laplacian_triangle"]["combinatorial_alpha4"]))
    assert not warned
    _, warned = po.shifted_laplacian(triangle(), 0, 3.0)
    assert warned
    tn, _ = po.shifted_laplacian(triangle(), 1, 2.0)
    w, _ = po.sym_eig(tn.dense(), 1)
    assert np.allclose(w, GOLD["laplacian_triangle"]["normalized_eigs_alg_desc"], atol=1e-12)
    lone, _ = po.shifted_laplacian(po.from_edges(1, []), 1, 2.0)
    assert lone.coeff(0, 0) == 2.0
    with pytest.raises(po.OracleError, match="alpha == 2"):
        po.shifted_laplacian(triangle(), 1, 4.0)


def test_weighted_normalized_shift_is_exactly_symmetric():
    # test_laplacian.cpp:75-92
    for seed in range(20):
        n = 12
        iu, ju = np.triu_indices(n, 1)
        u = uniforms(900 + seed, 4 * len(iu))
        edges, t = [], 0
        for i, j in zip(iu, ju):
            x = u[t]; t += 1
            if x < 0.4:
                edges.append((int(i), int(j), 0.25 + u[t])); t += 1
        a = po.from_edges(n, edges)
        ad = a.dense()
        deg = ad.sum(1)
        if deg.min() <= 0:
            continue
        tn, _ = po.shifted_laplacian(a, 1, 2.0)  # symmetric validation inside from_triplets
        s = 1 / np.sqrt(deg)
        expected = 2 * np.eye(n) - (np.eye(n) - s[:, None] * ad * s[None, :])
        assert np.abs(tn.dense() - expected).max() <= 1e-12


def test_laplacian_session_reshift_and_bitwise_delta():
    # test_laplacian.cpp:127-147: pad(T_before) + delta == T_after bitwise
    start = po.from_edges(4, [(0, 1), (1, 2)])
    s = po.Session(start, kind="grest3", k=1, operator="laplacian", values=[1.0], vectors=np.eye(4, 1))
    assert s.info()[3] == 4.0
    t0 = s.csr(1)
    s.step(po.Update.make([(2, 3, 1.0)]))
    assert s.info()[3] == 4.0
    d1 = s.csr(2)
    assert np.array_equal(t0.dense() + d1.dense(), s.csr(1).dense())
    t1 = s.csr(1)
    s.step(po.Update.make([(1, 3, 1.0)], n_new=1, new_edges=[(1, 4, 1.0)]))
    assert s.info()[3] == 8.0
    d2 = s.csr(2)
    padded = np.zeros((5, 5))
    padded[:4, :4] = t1.dense()
    assert np.array_equal(padded + d2.dense(), s.csr(1).dense())
    t_ref, _ = po.shifted_laplacian(s.csr(0), 0, 8.0)
    assert s.csr(1).equal(t_ref)


def test_laplacian_session_empty_update_and_mismatch():
    # test_laplacian.cpp:149-161
    for op in ("laplacian", "normalized-laplacian"):
        a = random_graph(6, 0.5, 4)
        s = po.Session(a, kind="grest2", k=1, operator=op, values=[1.0], vectors=np.eye(6, 1))
        s.step(po.Update.make())
        assert s.csr(2).nnz == 0
    with pytest.raises(po.OracleError):
        po.update_delta(5, po.Update.make([(0, 9, 1.0)]))
