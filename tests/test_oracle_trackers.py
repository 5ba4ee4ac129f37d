"""The oracle's perturbation trackers (TRIP-Basic, TRIP, residual modes) and
TIMERS, pinned to the reference's own tracker tests
(proj/tests/test_trackers.cpp:73-320) before the device path is compared
with them."""
import math

import numpy as np
import pytest

import pyoracle as po
from support import col_angle, random_graph

KINDS = ["trip-basic", "trip", "rm", "iasc", "grest2", "grest3", "grest-rsvd", "timers"]


def small_edit(a: po.Csr, w: float, seed: int) -> po.Update:
    """test_trackers.cpp:36-45: one random non-edge (i, j) of weight w, drawn
    with GaussianSampler(seed).uniform_index (raw() % n)."""
    raw = po.mt_raw(seed, 4096)
    dense = a.dense()
    q = 0
    while True:
        i, j = int(raw[q] % np.uint64(a.n)), int(raw[q + 1] % np.uint64(a.n))
        q += 2
        if i != j and dense[i, j] == 0.0:
            return po.Update.make([(i, j, w)])


def test_empty_update_leaves_every_tracker_untouched():
    a = random_graph(24, 0.2, 3)
    for kind in KINDS:
        s = po.Session(a, kind=kind, k=4)
        v0, x0 = s.embedding()
        s.step(po.Update.make())
        v1, x1 = s.embedding()
        assert np.array_equal(v0, v1) and np.array_equal(x0, x1), kind
        n, _, steps, _ = s.info()
        assert n == 24 and steps == 1, kind


def test_pure_expansion_keeps_eigenvalues_bitwise():
    for seed in range(5):
        a = random_graph(30, 0.15, 100 + seed)
        without_c = po.Update.make([], [], 2, [(0, 30, 1.0), (5, 31, 1.0), (9, 30, 1.0)])
        with_c = po.Update.make([], [], 2, [(0, 30, 1.0), (5, 31, 1.0), (9, 30, 1.0), (30, 31, 1.0)])
        for kind in ("trip-basic", "trip", "rm"):
            s1 = po.Session(a, kind=kind, k=5, seed=seed)
            s2 = po.Session(a, kind=kind, k=5, seed=seed)
            v0, _ = s1.embedding()
            s1.step(without_c)
            s2.step(with_c)
            v1, x1 = s1.embedding()
            v2, x2 = s2.embedding()
            assert np.array_equal(v1, v0), kind
            assert np.array_equal(v1, v2) and np.array_equal(x1, x2), kind


def test_trip_pure_expansion_keeps_padded_vectors():
    a = random_graph(20, 0.25, 11)
    s = po.Session(a, kind="trip", k=4)
    _, x0 = s.embedding()
    s.step(po.Update.make([], [], 1, [(3, 20, 1.0), (7, 20, 1.0)]))
    _, x1 = s.embedding()
    assert not s.tracker_stats()[3]  # zero right-hand side short-circuits the solve
    assert np.abs(x1[:20] - x0).max() <= 1e-14
    assert np.abs(x1[20:]).max() == 0.0


def test_trip_basic_second_order():
    a = po.from_edges(6, [(0, 1, 1.2), (1, 2, 0.9), (0, 2, 0.8), (2, 3, 1.7), (3, 4, 0.6), (4, 5, 1.1)])
    edit = po.Update.make([(0, 3, 0.05)])
    s = po.Session(a, kind="trip-basic", k=3)
    s.step(edit)
    v, _ = s.embedding()
    w, _ = po.sym_eig(po.apply_update(a, edit).dense(), 0)
    gap = min(abs(w[i] - w[i + 1]) for i in range(5))
    bound = 4.0 * (2.0 * 0.05 * 0.05) / gap
    assert np.all(np.abs(v - w[:3]) <= bound)


def _residual(a_next: po.Csr, vals, vecs):
    d = a_next.dense()
    return math.sqrt(sum(float(np.sum((d @ vecs[:, j] - vals[j] * vecs[:, j]) ** 2)) for j in range(vecs.shape[1])))


def test_trip_beats_trip_basic_on_most_edits():
    wins = 0
    for seed in range(10):
        a = random_graph(6, 0.5, 200 + seed)
        if a.nnz == 0:
            continue
        edit = small_edit(a, 1.0, 300 + seed)
        a_next = po.apply_update(a, edit)
        res = {}
        for kind in ("trip-basic", "trip"):
            s = po.Session(a, kind=kind, k=3, seed=seed)
            s.step(edit)
            res[kind] = _residual(a_next, *s.embedding())
        wins += res["trip"] <= res["trip-basic"] + 1e-12
    assert wins >= 7


def test_residual_modes_tighten_angles():
    wins = 0
    for seed in range(10):
        a = random_graph(6, 0.5, 400 + seed)
        if a.nnz == 0:
            continue
        edit = small_edit(a, 1.0, 500 + seed)
        _, wv = po.sym_eig(po.apply_update(a, edit).dense(), 0)
        ang = {}
        for kind in ("trip-basic", "rm"):
            s = po.Session(a, kind=kind, k=3, seed=seed)
            s.step(edit)
            _, x = s.embedding()
            ang[kind] = sum(col_angle(x[:, j], wv[:, j]) for j in range(3)) / 3.0
        wins += ang["rm"] <= ang["trip-basic"] + 1e-12
    assert wins >= 7


def test_residual_modes_reject_colliding_mu():
    a = random_graph(12, 0.3, 21)
    s = po.Session(a, kind="rm", k=3)
    v, _ = s.embedding()
    s2 = po.Session(a, kind="rm", k=3, mu=float(v[1]))
    with pytest.raises(po.OracleError, match="mu collides"):
        s2.step(small_edit(a, 1.0, 22))


def test_trip_span_replacement_is_distinct():
    a = random_graph(12, 0.4, 31)
    edit = small_edit(a, 1.0, 32)
    corr = po.Session(a, kind="trip", k=4)
    repl = po.Session(a, kind="trip", k=4, trip_replace_span=True)
    corr.step(edit)
    repl.step(edit)
    vc, xc = corr.embedding()
    vr, xr = repl.embedding()
    assert np.array_equal(vc, vr)
    assert not np.array_equal(xc, xr)
    assert np.allclose(np.linalg.norm(xr, axis=0), 1.0, rtol=0, atol=1e-12)


def test_trackers_resort_when_spectrum_reorders():
    a = po.from_edges(6, [(0, 1, 1.0), (1, 2, 1.0), (0, 2, 1.0), (3, 4, 0.9), (4, 5, 0.9), (3, 5, 0.9)])
    s = po.Session(a, kind="trip-basic", k=2)
    v, _ = s.embedding()
    assert abs(v[0] - 2.0) < 1e-9 and abs(v[1] - 1.8) < 1e-9
    s.step(po.Update.make([(3, 4, 0.3), (4, 5, 0.3), (3, 5, 0.3)]))
    v, x = s.embedding()
    assert abs(v[0] - 2.4) <= 2.4e-12 and abs(v[1] - 2.0) <= 2e-12
    assert abs(x[0, 0]) < 1e-8
    assert abs(abs(x[3, 0]) - 1 / math.sqrt(3)) < 1e-12


class _Evolving:
    def __init__(self, a, seed):
        self.a, self.seed, self.t = a, seed, 0

    def next(self):
        e = small_edit(self.a, 1.0, self.seed + self.t)
        self.t += 1
        self.a = po.apply_update(self.a, e)
        return e


def test_timers_forced_cadence():
    g = _Evolving(random_graph(20, 0.2, 41), 600)
    s = po.Session(g.a, kind="timers", k=3, theta=0.0, min_restart_gap=5)
    restarts = []
    for t in range(1, 13):
        s.step(g.next())
        if s.tracker_stats()[1] == 0:
            restarts.append(t)
    assert restarts == [5, 10]


def test_timers_infinite_threshold_is_the_inner_tracker():
    g1 = _Evolving(random_graph(20, 0.2, 51), 700)
    g2 = _Evolving(random_graph(20, 0.2, 51), 700)
    t = po.Session(g1.a, kind="timers", k=3, theta=float("inf"))
    i = po.Session(g2.a, kind="iasc", k=3)
    for _ in range(6):
        t.step(g1.next())
        i.step(g2.next())
        vt, xt = t.embedding()
        vi, xi = i.embedding()
        assert np.array_equal(vt, vi) and np.array_equal(xt, xi)


def test_timers_restart_equals_fresh_init():
    g = _Evolving(random_graph(18, 0.25, 61), 800)
    s = po.Session(g.a, kind="timers", k=3, seed=9, theta=0.0, min_restart_gap=1)
    for _ in range(3):
        s.step(g.next())
        fresh = po.Session(g.a, kind="timers", k=3, seed=9)
        v, x = s.embedding()
        fv, fx = fresh.embedding()
        assert np.array_equal(v, fv) and np.array_equal(x, fx)


def test_solve_linear_small_ridge():
    """solve.hpp:23-45: a singular system takes the ridge fallback."""
    assert po.Session  # the solver is exercised through trip; a singular c gives ridge_used
    a = po.from_edges(4, [(0, 1, 1.0), (2, 3, 1.0)])  # two identical components: degenerate spectrum
    s = po.Session(a, kind="trip", k=4)
    s.step(po.Update.make([(0, 2, 1.0)]))
    v, x = s.embedding()
    assert np.all(np.isfinite(v)) and np.all(np.isfinite(x))
