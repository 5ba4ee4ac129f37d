"""The non-projection tracker kinds on the device (TRIP-Basic, TRIP, residual
modes, TIMERS; trackers.cpp:147-224, 310-339) against the oracle on the same
stream, plus the reference's own tracker properties (test_trackers.cpp)."""
import math

import numpy as np
import pytest

import pyoracle as po
from harness import SIN_TOL, csr_equal, sin_angle
from support import random_graph

pytestmark = pytest.mark.gpu


def _per_value(va, vb):
    return float((np.abs(np.asarray(va) - np.asarray(vb)) / np.maximum(np.abs(vb), 1e-300)).max())


def _pair(a: po.Csr, kind, k, **opts):
    from paper_2603_19439_b200 import TrackerSession

    o = po.Session(a, kind=kind, k=k, seed=0, **opts)
    vals, vecs = o.embedding()
    g = TrackerSession(a.rowptr, a.col, a.val, vals, vecs, kind=kind, k=k, seed=0)
    g.set_tracker_options(**opts)
    return g, o


OPTS = {
    "trip-basic": {},
    "trip": {},
    "trip-replace": {"trip_replace_span": True},
    "rm": {"mu": 0.5},
    "timers-iasc": {"theta": 0.05, "min_restart_gap": 2},
    "timers-grest2": {"theta": 0.05, "min_restart_gap": 3, "restart_inner": "grest2"},
    "timers-trip": {"theta": 0.02, "min_restart_gap": 2, "restart_inner": "trip"},
}


@pytest.mark.parametrize("case", list(OPTS))
def test_tracker_kinds_match_oracle(case):
    from paper_2603_19439_b200 import streams

    kind = "timers" if case.startswith("timers") else "trip" if case == "trip-replace" else case
    # trip_replace_span takes x_j = X b_j with b_j from a system whose (j, j)
    # entry is lambda_new_j - lambda_j - C_jj = 0: the direction is sensitive to
    # the rounding of C, and the difference between two correct implementations
    # grows ~30x per step (measured: sin 3e-15, 1e-14, 1e-11, 4e-10, 2e-7), so
    # that reading is compared over its first three steps
    s = streams.config1(n=2000, steps=3 if case == "trip-replace" else 6)
    rp, col, val = s.csr0()
    a = po.Csr(len(rp) - 1, rp, col, val)
    g, o = _pair(a, kind, 8, **OPTS[case])
    for t, u in enumerate(s.updates):
        g.step(u)
        o.step(u)
        gv, gx = g.embedding()
        ov, ox = o.embedding()
        ve, sa = _per_value(gv, ov), sin_angle(gx, ox)
        print(f"{case} step {t}: value err {ve:.2e} sin {sa:.2e} state {g.tracker_state()} oracle {o.tracker_stats()}")
        assert csr_equal(g.csr(0), o.csr(0))
        assert ve <= 1e-10, (t, ve)
        assert sa <= SIN_TOL, (t, sa)
        # per-column: the perturbation trackers' vectors are individually defined
        if not case.startswith("timers"):
            cs = np.abs(np.sum(gx * ox, axis=0))
            assert np.all(np.abs(cs - 1.0) <= 1e-9), (t, cs)
        ga, gs, gr, gridge = g.tracker_state()
        oa, os_, orr, oridge = o.tracker_stats()
        assert gs == os_ and abs(ga - oa) <= 1e-12 * max(1.0, abs(oa)) and gridge == oridge


def test_laplacian_operator_trip():
    from paper_2603_19439_b200 import TrackerSession, streams

    s = streams.config1(n=1500, steps=3)
    rp, col, val = s.csr0()
    a = po.Csr(len(rp) - 1, rp, col, val)
    o = po.Session(a, kind="trip", k=6, order="alg_desc", operator="normalized-laplacian", seed=0)
    vals, vecs = o.embedding()
    g = TrackerSession(rp, col, val, vals, vecs, kind="trip", k=6, order="alg_desc", operator="normalized-laplacian")
    for u in s.updates:
        g.step(u)
        o.step(u)
        gv, gx = g.embedding()
        ov, ox = o.embedding()
        assert _per_value(gv, ov) <= 1e-10 and sin_angle(gx, ox) <= SIN_TOL
        assert csr_equal(g.csr(1), o.csr(1))


def test_resort_two_triangles():
    """test_trackers.cpp:219-250 on the device."""
    from paper_2603_19439_b200 import TrackerSession, Update

    a = po.from_edges(6, [(0, 1, 1.0), (1, 2, 1.0), (0, 2, 1.0), (3, 4, 0.9), (4, 5, 0.9), (3, 5, 0.9)])
    o = po.Session(a, kind="trip-basic", k=2)
    vals, vecs = o.embedding()
    g = TrackerSession(a.rowptr, a.col, a.val, vals, vecs, kind="trip-basic", k=2)
    g.step(Update.make([(3, 4, 0.3), (4, 5, 0.3), (3, 5, 0.3)]))
    v, x = g.embedding()
    assert abs(v[0] - 2.4) <= 2.4e-12 and abs(v[1] - 2.0) <= 2e-12
    assert abs(x[0, 0]) < 1e-8 and abs(abs(x[3, 0]) - 1 / math.sqrt(3)) < 1e-12


def test_pure_expansion_keeps_values_bitwise():
    """test_trackers.cpp:100-121: a pure expansion leaves lambda + diag(C) = lambda."""
    from paper_2603_19439_b200 import TrackerSession, Update

    a = random_graph(30, 0.15, 101)
    for kind in ("trip-basic", "trip", "rm"):
        o = po.Session(a, kind=kind, k=5)
        vals, vecs = o.embedding()
        g1 = TrackerSession(a.rowptr, a.col, a.val, vals, vecs, kind=kind, k=5)
        g2 = TrackerSession(a.rowptr, a.col, a.val, vals, vecs, kind=kind, k=5)
        g1.step(Update.make([], [], 2, [(0, 30, 1.0), (5, 31, 1.0), (9, 30, 1.0)]))
        g2.step(Update.make([], [], 2, [(0, 30, 1.0), (5, 31, 1.0), (9, 30, 1.0), (30, 31, 1.0)]))
        v1, x1 = g1.embedding()
        v2, x2 = g2.embedding()
        assert np.array_equal(v1, vals), kind
        assert np.array_equal(v1, v2) and np.array_equal(x1, x2), kind


def test_timers_cadence_and_infinite_threshold():
    """test_trackers.cpp:252-283: restarts at steps 5 and 10 with theta = 0;
    theta = inf is bitwise the inner tracker."""
    from paper_2603_19439_b200 import TrackerSession, streams

    s = streams.config1(n=1200, steps=12)
    rp, col, val = s.csr0()
    a = po.Csr(len(rp) - 1, rp, col, val)
    o = po.Session(a, kind="timers", k=4)
    vals, vecs = o.embedding()
    g = TrackerSession(rp, col, val, vals, vecs, kind="timers", k=4)
    g.set_tracker_options(theta=0.0, min_restart_gap=5)
    t_inf = TrackerSession(rp, col, val, vals, vecs, kind="timers", k=4)
    t_inf.set_tracker_options(theta=float("inf"))
    iasc = TrackerSession(rp, col, val, vals, vecs, kind="iasc", k=4)
    restarts = []
    for t, u in enumerate(s.updates, start=1):
        g.step(u)
        t_inf.step(u)
        iasc.step(u)
        if g.tracker_state()[1] == 0:
            restarts.append(t)
        vi, xi = t_inf.embedding()
        va, xa = iasc.embedding()
        assert np.array_equal(vi, va) and np.array_equal(xi, xa)
    assert restarts == [5, 10]


def test_residual_modes_mu_collision_leaves_state():
    from paper_2603_19439_b200 import TrackerError, TrackerSession, streams

    s = streams.config1(n=1000, steps=1)
    rp, col, val = s.csr0()
    a = po.Csr(len(rp) - 1, rp, col, val)
    o = po.Session(a, kind="rm", k=3)
    vals, vecs = o.embedding()
    g = TrackerSession(rp, col, val, vals, vecs, kind="rm", k=3)
    g.set_tracker_options(mu=float(vals[1]))
    with pytest.raises(TrackerError, match="mu collides") as e:
        g.step(s.updates[0])
    assert e.value.kind == "invalid_argument"
    assert g.info()["steps_taken"] == 0 and np.array_equal(g.embedding()[1], vecs)
    with pytest.raises(TrackerError, match="timers cannot delegate to itself"):
        t = TrackerSession(rp, col, val, vals, vecs, kind="timers", k=3)
        t.set_tracker_options(restart_inner="timers")
