"""Shared fixtures mirroring proj/tests/support/test_support.hpp:18-66."""
import numpy as np

import pyoracle as po


def uniforms(seed: int, count: int) -> np.ndarray:
    """GaussianSampler(seed).uniform() draws (rng.hpp:33): top 53 bits * 2^-53."""
    raw = po.mt_raw(seed, count)
    return (raw >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def random_edges(n: int, p: float, seed: int):
    """test_support.hpp:57-64: Erdos-Renyi pairs i<j kept when uniform() < p."""
    iu, ju = np.triu_indices(n, 1)
    # triu_indices enumerates row-major (i ascending, then j), the loop order of the fixture
    u = uniforms(seed, len(iu))
    keep = u < p
    return list(zip(iu[keep].tolist(), ju[keep].tolist()))


def random_graph(n: int, p: float, seed: int) -> po.Csr:
    return po.from_edges(n, random_edges(n, p, seed))


def col_angle(x, y) -> float:
    d = abs(float(x @ y)) / (np.linalg.norm(x) * np.linalg.norm(y))
    return float(np.arccos(min(1.0, max(0.0, d))))


def orthonormality_error(q) -> float:
    if q.shape[1] == 0:
        return 0.0
    return float(np.abs(q.T @ q - np.eye(q.shape[1])).max())


def span_residual(z, cols) -> float:
    if cols.shape[1] == 0:
        return 0.0
    return float(np.linalg.norm(cols - z @ (z.T @ cols)))
