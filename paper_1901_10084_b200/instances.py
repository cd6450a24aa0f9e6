"""Seeded synthetic correlation-clustering instances for BASELINE.json's five
configs.

The reference ships no generators (it builds instances from SNAP edge lists,
instance.py:143-159, which are not in this container).  These stand-ins have
the configs' shapes: an undirected graph A, d_ij = 1 - A_ij (0 on edges),
w_ij = 1 on edges and lambda on non-edges, epsilon = 1/gamma,
W = I.  Everything is generated directly in the packed upper-triangle order
(core.py:40-44), one row at a time, so n = 18000 needs no n x n matrix.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import ProblemInstance, pair_count


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    n: int
    graph: str          # "planted" | "gnp" | "chung_lu"
    params: tuple
    gamma: float
    lam: float          # weight of non-edges
    passes: int
    seed: int


CONFIGS = {
    1: ConfigSpec("planted-4x25", 100, "planted", (4, 25, 0.8, 0.1), 5.0, 1.0, 50, 1),
    2: ConfigSpec("gnp-1000", 1000, "gnp", (0.01,), 5.0, 1.0, 100, 2),
    3: ConfigSpec("chunglu-4000", 4000, "chung_lu", (2.5, 10.0), 10.0, 0.5, 200, 3),
    4: ConfigSpec("planted-100x100", 10000, "planted", (100, 100, 0.3, 0.001), 10.0, 1.0, 100, 4),
    5: ConfigSpec("chunglu-18000", 18000, "chung_lu", (2.2, 8.0), 10.0, 1.0, 20, 5),
}


def _edge_prob_rows(spec: ConfigSpec):
    """Yield (i, p_row) with p_row[t] = P(edge (i, i+1+t))."""
    n = spec.n
    if spec.graph == "gnp":
        (p,) = spec.params
        for i in range(n - 1):
            yield i, np.full(n - 1 - i, p)
    elif spec.graph == "planted":
        ncl, size, p_in, p_out = spec.params
        label = np.arange(n) // size
        for i in range(n - 1):
            same = label[i + 1:] == label[i]
            yield i, np.where(same, p_in, p_out)
    elif spec.graph == "chung_lu":
        beta, mean_deg = spec.params
        w = (np.arange(n) + 1.0) ** (-1.0 / (beta - 1.0))
        w *= mean_deg / w.mean()
        tot = w.sum()
        for i in range(n - 1):
            yield i, np.minimum(1.0, w[i] * w[i + 1:] / tot)
    else:
        raise ValueError(f"unknown graph model {spec.graph!r}")


def adjacency_flat(spec: ConfigSpec) -> np.ndarray:
    """Packed 0/1 adjacency (upper triangle, row-major), seeded."""
    rng = np.random.default_rng(spec.seed)
    out = np.empty(pair_count(spec.n), dtype=np.float64)
    pos = 0
    for i, prob in _edge_prob_rows(spec):
        u = rng.random(prob.shape[0])
        out[pos:pos + prob.shape[0]] = (u < prob).astype(np.float64)
        pos += prob.shape[0]
    return out


def config_instance(config: int, n: int | None = None, seed: int | None = None) -> ProblemInstance:
    """ProblemInstance for BASELINE config 1..5 (optionally resized: same
    model at another n, used for small parity cases)."""
    spec = CONFIGS[config]
    if n is not None or seed is not None:
        params = spec.params
        if spec.graph == "planted" and n is not None:
            ncl, size, p_in, p_out = params
            size = max(1, n // ncl)
            params = (ncl, size, p_in, p_out)
        spec = ConfigSpec(spec.name, n or spec.n, spec.graph, params, spec.gamma, spec.lam,
                          spec.passes, spec.seed if seed is None else seed)
    A = adjacency_flat(spec)
    d = 1.0 - A
    w = A + spec.lam * (1.0 - A)
    return ProblemInstance.from_flat(spec.n, d, w, epsilon=1.0 / spec.gamma)


def random_instance(n, seed, epsilon=0.5):
    """Random CC-shaped instance in the style of the reference tests'
    helper (D in {0,1}, W ~ U(0.5, 1.5)); built from the same numpy calls so
    a seed gives the same instance as there."""
    rng = np.random.default_rng(seed)
    D = np.triu(rng.integers(0, 2, (n, n)).astype(float), 1)
    D = D + D.T
    Wt = np.triu(rng.uniform(0.5, 1.5, (n, n)), 1)
    Wt = Wt + Wt.T
    return ProblemInstance(n, D, Wt, epsilon=epsilon)
