"""Drop-in generator API (hrgen generator.py) on the B200 path.

Same names, parameters, validation and exceptions as the reference; the
work runs in libhrgen_b200.so:

  sample_points        -> hrg_sample_points   (Philox4x32-10, one counter per vertex)
  generate[_with_stats]-> hrg_generate        (sample + band index + range query + CSR)
  generate_brute_force / edges_from_coordinates
                       -> hrg_edges_from_coords (edges among given coordinates)

Differences from hrgen, all documented in DESIGN.md:
  * the coordinate stream is Philox, not numpy's PCG64, so a seed gives a
    different (equally distributed) point set than hrgen's for that seed;
    for any fixed coordinates the edge set is hrgen's;
  * `threads` and `leaf_capacity` are accepted and validated for
    compatibility; they do not change the GPU schedule or the output
    (hrgen guarantees the same invariance).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .engine import Shard, get_engine
from .errors import InfeasibleParametersError, ParameterDomainError
from .geometry import (
    TWO_PI,
    ModelParams,
    alpha_from_gamma,
    target_radius,
    to_poincare_radius,
)
from .graph import Graph

DEFAULT_GENERATOR_CAPACITY = 512
_LONG_RANGE_STREAM = 1   # hrgen generator.py:48

VERTEX_ORDERS = {"sample": _lib.ORDER_SAMPLE, "angular": _lib.ORDER_ANGULAR}


@dataclass(frozen=True)
class GeneratorParams:
    """hrgen generator.py:51-106.  Exactly one of (avg_degree, radius) and
    one of (gamma, alpha).  Extra field: vertex_order ("sample": vertex i is
    the i-th draw, hrgen's labelling; "angular": ids in (band, angle) order,
    whose CSR rows need no sort -- hrgen's edge rule applied to those labels,
    which decides a few borderline pairs differently from the sample-order
    graph: 1601 of 1.6e8 at config 2, so it is not exactly a relabelling)."""

    n: int
    avg_degree: float | None = None
    radius: float | None = None
    gamma: float | None = None
    alpha: float | None = None
    seed: int = 0
    threads: int = 1
    leaf_capacity: int = DEFAULT_GENERATOR_CAPACITY
    long_range_fraction: float = 0.0
    vertex_order: str = "sample"

    def __post_init__(self):
        if self.n < 1:
            raise ParameterDomainError("n must be at least 1")
        if (self.avg_degree is None) == (self.radius is None):
            raise ParameterDomainError("exactly one of avg_degree and radius must be set")
        if (self.gamma is None) == (self.alpha is None):
            raise ParameterDomainError("exactly one of gamma and alpha must be set")
        if self.avg_degree is not None and not self.avg_degree > 0.0:
            raise ParameterDomainError("avg_degree must be positive")
        if self.radius is not None and not self.radius > 0.0:
            raise ParameterDomainError("radius must be positive")
        if self.gamma is not None and not self.gamma > 2.0:
            raise ParameterDomainError("gamma must exceed 2")
        if self.alpha is not None and not self.alpha > 0.5:
            raise ParameterDomainError("alpha must exceed 0.5")
        if not 0 <= self.seed < 2**64:
            raise ParameterDomainError("seed must be a 64-bit unsigned integer")
        if self.threads < 1:
            raise ParameterDomainError("threads must be at least 1")
        if self.leaf_capacity < 1:
            raise ParameterDomainError("leaf_capacity must be at least 1")
        if not 0.0 <= self.long_range_fraction < 1.0:
            raise ParameterDomainError("long_range_fraction must be in [0, 1)")
        if self.vertex_order not in VERTEX_ORDERS:
            raise ParameterDomainError(f"vertex_order must be one of {sorted(VERTEX_ORDERS)}")

    def resolve(self) -> ModelParams:
        alpha = self.alpha if self.alpha is not None else alpha_from_gamma(self.gamma)
        if self.radius is not None:
            R = self.radius
        else:
            R = target_radius(self.n, self.avg_degree, alpha)
        return ModelParams(n=self.n, alpha=alpha, R=R, target_avg_degree=self.avg_degree)


@dataclass(frozen=True)
class VertexCoordinates:
    """hrgen generator.py:109-122: positions in both coordinate systems."""

    phi: np.ndarray
    r_native: np.ndarray
    r_poincare: np.ndarray

    def __len__(self):
        return self.phi.size

    @property
    def n(self):
        return self.phi.size


@dataclass(frozen=True)
class GenerationStats:
    """hrgen generator.py:125-139.  Phase times are CUDA-event device times
    in nanoseconds: sample (Philox + keys), build (sort + index), edges
    (count, scan, write, row order)."""

    n: int
    m: int
    radius: float
    alpha: float
    t_sample_ns: int
    t_build_ns: int
    t_edges_ns: int
    candidates: int = 0
    kernel_launches: int = 0

    @property
    def t_total_ns(self):
        return self.t_sample_ns + self.t_build_ns + self.t_edges_ns


def radial_inverse_cdf(u, alpha, radius):
    """Quantile of the radial density (hrgen generator.py:142-157), host
    numpy form; the GPU sampler evaluates the same expression per vertex."""
    if not alpha > 0.0:
        raise ParameterDomainError("alpha must be positive")
    if not radius > 0.0:
        raise ParameterDomainError("radius must be positive")
    u_arr = np.asarray(u, dtype=np.float64)
    if np.any(u_arr < 0.0) or np.any(u_arr > 1.0):
        raise ParameterDomainError("u must lie in [0, 1]")
    out = (2.0 / alpha) * np.arcsinh(np.sqrt(u_arr) * math.sinh(alpha * radius / 2.0))
    return out if np.ndim(u) else float(out)


def _check_model_domain(model: ModelParams):
    if not to_poincare_radius(model.R) < 1.0:
        # hrgen builds PolarQuadtree(max_r=tanh(R/2)) which rejects max_r >= 1
        raise ValueError("max_r must be in (0, 1)")


def sample_points(n, alpha, radius, seed, *, vertex_order="sample", device=None):
    """n vertex positions from the seeded counter-based stream; vertex i of
    generate() with the same (n, alpha, radius, seed, vertex_order) sits at
    index i.  hrgen generator.py:160-179."""
    if n < 1:
        raise ParameterDomainError("n must be at least 1")
    model = ModelParams(n=int(n), alpha=float(alpha), R=float(radius))
    _check_model_domain(model)
    phi, rn, rp = get_engine(device).sample_points(model, seed, VERTEX_ORDERS[vertex_order])
    return VertexCoordinates(phi=phi, r_native=rn, r_poincare=rp)


def _stats(model, st) -> GenerationStats:
    return GenerationStats(
        n=int(model.n), m=int(st.m), radius=float(model.R), alpha=float(model.alpha),
        t_sample_ns=int(st.t_sample_ms * 1e6), t_build_ns=int(st.t_build_ms * 1e6),
        t_edges_ns=int(st.t_edges_ms * 1e6), candidates=int(st.candidates),
        kernel_launches=int(st.kernel_launches))


def generate_with_stats(params: GeneratorParams, *, device=None, shard: Shard | None = None,
                        pinned: bool = True):
    """hrgen generator.py:190-239.  With `shard`, only that angular sector's
    rows are emitted (multi-GPU; see distributed.py)."""
    if shard is not None and shard.count > 1 and params.long_range_fraction > 0.0:
        raise ParameterDomainError(
            "long_range_fraction > 0 needs the whole graph, not one shard's rows")
    model = params.resolve()
    _check_model_domain(model)
    eng = get_engine(device)
    with eng.lock:  # the result read back is this call's
        st = eng.generate(model, params.seed, VERTEX_ORDERS[params.vertex_order], shard)
        indptr, indices = eng.copy_csr(np.int64, pinned=pinned)
    graph = Graph(indptr=indptr, indices=indices)
    if params.long_range_fraction > 0.0:
        graph = add_long_range_edges(graph, params.long_range_fraction, params.seed)
    stats = _stats(model, st)
    if params.long_range_fraction > 0.0:
        stats = GenerationStats(**{**stats.__dict__, "m": graph.m})
    return graph, stats


def generate_with_coordinates(params: GeneratorParams, *, device=None, pinned: bool = True):
    """The north star's "coordinates plus an edge list" in one call: the
    Graph of generate() and the VertexCoordinates it was built on (vertex i
    at index i; the same arrays sample_points returns for these parameters),
    both read back from the one generation."""
    model = params.resolve()
    _check_model_domain(model)
    eng = get_engine(device)
    with eng.lock:
        eng.generate(model, params.seed, VERTEX_ORDERS[params.vertex_order])
        indptr, indices = eng.copy_csr(np.int64, pinned=pinned)
        phi, rn, rp = eng.copy_coords()
    graph = Graph(indptr=indptr, indices=indices)
    if params.long_range_fraction > 0.0:
        graph = add_long_range_edges(graph, params.long_range_fraction, params.seed)
    return graph, VertexCoordinates(phi=phi, r_native=rn, r_poincare=rp)


def generate(params: GeneratorParams, *, device=None) -> Graph:
    """hrgen generator.py:242-246."""
    graph, _ = generate_with_stats(params, device=device)
    return graph


def edges_from_coordinates(coords, radius, *, alpha=1.0, device=None, shard=None,
                           pinned=True) -> Graph:
    """The edge set hrgen.generate produces for these coordinates and disk
    radius: {v,w}, v<w, iff w is strictly inside v's circle (generator.py:
    182-187, quadtree.py:611-613).  Coordinates must lie in the quadtree
    region (phi in [0, 2pi), r_poincare in [0, tanh(R/2))), else
    OutOfBoundsError.  The edge set does not depend on alpha (in hrgen it
    only shapes the quadtree); it is recorded in the model for completeness."""
    if not radius > 0.0:
        raise ParameterDomainError("radius must be positive")
    phi = coords.phi
    rp = coords.r_poincare
    n = int(len(phi))
    model = ModelParams(n=max(n, 1), alpha=float(alpha), R=float(radius))
    _check_model_domain(model)
    if n == 0:
        return Graph.from_edge_arrays(0, [], [])
    eng = get_engine(device)
    with eng.lock:
        eng.edges_from_coords(model, phi, rp, shard)
        indptr, indices = eng.copy_csr(np.int64, pinned=pinned)
    return Graph(indptr=indptr, indices=indices)


def generate_brute_force(coords, radius, *, device=None) -> Graph:
    """hrgen generator.py:249-274: all-pairs edges, {i, j} iff
    2 asinh(sqrt(d2 / (b_i b_j))) < radius, evaluated in hrgen's order on the
    device (O(n^2); a validation reference, like hrgen's).  Pairs within 4
    ulps of the radius, where the device's asinh and numpy's may round
    differently, are counted in `generate_brute_force.last_near_ties`."""
    if not radius > 0.0:
        raise ParameterDomainError("radius must be positive")
    n = len(coords)
    if n == 0:
        return Graph.from_edge_arrays(0, [], [])
    eng = get_engine(device)
    with eng.lock:
        generate_brute_force.last_near_ties = eng.edges_brute_force(coords.phi, coords.r_poincare,
                                                                    float(radius))
        indptr, indices = eng.copy_csr(np.int64)
    return Graph(indptr=indptr, indices=indices)


generate_brute_force.last_near_ties = 0


def add_long_range_edges(graph: Graph, fraction, seed) -> Graph:
    """hrgen generator.py:277-316: add ceil(fraction*m) uniformly random
    absent edges drawn by rejection from numpy's default_rng([seed, 1]).
    Host-side by nature (a sequential rejection stream); bit-identical to
    hrgen for the same input graph and seed."""
    if not 0.0 <= fraction < 1.0:
        raise ParameterDomainError("fraction must be in [0, 1)")
    want = math.ceil(fraction * graph.m)
    if want == 0:
        return graph
    n = graph.n
    free = n * (n - 1) // 2 - graph.m
    if want > free:
        raise InfeasibleParametersError(
            f"cannot add {want} edges, only {free} vertex pairs are free")
    rng = np.random.default_rng([seed, _LONG_RANGE_STREAM])
    seen = set()
    new_u = np.empty(want, dtype=np.int64)
    new_v = np.empty(want, dtype=np.int64)
    k = 0
    while k < want:
        a, b = rng.integers(0, n, size=2)
        if a == b:
            continue
        lo, hi = (a, b) if a < b else (b, a)
        if (lo, hi) in seen or graph.has_edge(lo, hi):
            continue
        seen.add((lo, hi))
        new_u[k] = lo
        new_v[k] = hi
        k += 1
    old = graph.edge_array()
    return Graph.from_edge_arrays(n, np.concatenate((old[:, 0], new_u)),
                                  np.concatenate((old[:, 1], new_v)))


__all__ = [
    "DEFAULT_GENERATOR_CAPACITY", "GenerationStats", "GeneratorParams", "VertexCoordinates",
    "add_long_range_edges", "edges_from_coordinates", "generate", "generate_brute_force",
    "generate_with_coordinates",
    "generate_with_stats", "radial_inverse_cdf", "sample_points", "TWO_PI",
]
