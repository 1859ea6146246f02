"""Host-side logic of the drop-in API (no GPU): parameter handling,
the radius solver and derived constants (bit-identical to hrgen, pinned by
golden fixtures), the Graph container and the long-range augmentation."""

import math

import numpy as np
import pytest

import golden_data as gd
import paper_1501_03545_b200 as P
from paper_1501_03545_b200 import (
    GeneratorParams,
    Graph,
    InfeasibleParametersError,
    ParameterDomainError,
)


def test_params_require_exactly_one_of_each_pair():
    # mirrors hrgen tests/test_generator.py:29-49
    bad = [
        dict(n=10, gamma=3.0),
        dict(n=10, avg_degree=4.0, radius=10.0, gamma=3.0),
        dict(n=10, avg_degree=4.0),
        dict(n=10, avg_degree=4.0, gamma=3.0, alpha=1.0),
        dict(n=0, avg_degree=4.0, gamma=3.0),
        dict(n=10, avg_degree=4.0, gamma=2.0),
        dict(n=10, avg_degree=4.0, alpha=0.5),
        dict(n=10, avg_degree=4.0, gamma=3.0, seed=-1),
        dict(n=10, avg_degree=4.0, gamma=3.0, seed=2**64),
        dict(n=10, avg_degree=4.0, gamma=3.0, long_range_fraction=1.0),
        dict(n=10, avg_degree=4.0, gamma=3.0, threads=0),
        dict(n=10, avg_degree=4.0, gamma=3.0, leaf_capacity=0),
        dict(n=10, avg_degree=4.0, gamma=3.0, vertex_order="random"),
    ]
    for kw in bad:
        with pytest.raises(ParameterDomainError):
            GeneratorParams(**kw)


def test_resolve_translates_gamma_and_degree():
    m = GeneratorParams(n=1000, avg_degree=8.0, gamma=3.0).resolve()
    assert m.alpha == pytest.approx(1.0) and m.n == 1000 and m.R > 0
    q = GeneratorParams(n=1000, radius=12.0, alpha=0.75).resolve()
    assert q.R == 12.0 and q.target_avg_degree is None


def test_target_radius_bit_identical_to_reference():
    for row in gd.target_radius_table():
        alpha = (row["gamma"] - 1.0) / 2.0
        if "R" in row:
            assert P.target_radius(row["n"], row["k"], alpha) == float.fromhex(row["R"]), row
        else:
            with pytest.raises(ValueError) as ei:
                P.target_radius(row["n"], row["k"], alpha)
            assert type(ei.value).__name__ == row["error"]


def test_model_constants_bit_identical_to_reference():
    for run in gd.runs():
        c = P.model_constants(run.R, run.alpha)
        assert c["cosh_r_minus_1"] == run.a
        assert c["max_r"] == run.max_r
        assert c["rp_cap"] == run.rp_cap


def test_infeasible_degree_raises():
    with pytest.raises(InfeasibleParametersError):
        P.target_radius(100, 64.0, 1.0)   # hrgen test_acceptance.py:70-76
    with pytest.raises(ParameterDomainError):
        P.target_radius(10, 20.0, 1.0)


def test_radial_inverse_cdf_inverts_cdf():
    rng = np.random.default_rng(0)
    for _ in range(200):
        u, alpha, R = rng.random(), rng.uniform(0.55, 3.0), rng.uniform(2.0, 25.0)
        r = P.radial_inverse_cdf(u, alpha, R)
        assert 0.0 <= r <= R
        cdf = (math.cosh(alpha * r) - 1.0) / (math.cosh(alpha * R) - 1.0)
        assert cdf == pytest.approx(u, abs=1e-9)
    with pytest.raises(ValueError):
        P.radial_inverse_cdf(1.1, 1.0, 10.0)


def test_graph_contract():
    g = Graph.from_edges(5, [(0, 1), (3, 1), (4, 2)])
    assert g.n == 5 and g.m == 3
    assert g.neighbors(1).tolist() == [0, 3]
    assert g.has_edge(1, 3) and g.has_edge(3, 1) and not g.has_edge(0, 4)
    assert g.edge_array().tolist() == [[0, 1], [1, 3], [2, 4]]
    with pytest.raises(ValueError):
        Graph.from_edges(3, [(0, 0)])
    with pytest.raises(ValueError):
        Graph.from_edges(3, [(0, 1), (1, 0)])
    with pytest.raises(ValueError):
        Graph.from_edges(3, [(0, 3)])


@pytest.mark.parametrize("row", gd.long_range_table(), ids=lambda r: f"n{r['n']}")
def test_long_range_bit_identical_to_reference(oracle, row):
    """hrgen.add_long_range_edges on the reference base graph (rebuilt by the
    oracle from the reference coordinates) -> same augmented edge set."""
    tag = "lr1" if row["n"] == 3000 else "lr2"
    run = gd.runs([tag])[0]
    pairs = oracle.edges_brute(run.phi, run.r_poincare, run.a)
    assert oracle.edge_hash(pairs) == row["base_sha256"]
    base = Graph.from_edge_arrays(run.n, pairs[:, 0], pairs[:, 1])
    aug = P.add_long_range_edges(base, row["fraction"], seed=row["seed"])
    assert aug.m == row["m"]
    assert oracle.edge_hash(aug.edge_array()) == row["edge_sha256"]


def test_long_range_rejects_full_graph():
    full = Graph.from_edges(4, [(a, b) for a in range(4) for b in range(a + 1, 4)])
    with pytest.raises(InfeasibleParametersError):
        P.add_long_range_edges(full, 0.5, seed=0)
