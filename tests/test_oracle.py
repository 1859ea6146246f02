"""The CPU oracle is pinned to the reference before it is trusted.

Every fixture in tests/golden/ was produced by running hrgen itself
(tests/golden/make_golden.py).  These tests need no GPU.
"""

import math

import numpy as np
import pytest

import golden_data as gd

RUNS = gd.runs()
SMALL = [r for r in RUNS if r.n <= 3000]
LARGE = [r for r in RUNS if r.n > 3000]


def test_phi_regenerates_exactly():
    # golden_data asserts the sha256 of phi for every run on load
    assert len(RUNS) >= 150


@pytest.mark.parametrize("run", SMALL, ids=lambda r: f"{r.tag}-n{r.n}-s{r.seed}-R{r.R:.2f}")
def test_brute_force_oracle_matches_reference(oracle, run):
    """orc_edges_brute == hrgen.generate edge set, bit for bit (sha256)."""
    e = oracle.edges_brute(run.phi, run.r_poincare, run.a, oracle.TRIG_LIBM)
    assert len(e) == run.m
    assert oracle.edge_hash(e) == run.edge_sha256


@pytest.mark.parametrize("run", RUNS, ids=lambda r: f"{r.tag}-n{r.n}-s{r.seed}-R{r.R:.2f}")
def test_quadtree_oracle_matches_reference(oracle, run):
    """The restated polar quadtree (build/pack/query_many) reproduces hrgen."""
    e, m, _ = oracle.edges_quadtree(run.phi, run.r_poincare, run.a, run.alpha, run.max_r, 512,
                                    oracle.TRIG_LIBM)
    assert m == run.m
    assert oracle.edge_hash(e) == run.edge_sha256


@pytest.mark.parametrize("capacity", [1, 7, 128, 2048])
def test_quadtree_capacity_invariance(oracle, capacity):
    """hrgen tests/test_generator.py:170-174: leaf capacity never changes the edges."""
    run = gd.runs(["config0"])[0]
    e, m, _ = oracle.edges_quadtree(run.phi, run.r_poincare, run.a, run.alpha, run.max_r,
                                    capacity, oracle.TRIG_LIBM)
    assert oracle.edge_hash(e) == run.edge_sha256


def test_config0_full_edges(oracle):
    run = gd.runs(["config0"])[0]
    want = gd.config0_edges()
    got = oracle.edges_brute(run.phi, run.r_poincare, run.a, oracle.TRIG_LIBM)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("trig", [0, 1])
def test_rows_brute_matches_whole_edge_set(oracle, trig):
    """orc_rows_brute (sampled full rows, the full-size parity checker) equals
    the rows of the all-pairs edge set, on reference runs incl. large R."""
    rng = np.random.default_rng(3)
    runs = [r for r in RUNS if r.n >= 10_000][:4] + [max(RUNS, key=lambda r: r.R)]
    for run in runs:
        pairs = oracle.edges_brute(run.phi, run.r_poincare, run.a, trig)
        ip, ix = oracle.csr_from_pairs(run.n, pairs)
        q = np.concatenate([rng.choice(run.n, 60, replace=False),
                            np.argsort(np.diff(ip))[-4:], [0, run.n - 1]])
        rp, ri = oracle.rows_brute(run.phi, run.r_poincare, run.a, q, trig)
        for k, v in enumerate(q):
            assert np.array_equal(ri[rp[k]:rp[k + 1]], ix[ip[v]:ip[v + 1]]), (run.tag, v)


def test_trig_modes_agree_on_reference_runs(oracle):
    """Correctly rounded sin/cos (what the GPU computes) and libm (what numpy
    computes) give the same edge sets on every golden run."""
    for run in [r for r in RUNS if r.n >= 10_000]:
        e_cr, _, _ = oracle.edges_quadtree(run.phi, run.r_poincare, run.a, run.alpha, run.max_r,
                                           512, oracle.TRIG_CR)
        assert oracle.edge_hash(e_cr) == run.edge_sha256, run


def test_csr_matches_reference_graph_layout(oracle):
    run = gd.runs(["config0"])[0]
    e = gd.config0_edges()
    indptr, indices = oracle.csr_from_pairs(run.n, e)
    assert indptr[-1] == 2 * run.m
    # rows sorted, symmetric
    for v in range(0, run.n, 97):
        row = indices[indptr[v]:indptr[v + 1]]
        assert np.all(np.diff(row) > 0)
        for w in row[:5]:
            rw = indices[indptr[w]:indptr[w + 1]]
            assert v in rw


def test_philox_known_answers(oracle):
    """Philox4x32-10 known-answer vectors (Salmon et al. SC'11 / Random123
    kat_vectors): counter 0 / key 0, all-ones, and the pi-digits vector."""
    assert oracle.philox_raw([0, 0, 0, 0], [0, 0]) == [0x6627e8d5, 0xe169c58d, 0xbc57ac4c,
                                                       0x9b00dbd8]
    ones = 0xffffffff
    assert oracle.philox_raw([ones] * 4, [ones, ones]) == [0x408f276d, 0x41c83b0e, 0xa20bc7c6,
                                                         0x6d5451fd]
    assert oracle.philox_raw([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344],
                             [0xa4093822, 0x299f31d0]) == [0xd16cfe09, 0x94fdcceb, 0x5001e420,
                                                           0x24126ea1]
    # and the uniforms the sampler derives from counter (i, 0, 0, 0):
    u1, u2 = oracle.philox_uniforms(4, 0, 0)
    # counter 0, key 0 -> 0x6627e8d5 0xe169c58d 0xbc57ac4c 0x9b00dbd8
    a = (0xe169c58d << 32 | 0x6627e8d5) >> 11
    b = (0x9b00dbd8 << 32 | 0xbc57ac4c) >> 11
    assert u1[0] == a * 2.0**-53
    assert u2[0] == b * 2.0**-53


def test_cr_sincos_is_correctly_rounded(oracle):
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.prec = 256
    rng = np.random.default_rng(5)
    x = np.concatenate([
        rng.random(3000) * 2 * math.pi,
        np.array([0.0, 5e-324, 1e-300, math.pi / 2, math.pi, 3 * math.pi / 2,
                  np.nextafter(2 * math.pi, 0.0), 0.7853981633974483, 2.356194490192345]),
        math.pi / 2 + (rng.random(200) - 0.5) * 1e-9,
        math.pi + (rng.random(200) - 0.5) * 1e-12,
    ])
    s, c = oracle.sincos_cr(x)

    def cr(f, v):
        exact = f(mpmath.mpf(float(v)))
        best = float(exact)
        for cand in (np.nextafter(best, -np.inf), best, np.nextafter(best, np.inf)):
            if abs(mpmath.mpf(float(cand)) - exact) < abs(mpmath.mpf(best) - exact):
                best = float(cand)
        return best

    for v, sv, cv in zip(x, s, c):
        assert sv == cr(mpmath.sin, v), v
        assert cv == cr(mpmath.cos, v), v


def test_libm_cos_vs_correct_rounding_rate(oracle):
    """Documents how often glibc's cos/sin (numpy's) differ from correct
    rounding on uniform angles: a fraction of a percent, never more than 1 ulp."""
    rng = np.random.default_rng(11)
    x = rng.random(200_000) * 2 * math.pi
    s, c = oracle.sincos_cr(x)
    dc = np.cos(x) != c
    ds = np.sin(x) != s
    assert dc.mean() < 0.01 and ds.mean() < 0.01
    ulp = np.abs(np.cos(x)[dc] - c[dc]) / np.spacing(np.abs(c[dc]))
    assert np.all(ulp <= 1.0)


def test_sampler_formula_matches_reference_expression(oracle):
    """orc_sample_from_uniforms is hrgen's radial_inverse_cdf + clamps
    (generator.py:156-178) evaluated with libm."""
    rng = np.random.default_rng(3)
    u1 = rng.random(10000)
    u2 = rng.random(10000)
    alpha, R = 0.75, 28.789361743909193
    from paper_1501_03545_b200.geometry import model_constants
    k = model_constants(R, alpha)
    phi, rn, rp = oracle.sample_from_uniforms(u1, u2, k["two_over_alpha"], k["sinh_half_alpha_r"],
                                             k["r_cap"], k["rp_cap"])
    assert np.array_equal(phi, 2.0 * math.pi * u1)
    want = (2.0 / alpha) * np.arcsinh(np.sqrt(u2) * math.sinh(alpha * R / 2.0))
    want = np.minimum(want, np.nextafter(R, 0.0))
    assert np.allclose(rn, want, rtol=4e-16, atol=0)
    assert np.all(rp < k["max_r"])


def test_reference_pruning_drop_fixture(oracle):
    """tests/golden/prune_drop.npz (made by running hrgen): hrgen's quadtree
    drops exactly one pair that its own leaf predicate accepts, a pair with a
    point 1 ulp below the rim; the oracle's all-pairs predicate finds it."""
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "prune_drop.npz"))
    ref, allp = z["hrgen_edges"], z["allpairs_edges"]
    assert len(allp) == len(ref) + 1
    d = oracle.compare_edge_sets(allp, ref, z["phi"], z["r_poincare"], float(z["R"]))
    assert d["only_got"] == 1 and d["only_want"] == 0
    a = float(2.0 * np.sinh(np.asarray(float(z["R"])) / 2.0) ** 2)
    cls = oracle.classify_mismatches(d, z["phi"], z["r_poincare"], a)
    assert cls == {"band": 0, "ref_drop": 1, "unexplained": 0}
    again = oracle.edges_brute(z["phi"], z["r_poincare"], a, oracle.TRIG_LIBM)
    assert np.array_equal(again, allp)
