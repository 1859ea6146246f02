"""GPU parity: the CUDA path against the reference (golden fixtures) and the
CPU oracle, through the C ABI.  Integer/index results must be bit-exact;
sampled radii (libm vs CUDA asinh/tanh) are compared within a stated ulp
tolerance.  Run on a B200: pytest -m gpu."""

import math

import numpy as np
import pytest

import golden_data as gd
import paper_1501_03545_b200 as P
from paper_1501_03545_b200 import GeneratorParams, Graph, VertexCoordinates

pytestmark = pytest.mark.gpu

RUNS = gd.runs()


def edge_set_hash(oracle, g: Graph):
    return oracle.edge_hash(g.edge_array())


def check_csr(g: Graph):
    """hrgen Graph invariants: symmetric, rows strictly increasing, no loops."""
    ip, ix = np.asarray(g.indptr), np.asarray(g.indices)
    n = ip.size - 1
    assert ip[0] == 0 and np.all(np.diff(ip) >= 0) and ip[-1] == ix.size
    if ix.size == 0:
        return
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ip))
    assert ix.min() >= 0 and ix.max() < n
    assert not np.any(ix == rows)
    inner = np.ones(ix.size - 1, bool)
    starts = ip[1:-1]
    starts = starts[(starts > 0) & (starts < ix.size)]
    inner[starts - 1] = False
    assert np.all(ix[1:][inner] > ix[:-1][inner])
    # symmetry: a random 64-bit multiplicative hash of (row, col) summed over
    # all entries equals the same over (col, row)
    rng = np.random.default_rng(1)
    h1 = rng.integers(1, 2**62, n, dtype=np.int64).astype(np.uint64)
    h2 = rng.integers(1, 2**62, n, dtype=np.int64).astype(np.uint64)
    with np.errstate(over="ignore"):
        a = np.sum(h1[rows] * h2[ix], dtype=np.uint64)
        b = np.sum(h1[ix] * h2[rows], dtype=np.uint64)
    assert a == b


# ---------------------------------------------------------------- arithmetic
def _trig_inputs():
    rng = np.random.default_rng(0)
    u = rng.integers(0, 2**53, 4_000_000, dtype=np.int64).astype(np.float64) * 2.0**-53
    return np.concatenate([
        2 * math.pi * u,                                   # the sampler's angles
        rng.random(2_000_000) * 2 * math.pi,
        np.array([0.0, 5e-324, 1e-300, 1e-8, 2.0**-27, 2.0**-26, 0.126, 0.85546875,
                  2.426265, math.pi / 4, math.pi / 2, math.pi, 3 * math.pi / 2,
                  np.nextafter(2 * math.pi, 0.0)]),
        np.arange(110) / 128.0 + (rng.random(110) - 0.5) * 1e-12,
        math.pi / 2 + (rng.random(10000) - 0.5) * 1e-9,
        math.pi + (rng.random(10000) - 0.5) * 1e-12,
        2 * math.pi - rng.random(10000) * 1e-10,
    ])


def test_device_sincos_matches_numpy():
    """The product's sin/cos (HRG_TRIG_LIBM, the default) are numpy's --
    hrgen's own cos/sin (quadtree.py:474-475) -- bit for bit."""
    eng = P.get_engine()
    x = _trig_inputs()
    s, c = eng.debug_sincos(x, mode=0)
    assert np.array_equal(s, np.sin(x)), np.count_nonzero(s != np.sin(x))
    assert np.array_equal(c, np.cos(x)), np.count_nonzero(c != np.cos(x))


@pytest.mark.parametrize("mode", [1, 2], ids=["fast", "full"])
def test_device_sincos_cr_is_correctly_rounded(oracle, mode):
    eng = P.get_engine()
    x = _trig_inputs()
    s, c = eng.debug_sincos(x, mode=mode)
    s_ref, c_ref = oracle.sincos_cr(x)
    assert np.array_equal(s, s_ref)
    assert np.array_equal(c, c_ref)


def test_fast_sincos_equals_full_evaluation():
    """The gather's fast sin/cos (table + short series + rounding test) is
    bit-identical to the full double-double evaluation (itself pinned to
    __float128 above) on 4e8 seeded angles, a quarter of them within 2^-20 of
    a multiple of pi/4; and the rounding test rejects under 0.2% of them."""
    eng = P.get_engine()
    total_rej = 0
    for seed in range(4):
        mm, rj = eng.debug_sincos_compare(100_000_000, seed)
        assert mm == 0, (seed, mm)
        total_rej += rj
    print(f"[sincos] fast path rejected {total_rej} of 4e8")
    assert total_rej < 0.002 * 4e8


def test_sampler_matches_oracle(oracle):
    """Philox uniforms bit-exact (phi = 2pi*u1 is one multiply); radii from
    CUDA asinh/tanh within 4 ulp of libm's."""
    n, alpha, R, seed = 200_000, 0.75, 28.789361743909193, 2
    co = P.sample_points(n, alpha, R, seed)
    u1, u2 = oracle.philox_uniforms(n, seed)
    k = P.model_constants(R, alpha)
    phi, rn, rp = oracle.sample_from_uniforms(u1, u2, k["two_over_alpha"],
                                             k["sinh_half_alpha_r"], k["r_cap"], k["rp_cap"])
    assert np.array_equal(co.phi, phi)
    assert np.all(np.abs(co.r_native - rn) <= 4 * np.spacing(rn))
    assert np.all(np.abs(co.r_poincare - rp) <= 4 * np.spacing(rp))
    assert co.r_native.max() < R and co.r_poincare.max() < k["max_r"]


def test_sampled_distributions_fit():
    # hrgen tests/test_generator.py:107-116
    from scipy import stats
    alpha, R = 0.7, 16.0
    co = P.sample_points(40_000, alpha, R, seed=123)
    assert stats.kstest(co.phi / (2 * math.pi), "uniform").pvalue > 0.01
    cdf = lambda r: (np.cosh(alpha * r) - 1.0) / (math.cosh(alpha * R) - 1.0)  # noqa: E731
    assert stats.kstest(co.r_native, cdf).pvalue > 0.01


def test_sample_points_deterministic_and_in_range():
    a = P.sample_points(5000, 0.8, 14.0, seed=42)
    b = P.sample_points(5000, 0.8, 14.0, seed=42)
    c = P.sample_points(5000, 0.8, 14.0, seed=43)
    assert np.array_equal(a.phi, b.phi) and np.array_equal(a.r_poincare, b.r_poincare)
    assert not np.array_equal(a.phi, c.phi)
    assert a.phi.min() >= 0.0 and a.phi.max() < 2 * math.pi
    assert a.r_native.max() < 14.0 and a.r_poincare.max() < 1.0


# ---------------------------------------------------- reference edge sets
@pytest.mark.parametrize("run", RUNS, ids=lambda r: f"{r.tag}-n{r.n}-s{r.seed}-R{r.R:.2f}")
def test_reference_runs_bit_exact(oracle, run):
    """On hrgen's own coordinates the GPU edge set IS hrgen's (sha256)."""
    coords = VertexCoordinates(phi=run.phi, r_native=None, r_poincare=run.r_poincare)
    g = P.edges_from_coordinates(coords, run.R, alpha=run.alpha)
    assert g.m == run.m
    assert edge_set_hash(oracle, g) == run.edge_sha256
    check_csr(g)


def _brute_cases():
    import json
    import os
    with open(os.path.join(gd.GOLDEN, "brute.json")) as fh:
        return json.load(fh)


def test_brute_force_equals_reference_brute_force(oracle):
    """GPU all-pairs path == hrgen.generate_brute_force (fixtures made by
    running it, tests/golden/make_brute_golden.py) on 146 golden runs."""
    cases = _brute_cases()
    assert len(cases) >= 140
    runs = gd.runs()
    ties = 0
    for case in cases:
        run = runs[case["run"]]
        coords = VertexCoordinates(phi=run.phi, r_native=None, r_poincare=run.r_poincare)
        g = P.generate_brute_force(coords, run.R)
        ties += P.generate_brute_force.last_near_ties
        assert g.m == case["m"], case
        assert edge_set_hash(oracle, g) == case["edge_sha256"], case
        check_csr(g)
    print(f"[brute] {len(cases)} runs, near ties {ties}")


def test_config0_edges_exact():
    run = gd.runs(["config0"])[0]
    coords = VertexCoordinates(phi=run.phi, r_native=None, r_poincare=run.r_poincare)
    g = P.edges_from_coordinates(coords, run.R)
    assert np.array_equal(g.edge_array(), gd.config0_edges())


# ------------------------------------------------------ generated graphs
GEN_CASES = [
    dict(n=100_000, avg_degree=10.0, gamma=3.0, seed=1),
    dict(n=60_000, avg_degree=32.0, gamma=2.5, seed=2),
    dict(n=50_000, avg_degree=4.0, gamma=2.2, seed=4),
    dict(n=20_000, avg_degree=256.0, gamma=5.0, seed=4),
    dict(n=100_000, radius=33.165607448498854, alpha=1.0, seed=3),
    dict(n=100_000, radius=35.50799080982715, alpha=0.6, seed=4),
]


@pytest.mark.parametrize("kw", GEN_CASES, ids=lambda k: "-".join(f"{a}{b}" for a, b in k.items()))
def test_generate_matches_oracle(oracle, kw):
    """generate() == the oracle quadtree with libm trig (hrgen's arithmetic)
    on the GPU's own coordinates, exactly; with the context in correctly
    rounded mode it equals the CR-trig oracle exactly.  The pairs on which the
    two trig modes disagree are printed with their cosh-distance gap."""
    p = GeneratorParams(**kw)
    model = p.resolve()
    g, st = P.generate_with_stats(p)
    check_csr(g)
    co = P.sample_points(model.n, model.alpha, model.R, p.seed)
    a = P.model_constants(model.R, model.alpha)["cosh_r_minus_1"]
    max_r = P.to_poincare_radius(model.R)
    e_lm, m_lm, _ = oracle.edges_quadtree(co.phi, co.r_poincare, a, model.alpha, max_r, 512,
                                          oracle.TRIG_LIBM)
    assert g.m == m_lm
    assert edge_set_hash(oracle, g) == oracle.edge_hash(e_lm)
    eng = P.get_engine()
    try:
        eng.set_trig(P.TRIG_CR)
        g_cr = P.generate(p)
    finally:
        eng.set_trig(P.TRIG_LIBM)
    e_cr, m_cr, _ = oracle.edges_quadtree(co.phi, co.r_poincare, a, model.alpha, max_r, 512,
                                          oracle.TRIG_CR)
    assert g_cr.m == m_cr and edge_set_hash(oracle, g_cr) == oracle.edge_hash(e_cr)
    d = oracle.compare_edge_sets(e_cr, e_lm, co.phi, co.r_poincare, model.R)
    print(f"[parity] {kw}: m={g.m} candidates={st.candidates} libm==GPU exact; "
          f"CR-vs-libm trig pairs={d['only_got'] + d['only_want']} max_gap={d['max_gap']:.3g}")


@pytest.mark.parametrize("wide", ["0", "1"])
@pytest.mark.parametrize("kw", [GEN_CASES[1], GEN_CASES[2], GEN_CASES[5]],
                         ids=["k32-g2.5", "k4-g2.2", "R35.5"])
def test_light_query_variants_match_oracle(oracle, kw, wide, monkeypatch):
    """Both light-query variants (12 and 36 segment slots; the model picks
    one, HRG_LIGHT_WIDE forces it) give the oracle's edge set exactly."""
    monkeypatch.setenv("HRG_LIGHT_WIDE", wide)
    p = GeneratorParams(**kw)
    model = p.resolve()
    g = P.generate(p)
    co = P.sample_points(model.n, model.alpha, model.R, p.seed)
    a = P.model_constants(model.R, model.alpha)["cosh_r_minus_1"]
    e, m, _ = oracle.edges_quadtree(co.phi, co.r_poincare, a, model.alpha,
                                    P.to_poincare_radius(model.R), 512, oracle.TRIG_LIBM)
    assert g.m == m and np.array_equal(g.edge_array(), e)


@pytest.mark.parametrize("mix", ["0", "3", "32"])
@pytest.mark.parametrize("order", ["sample", "angular"])
def test_tile_order_and_dense_block_match_oracle(oracle, mix, order, monkeypatch):
    """The light pass's tile table (outermost HRG_TILE_MIX bands interleaved by
    an exact rank: every tile must appear exactly once) and its dense block
    (small tile-union windows tested by all 32 queries; with angular ids only
    bands inside every walked band, so rows leave sorted) give the oracle's
    edge set on the GPU's own coordinates, in both vertex orders."""
    monkeypatch.setenv("HRG_TILE_MIX", mix)
    p = GeneratorParams(n=300_000, avg_degree=24.0, gamma=2.6, seed=11, vertex_order=order)
    model = p.resolve()
    g, co = P.generate_with_coordinates(p)
    check_csr(g)
    a = P.model_constants(model.R, model.alpha)["cosh_r_minus_1"]
    e, m, _ = oracle.edges_quadtree(co.phi, co.r_poincare, a, model.alpha,
                                    P.to_poincare_radius(model.R), 512, oracle.TRIG_LIBM)
    assert g.m == m and np.array_equal(g.edge_array(), e)


def test_result_copy_paths_agree(monkeypatch):
    """hrg_copy_result's int64 index copy into host memory has several paths
    (ids widened on the device; crossing PCIe as int32 or, for n <= 2^24, as
    3-byte ids and widened by host threads with non-temporal stores; any split
    between the two; pinned or pageable destination).  All give the int32 copy
    widened by numpy."""
    p = GeneratorParams(n=1_500_000, avg_degree=12.0, gamma=2.8, seed=21)
    eng = P.get_engine()
    eng.generate(p.resolve(), p.seed, P.generator.VERTEX_ORDERS[p.vertex_order])
    ip32, ix32 = eng.copy_csr(np.int32, pinned=False)
    assert ix32.size >= 1 << 22  # large enough for the split paths
    want = ix32.astype(np.int64)
    for frac in ("0", "0.3", "0.97", "1"):
        for pack in ("0", "1"):
            for pinned in (True, False):
                monkeypatch.setenv("HRG_WIDEN_DEVICE_FRAC", frac)
                monkeypatch.setenv("HRG_PACK3", pack)
                ip, ix = eng.copy_csr(np.int64, pinned=pinned)
                assert np.array_equal(ix, want), (frac, pack, pinned)
                assert np.array_equal(ip, ip32)
    monkeypatch.delenv("HRG_WIDEN_DEVICE_FRAC")
    monkeypatch.delenv("HRG_PACK3")
    for _ in range(4):  # the adaptive share
        ip, ix = eng.copy_csr(np.int64, pinned=True)
        assert np.array_equal(ix, want)


def test_config1_full_size_matches_oracle(oracle):
    """BASELINE config 1 (n=1e6, k=10, gamma=3, seed 1) end to end."""
    p = GeneratorParams(n=1_000_000, avg_degree=10.0, gamma=3.0, seed=1)
    model = p.resolve()
    g = P.generate(p)
    co = P.sample_points(model.n, model.alpha, model.R, p.seed)
    a = P.model_constants(model.R, model.alpha)["cosh_r_minus_1"]
    e, m, _ = oracle.edges_quadtree(co.phi, co.r_poincare, a, model.alpha,
                                    P.to_poincare_radius(model.R), 512, oracle.TRIG_LIBM)
    assert g.m == m
    assert edge_set_hash(oracle, g) == oracle.edge_hash(e)
    assert 2 * g.m / model.n == pytest.approx(10.0, rel=0.1)


def test_angular_order_is_hrgen_on_angular_labels(oracle):
    """vertex_order="angular" labels the same point set by (band, angle)
    rank; the edge set is hrgen's rule applied to THOSE labels (the circle of
    the smaller label decides), i.e. the oracle on the angularly ordered
    coordinates, exactly.  Relabelled back to draw order it is the
    sample-order graph except on borderline pairs whose decision depends on
    which circle decides (0 here; 455 of 1.6e8 at config 2 -- see
    tests/test_full_size.py)."""
    kw = dict(n=50_000, avg_degree=16.0, gamma=2.5, seed=7)
    model = GeneratorParams(**kw).resolve()
    gs = P.generate(GeneratorParams(**kw))
    ga = P.generate(GeneratorParams(**kw, vertex_order="angular"))
    check_csr(ga)
    cs = P.sample_points(model.n, model.alpha, model.R, 7)
    ca = P.sample_points(model.n, model.alpha, model.R, 7, vertex_order="angular")
    a = P.model_constants(model.R, model.alpha)["cosh_r_minus_1"]
    e, m, _ = oracle.edges_quadtree(ca.phi, ca.r_poincare, a, model.alpha,
                                    P.to_poincare_radius(model.R), 512, oracle.TRIG_LIBM)
    assert ga.m == m and np.array_equal(ga.edge_array(), e)
    perm = angular_to_sample(cs, ca)
    ea = ga.edge_array()
    mapped = np.sort(np.column_stack((perm[ea[:, 0]], perm[ea[:, 1]])), axis=1)
    mapped = mapped[np.lexsort((mapped[:, 1], mapped[:, 0]))]
    d = oracle.compare_edge_sets(mapped, gs.edge_array(), cs.phi, cs.r_poincare, model.R)
    print(f"[angular] relabelled vs sample order: {d['only_got'] + d['only_want']} pairs differ")
    assert d["only_got"] + d["only_want"] <= max(2, gs.m // 100_000)


def angular_to_sample(cs, ca):
    """perm[angular label] = draw index, by matching (phi, r_poincare)."""
    os_ = np.lexsort((cs.r_poincare, cs.phi))
    oa = np.lexsort((ca.r_poincare, ca.phi))
    assert np.array_equal(cs.phi[os_], ca.phi[oa])
    perm = np.empty(len(ca.phi), np.int64)
    perm[oa] = os_
    return perm


def test_shards_partition_the_rows():
    from paper_1501_03545_b200 import distributed as D
    p = GeneratorParams(n=200_000, avg_degree=16.0, gamma=2.5, seed=9)
    full = P.generate(p)
    model = p.resolve()
    co = P.sample_points(model.n, model.alpha, model.R, p.seed)
    sector = D.sector_of(co.phi, 4)
    acc_rows = np.zeros(full.n, np.int64)
    parts = []
    for k in range(4):
        g, st = P.generate_with_stats(p, shard=P.Shard(k, 4))
        deg = np.diff(g.indptr)
        assert np.all(acc_rows[deg > 0] == 0)   # disjoint row sets
        assert np.all(sector[deg > 0] == k)     # device sectors == host mirror
        acc_rows += deg
        parts.append(g)
    assert np.array_equal(acc_rows, np.diff(full.indptr))
    for g in parts:
        for v in np.flatnonzero(np.diff(g.indptr))[:2000]:
            assert np.array_equal(g.neighbors(v), full.neighbors(v))


@pytest.mark.parametrize("kw,count", [
    (dict(n=5, radius=3.0, alpha=1.0, seed=1), 8),
    (dict(n=3_000, avg_degree=8.0, gamma=3.0, seed=2), 7),
    (dict(n=100_000, radius=35.50799080982715, alpha=0.6, seed=4), 8),
    (dict(n=300_000, avg_degree=64.0, gamma=2.2, seed=4), 8),
], ids=["n5-x8", "n3000-x7", "R35.5-x8", "k64-g2.2-x8"])
def test_shards_union_is_the_graph(oracle, kw, count):
    """Sharded sampling (each rank samples and indexes only the points its
    sector can reach) reproduces the single-GPU graph row for row, and that
    graph is the oracle's (hrgen's quadtree arithmetic) on its coordinates."""
    p = GeneratorParams(**kw)
    full = P.generate(p)
    model = p.resolve()
    co = P.sample_points(model.n, model.alpha, model.R, p.seed)
    a = P.model_constants(model.R, model.alpha)["cosh_r_minus_1"]
    e, m, _ = oracle.edges_quadtree(co.phi, co.r_poincare, a, model.alpha,
                                    P.to_poincare_radius(model.R), 512, oracle.TRIG_LIBM)
    assert full.m == m and np.array_equal(full.edge_array(), e)
    acc = np.zeros(full.n, np.int64)
    for k in range(count):
        g, _ = P.generate_with_stats(p, shard=P.Shard(k, count))
        deg = np.diff(g.indptr)
        assert np.all(acc[deg > 0] == 0)
        acc += deg
        rows = np.flatnonzero(deg)
        if rows.size:
            sel = np.concatenate([rows[:300], rows[np.argsort(deg[rows])[-20:]]])
            for v in sel:
                assert np.array_equal(g.neighbors(v), full.neighbors(v))
    assert np.array_equal(acc, np.diff(full.indptr))


def test_shards_from_coordinates(oracle):
    """Sharded runs on caller-given coordinates (hrgen's own, R = 33.2) give
    the reference rows; their union is the reference graph."""
    run = max([r for r in RUNS if r.n >= 10_000], key=lambda r: r.R)
    coords = VertexCoordinates(phi=run.phi, r_native=None, r_poincare=run.r_poincare)
    full = P.edges_from_coordinates(coords, run.R, alpha=run.alpha)
    assert edge_set_hash(oracle, full) == run.edge_sha256
    acc = np.zeros(full.n, np.int64)
    for k in range(5):
        g = P.edges_from_coordinates(coords, run.R, alpha=run.alpha, shard=P.Shard(k, 5))
        deg = np.diff(g.indptr)
        assert np.all(acc[deg > 0] == 0)
        acc += deg
        for v in np.flatnonzero(deg)[:500]:
            assert np.array_equal(g.neighbors(v), full.neighbors(v))
    assert np.array_equal(acc, np.diff(full.indptr))


# ------------------------------------------------------------ properties
def test_full_size_config2_properties():
    """BASELINE config 2 (n=1e7, k=32, gamma=2.5, seed 2): hrgen Graph
    invariants and the realised degree at full size."""
    p = GeneratorParams(n=10_000_000, avg_degree=32.0, gamma=2.5, seed=2)
    g, st = P.generate_with_stats(p)
    check_csr(g)
    assert 2 * g.m / p.n == pytest.approx(32.0, rel=0.12)
    print(f"[config2] m={g.m} candidates={st.candidates} "
          f"t_sample={st.t_sample_ns/1e6:.2f}ms t_build={st.t_build_ns/1e6:.2f}ms "
          f"t_edges={st.t_edges_ns/1e6:.2f}ms")


def test_realized_degree_tracks_target():
    # hrgen tests/test_generator.py:177-185
    for alpha, kbar in ((1.0, 16.0), (1.5, 8.0)):
        g = P.generate(GeneratorParams(n=50_000, avg_degree=kbar, alpha=alpha, seed=1))
        assert 2.0 * g.m / 50_000 == pytest.approx(kbar, rel=0.05)


def test_determinism_and_invariance():
    base = dict(n=25_000, avg_degree=12.0, gamma=2.8, seed=4)
    g1 = P.generate(GeneratorParams(**base, threads=1, leaf_capacity=32))
    g2 = P.generate(GeneratorParams(**base, threads=3, leaf_capacity=2048))
    assert np.array_equal(g1.indptr, g2.indptr) and np.array_equal(g1.indices, g2.indices)
    g3 = P.generate(GeneratorParams(**{**base, "seed": 5}))
    assert not np.array_equal(g1.indices, g3.indices)


# ------------------------------------------------------------ edge cases
def test_single_vertex_and_tiny_graphs():
    g = P.generate(GeneratorParams(n=1, radius=5.0, alpha=1.0, seed=0))
    assert g.n == 1 and g.m == 0
    g = P.generate(GeneratorParams(n=2, radius=0.5, alpha=1.0, seed=0))
    assert g.n == 2 and g.m == 1


def test_degenerate_coordinates(oracle):
    """Duplicates, the origin, angles 0 and just below 2pi, rim points."""
    R = 12.0
    max_r = P.to_poincare_radius(R)
    rim = np.nextafter(max_r, 0.0)
    phi = np.array([0.0, 0.0, 1.0, 1.0, 1.0, np.nextafter(2 * math.pi, 0), 3.0, 3.0 + 1e-15,
                    math.pi, 0.5])
    rp = np.array([0.0, 0.5, 0.9, 0.9, 0.9, rim, rim, rim, 0.9999, 1e-300])
    coords = VertexCoordinates(phi=phi, r_native=None, r_poincare=rp)
    g = P.edges_from_coordinates(coords, R)
    a = P.model_constants(R, 1.0)["cosh_r_minus_1"]
    want = oracle.edges_brute(phi, rp, a)
    assert np.array_equal(g.edge_array(), want)


def test_random_coordinates_many_radii(oracle):
    rng = np.random.default_rng(3)
    for R in (0.3, 2.0, 9.0, 20.0, 30.0, 37.0):
        n = 3000
        max_r = P.to_poincare_radius(R)
        phi = rng.random(n) * 2 * math.pi
        rp = np.minimum(np.sqrt(rng.random(n)) * max_r, np.nextafter(max_r, 0))
        rp[: n // 3] = np.nextafter(max_r, 0) - rng.integers(0, 8, n // 3) * np.spacing(max_r)
        rp = np.minimum(rp, np.nextafter(max_r, 0))
        a = P.model_constants(R, 1.0)["cosh_r_minus_1"]
        want = oracle.edges_brute(phi, rp, a, oracle.TRIG_LIBM)
        g = P.edges_from_coordinates(VertexCoordinates(phi, None, rp), R)
        assert np.array_equal(g.edge_array(), want), R


def test_out_of_bounds_coordinates_raise():
    R = 10.0
    with pytest.raises(P.OutOfBoundsError):
        P.edges_from_coordinates(VertexCoordinates(np.array([0.0]), None, np.array([0.99995])), R)
    with pytest.raises(P.OutOfBoundsError):
        P.edges_from_coordinates(VertexCoordinates(np.array([-0.1]), None, np.array([0.5])), R)
    with pytest.raises(P.OutOfBoundsError):
        P.edges_from_coordinates(VertexCoordinates(np.array([2 * math.pi]), None,
                                                   np.array([0.5])), R)
    with pytest.raises(ValueError):
        P.generate(GeneratorParams(n=10, radius=80.0, alpha=1.0))


def test_two_contexts_concurrently():
    """Two generator contexts on their own streams, driven from two host
    threads at once (bench.py's e2e pattern), each reproduce the graph."""
    import threading
    import torch
    p = GeneratorParams(n=200_000, avg_degree=24.0, gamma=2.4, seed=11)
    ref = P.generate(p)
    model = p.resolve()
    streams = [torch.cuda.Stream() for _ in range(2)]
    engines = [P.Engine(0, stream=s.cuda_stream) for s in streams]
    out = {}

    def run(w):
        res = []
        for _ in range(3):
            engines[w].generate(model, p.seed)
            res.append(engines[w].copy_csr(np.int64))
        out[w] = res

    ths = [threading.Thread(target=run, args=(w,)) for w in range(2)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for w in range(2):
        for ip, ix in out[w]:
            assert np.array_equal(ip, ref.indptr) and np.array_equal(ix, ref.indices)


def test_device_csr_tensors():
    import torch
    eng = P.get_engine()
    g = P.generate(GeneratorParams(n=20_000, avg_degree=8.0, gamma=3.0, seed=1))
    ip, ix = eng.device_csr()
    assert ip.is_cuda and ix.dtype == torch.int32
    assert np.array_equal(ip.cpu().numpy(), g.indptr)
    assert np.array_equal(ix.cpu().numpy().astype(np.int64), g.indices)


@pytest.mark.parametrize("order", ["angle", "shuffled", "blocks"])
def test_hub_rows_any_id_order(oracle, order):
    """Rows far above one block's capacity (hubs near the origin) with ids in
    angular order (clustered, non-uniform in every row), shuffled (uniform)
    and in interleaved angular blocks: the long-row sorts (block bucket sort,
    giant-row split, bitonic fallback) must give hrgen's sorted rows."""
    rng = np.random.default_rng(11)
    n, R, alpha = 120_000, 14.0, 0.55
    max_r = P.to_poincare_radius(R)
    u = rng.random(n)
    r = np.arccosh(1 + (np.cosh(alpha * R) - 1) * u) / alpha
    rp = np.minimum(np.tanh(r / 2), np.nextafter(max_r, 0))
    phi = rng.random(n) * 2 * math.pi
    rp[:6] = [0.0, 0.01, 0.05, 0.2, 0.4, 0.6]  # hubs
    if order == "angle":
        perm = np.argsort(phi, kind="stable")
    elif order == "shuffled":
        perm = rng.permutation(n)
    else:
        perm = np.argsort(phi, kind="stable").reshape(-1, 1000)[rng.permutation(n // 1000)].ravel()
    phi, rp = phi[perm], rp[perm]
    coords = VertexCoordinates(phi=phi, r_native=None, r_poincare=rp)
    g = P.edges_from_coordinates(coords, R)
    check_csr(g)
    assert np.diff(g.indptr).max() > 40_000
    a = P.model_constants(R, alpha)["cosh_r_minus_1"]
    e, m, _ = oracle.edges_quadtree(phi, rp, a, alpha, max_r, 512, oracle.TRIG_LIBM)
    assert g.m == m
    assert edge_set_hash(oracle, g) == oracle.edge_hash(e)


def test_staging_regrowth_after_small_graph():
    """The staging buffer is sized from the previous call on a context; a
    much larger graph right after a tiny one overflows it, the pass is voided
    on the device and re-run, and the result equals a warm run's."""
    eng = P.get_engine()
    P.generate(GeneratorParams(n=2_000, avg_degree=6.0, gamma=3.0, seed=5))
    p = GeneratorParams(n=400_000, avg_degree=24.0, gamma=2.3, seed=6)
    g1 = P.generate(p)
    g2 = P.generate(p)
    check_csr(g1)
    assert np.array_equal(g1.indptr, g2.indptr) and np.array_equal(g1.indices, g2.indices)


def test_reference_pruning_drop_fixture(oracle):
    """On hrgen's coordinates where hrgen's quadtree drops a pair its own
    predicate accepts (tests/golden/make_prune_golden.py), the GPU returns
    the predicate's edge set: hrgen's edges plus exactly that rim pair."""
    import os
    z = np.load(os.path.join(gd.GOLDEN, "prune_drop.npz"))
    coords = VertexCoordinates(phi=z["phi"], r_native=None, r_poincare=z["r_poincare"])
    g = P.edges_from_coordinates(coords, float(z["R"]), alpha=float(z["alpha"]))
    assert np.array_equal(g.edge_array(), z["allpairs_edges"])
    d = oracle.compare_edge_sets(g.edge_array(), z["hrgen_edges"], z["phi"], z["r_poincare"],
                                 float(z["R"]))
    assert d["only_got"] == 1 and d["only_want"] == 0


def test_generate_with_coordinates(oracle):
    """Coordinates plus edge list from one generation: the coordinates are
    sample_points' and the graph is the oracle's edge set on them."""
    p = GeneratorParams(n=30_000, avg_degree=12.0, gamma=2.7, seed=21)
    model = p.resolve()
    g, co = P.generate_with_coordinates(p)
    ref = P.sample_points(model.n, model.alpha, model.R, p.seed)
    assert np.array_equal(co.phi, ref.phi) and np.array_equal(co.r_poincare, ref.r_poincare)
    assert np.array_equal(co.r_native, ref.r_native)
    a = P.model_constants(model.R, model.alpha)["cosh_r_minus_1"]
    e, m, _ = oracle.edges_quadtree(co.phi, co.r_poincare, a, model.alpha,
                                    P.to_poincare_radius(model.R), 512, oracle.TRIG_LIBM)
    assert g.m == m and np.array_equal(g.edge_array(), e)
