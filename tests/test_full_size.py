"""Full-size parity for BASELINE configs 2, 3 and the config-4 sweep.

* config 2 (the benchmarked graph, n = 1e7): the WHOLE edge set against the
  oracle's restatement of hrgen's polar quadtree with libm trig -- hrgen's
  own arithmetic -- on the GPU's coordinates (about 75 s on 16 host cores).
  Any pair the two disagree on must lie in the north star's exception band,
  |cosh d - cosh R| <= 1e-12 cosh R (checked in __float128); the count and
  the largest gap are printed (and appended to $HRG_PARITY_LOG if set).
* config 3 (n = 1e8) and the nine config-4 points (n = 1e7): every row of
  a contiguous slice of 10^6 query ids (all pairs whose smaller id is in the
  slice) against the oracle quadtree on the same slice, exactly; plus
  hrgen's Graph invariants over the WHOLE device CSR (row pointers, ids in
  range, no loops, strictly increasing rows, symmetry via a checksum of
  checksums) and a sample of rows (random vertices, the largest hubs, the
  first and last id) against the oracle's all-pairs rows.
Run on a B200: pytest -m gpu."""

import json
import os

import numpy as np
import pytest

import paper_1501_03545_b200 as P
from paper_1501_03545_b200 import GeneratorParams

pytestmark = pytest.mark.gpu

CONFIG2 = dict(n=10_000_000, avg_degree=32.0, gamma=2.5, seed=2)
CONFIG3 = dict(n=100_000_000, avg_degree=16.0, gamma=3.0, seed=3)
SWEEP = [dict(n=10_000_000, avg_degree=k, gamma=g, seed=4)
         for k in (4.0, 64.0, 256.0) for g in (2.2, 3.0, 5.0)]
SLICE_CASES = ([dict(CONFIG2, vertex_order="angular")] + SWEEP + [CONFIG3])
CHUNK = 1 << 27
SLICE = 1_000_000


def case_id(k):
    return (f"n{k['n']:.0e}-k{k['avg_degree']:g}-g{k['gamma']:g}-s{k['seed']}"
            + ("-angular" if "vertex_order" in k else ""))


def log_parity(record):
    print(f"[parity] {json.dumps(record)}")
    path = os.environ.get("HRG_PARITY_LOG")
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps(record) + "\n")


def device_invariants(ip, ix, n):
    """hrgen Graph invariants (graph.py:52-77) over the whole device CSR,
    in chunks; returns the degree vector (device)."""
    import torch
    nnz = ix.numel()
    assert int(ip[0]) == 0 and int(ip[-1]) == nnz
    deg = ip[1:] - ip[:-1]
    assert bool((deg >= 0).all())
    g = torch.Generator(device=ip.device)
    g.manual_seed(1)
    h1 = torch.randint(1, 2**62, (n,), device=ip.device, dtype=torch.int64, generator=g)
    h2 = torch.randint(1, 2**62, (n,), device=ip.device, dtype=torch.int64, generator=g)
    a = torch.zeros((), dtype=torch.int64, device=ip.device)
    b = torch.zeros((), dtype=torch.int64, device=ip.device)
    for s in range(0, nnz, CHUNK):
        e = min(nnz, s + CHUNK + 1)   # one entry of overlap for the order check
        pos = torch.arange(s, e, device=ip.device, dtype=torch.int64)
        row = torch.searchsorted(ip, pos, right=True) - 1
        col = ix[s:e].to(torch.int64)
        assert bool(((col >= 0) & (col < n)).all())
        assert not bool((col == row).any())
        same = row[1:] == row[:-1]
        assert bool((col[1:][same] > col[:-1][same]).all())
        w = slice(0, min(CHUNK, e - s))    # hash each entry once
        a += (h1[row[w]] * h2[col[w]]).sum()
        b += (h1[col[w]] * h2[row[w]]).sum()
    assert int(a) == int(b), "CSR is not symmetric"
    return deg


def upper_pairs(ip, ix, lo, hi, row0=0):
    """(v, w) pairs with v in [lo, hi) and w > v from a host CSR whose row k
    is vertex row0 + k, in the lexicographic order of hrgen's
    Graph.edge_array (graph.py:38-42)."""
    s, e = int(ip[lo]), int(ip[hi])
    rows = np.repeat(np.arange(row0 + lo, row0 + hi, dtype=np.int64), np.diff(ip[lo:hi + 1]))
    cols = np.asarray(ix[s:e], dtype=np.int64)
    keep = cols > rows
    return np.column_stack((rows[keep], cols[keep]))


def test_config2_whole_edge_set(oracle):
    """BASELINE config 2, every edge: GPU == hrgen's quadtree arithmetic."""
    p = GeneratorParams(**CONFIG2)
    model = p.resolve()
    eng = P.get_engine()
    with eng.lock:
        st = eng.generate(model, p.seed)
        ip, ix = eng.copy_csr(np.int64, pinned=False)
        phi, _, rp = eng.copy_coords()
    got = upper_pairs(ip, ix, 0, model.n)
    del ix
    consts = P.model_constants(model.R, model.alpha)
    want, m, tm = oracle.edges_quadtree(phi, rp, consts["cosh_r_minus_1"], model.alpha,
                                        consts["max_r"], 512, oracle.TRIG_LIBM)
    d = oracle.compare_edge_sets(got, want, phi, rp, model.R)
    cls = oracle.classify_mismatches(d, phi, rp, consts["cosh_r_minus_1"])
    log_parity(dict(case="config2", scope="whole edge set", n=model.n, m_gpu=d["m_got"],
                    m_ref=d["m_want"], only_gpu=d["only_got"], only_ref=d["only_want"],
                    max_rel_gap=d["max_gap"], outside_band=d["outside_band"], **cls,
                    ref="oracle quadtree, libm trig", t_ref_query_s=tm.t_query_s))
    assert cls["unexplained"] == 0
    assert d["only_got"] + d["only_want"] == cls["band"] + cls["ref_drop"]
    assert st.m == len(got)


@pytest.mark.parametrize("kw", SLICE_CASES, ids=case_id)
def test_full_size_slice_and_invariants(oracle, kw):
    import torch
    p = GeneratorParams(**kw)
    model = p.resolve()
    eng = P.get_engine()
    n = model.n
    with eng.lock:
        st = eng.generate(model, p.seed, P.generator.VERTEX_ORDERS[p.vertex_order])
        ip, ix = eng.device_csr()
        phi, _, rp = eng.copy_coords()
    deg = device_invariants(ip, ix, n)
    m = int(ip[-1]) // 2
    assert m == st.m
    # realised average degree near the target (hrgen's solver targets the
    # expectation; at gamma=2.2 the hub tail makes it noisier)
    assert 2 * m / n == pytest.approx(kw["avg_degree"], rel=0.2 if kw["gamma"] < 2.5 else 0.12)
    consts = P.model_constants(model.R, model.alpha)
    a = consts["cosh_r_minus_1"]

    # (1) a contiguous slice of query ids, every row, exact
    rng = np.random.default_rng(kw["seed"] + 11)
    lo = int(rng.integers(0, n - SLICE))
    hi = lo + SLICE
    ipq = ip[lo:hi + 1].cpu().numpy()
    got = upper_pairs(ipq - ipq[0], ix[int(ipq[0]):int(ipq[-1])].cpu().numpy(), 0, SLICE, row0=lo)
    want, mw, tm = oracle.edges_quadtree(phi, rp, a, model.alpha, consts["max_r"], 512,
                                         oracle.TRIG_LIBM, 0, lo, hi)
    d = oracle.compare_edge_sets(got, want, phi, rp, model.R)
    cls = oracle.classify_mismatches(d, phi, rp, a)
    log_parity(dict(case=case_id(kw), scope=f"rows [{lo}, {hi}) (pairs with smaller id there)",
                    n=n, m_gpu_slice=d["m_got"], m_ref_slice=d["m_want"],
                    only_gpu=d["only_got"], only_ref=d["only_want"], max_rel_gap=d["max_gap"],
                    outside_band=d["outside_band"], **cls, ref="oracle quadtree, libm trig"))
    # every difference is either in the north star's band or a pair the
    # reference's quadtree prunes although its own predicate accepts it
    # (rim points; oracle.classify_mismatches) -- none unexplained
    assert cls["unexplained"] == 0

    # (2) sampled rows incl. hubs against all-pairs rows
    hubs = torch.topk(deg, 6).indices.cpu().numpy()
    q = np.unique(np.concatenate([rng.choice(n, 40, replace=False), hubs, [0, n - 1]]))
    oi, ox = oracle.rows_brute(phi, rp, a, q, oracle.TRIG_LIBM)
    for k, v in enumerate(q.tolist()):
        s, e = int(ip[v]), int(ip[v + 1])
        got_row = ix[s:e].cpu().numpy().astype(np.int64)
        assert np.array_equal(got_row, ox[oi[k]:oi[k + 1]]), (v, got_row.size)
    print(f"[full] {kw}: R={model.R:.4f} m={m} candidates={st.candidates} "
          f"max_deg={int(deg.max())} slice_pairs={d['m_got']} rows_checked={q.size} "
          f"t_edges={st.t_edges_ms:.2f}ms")


def test_config2_angular_vs_sample_order(oracle):
    """The angular labelling is NOT a relabelling of the sample-order graph
    at this size: the circle of the smaller label decides a pair, and on
    borderline pairs (the predicate is not symmetric under rounding, and is
    ill-conditioned near the rim) the two labellings decide differently:
    1601 of 1.6e8 pairs at config 2 (largest cosh-distance gap 3e-4).  Each
    labelling is hrgen's own rule on its labels (checked exactly above and in
    tests/test_gpu_parity.py); this states the size of the difference."""
    p = GeneratorParams(**CONFIG2)
    model = p.resolve()
    eng = P.get_engine()
    with eng.lock:
        eng.generate(model, p.seed)
        ips, ixs = eng.copy_csr(np.int64, pinned=False)
        cs = eng.copy_coords()
        eng.generate(model, p.seed, P.generator.VERTEX_ORDERS["angular"])
        ipa, ixa = eng.copy_csr(np.int64, pinned=False)
        ca = eng.copy_coords()
    os_ = np.lexsort((cs[2], cs[0]))
    oa = np.lexsort((ca[2], ca[0]))
    assert np.array_equal(cs[0][os_], ca[0][oa])
    perm = np.empty(model.n, np.int64)
    perm[oa] = os_
    ea = upper_pairs(ipa, ixa, 0, model.n)
    mapped = np.sort(perm[ea], axis=1)
    mapped = mapped[np.lexsort((mapped[:, 1], mapped[:, 0]))]
    es = upper_pairs(ips, ixs, 0, model.n)
    d = oracle.compare_edge_sets(mapped, es, cs[0], cs[2], model.R)
    log_parity(dict(case="config2 angular-vs-sample", m_angular=d["m_got"], m_sample=d["m_want"],
                    differing_pairs=d["only_got"] + d["only_want"], max_rel_gap=d["max_gap"]))
    assert d["only_got"] + d["only_want"] <= len(es) // 50_000
