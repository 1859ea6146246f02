"""Full-size parity for BASELINE configs 2, 3 and the config-4 sweep.

The whole edge set at n = 1e7..1e8 is out of the CPU oracle's reach, so each
case checks (1) hrgen's Graph invariants over the WHOLE device CSR (row
pointers, ids in range, no loops, strictly increasing rows, symmetry via a
checksum of checksums) and (2) a sample of rows -- random vertices, the
highest-degree hubs, the lowest- and highest-id vertices -- bit-exact against
the oracle's all-pairs rows (oracle.rows_brute: every point tested, circle of
the smaller id, correctly rounded trig like the device).  Run on a B200:
pytest -m gpu."""

import numpy as np
import pytest

import paper_1501_03545_b200 as P
from paper_1501_03545_b200 import GeneratorParams

pytestmark = pytest.mark.gpu

SWEEP = [dict(n=10_000_000, avg_degree=k, gamma=g, seed=4)
         for k in (4.0, 64.0, 256.0) for g in (2.2, 3.0, 5.0)]
CASES = ([dict(n=10_000_000, avg_degree=32.0, gamma=2.5, seed=2),
          dict(n=10_000_000, avg_degree=32.0, gamma=2.5, seed=2, vertex_order="angular")]
         + SWEEP + [dict(n=100_000_000, avg_degree=16.0, gamma=3.0, seed=3)])
CHUNK = 1 << 27


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


@pytest.mark.parametrize("kw", CASES, ids=lambda k: f"n{k['n']:.0e}-k{k['avg_degree']:g}"
                         f"-g{k['gamma']:g}-s{k['seed']}" + ("-angular" if "vertex_order" in k else ""))
def test_full_size_rows_match_oracle(oracle, kw):
    import torch
    p = GeneratorParams(**kw)
    model = p.resolve()
    eng = P.get_engine()
    st = eng.generate(model, p.seed, P.generator.VERTEX_ORDERS[p.vertex_order])
    ip, ix = eng.device_csr()
    n = model.n
    deg = device_invariants(ip, ix, n)
    m = int(ip[-1]) // 2
    assert m == st.m
    # realised average degree near the target (hrgen's solver targets the
    # expectation; at gamma=2.2 the hub tail makes it noisier)
    assert 2 * m / n == pytest.approx(kw["avg_degree"], rel=0.2 if kw["gamma"] < 2.5 else 0.12)

    rng = np.random.default_rng(kw["seed"] + 11)
    hubs = torch.topk(deg, 6).indices.cpu().numpy()
    q = np.unique(np.concatenate([rng.choice(n, 40, replace=False), hubs, [0, n - 1]]))
    phi, _, rp = eng.copy_coords()
    a = P.model_constants(model.R, model.alpha)["cosh_r_minus_1"]
    oi, ox = oracle.rows_brute(phi, rp, a, q, oracle.TRIG_CR)
    ipq = ip.cpu().numpy() if n <= 10_000_000 else None
    for k, v in enumerate(q.tolist()):
        if ipq is not None:
            s, e = int(ipq[v]), int(ipq[v + 1])
        else:
            s, e = int(ip[v]), int(ip[v + 1])
        got = ix[s:e].cpu().numpy().astype(np.int64)
        want = ox[oi[k]:oi[k + 1]]
        assert np.array_equal(got, want), (v, got.size, want.size)
    print(f"[full] {kw}: R={model.R:.4f} m={m} candidates={st.candidates} "
          f"max_deg={int(deg.max())} rows_checked={q.size} "
          f"entries_checked={int(oi[-1])} t_edges={st.t_edges_ms:.2f}ms")
