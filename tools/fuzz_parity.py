"""Random models against the CPU oracle (libm trig), both vertex orders, plus
sharded unions: a wider net than the fixed parity cases for the light pass's
dense block / one-orientation margin / tile order.  usage: fuzz_parity.py CASES SEED"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1501_03545_b200 as P
from oracle import oracle as O
O.build()
cases, seed = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(seed)
bad = 0
for c in range(cases):
    n = int(10 ** rng.uniform(2.5, 5.4))
    k = float(min(n / 4, 10 ** rng.uniform(0.3, 2.5)))
    gamma = float(rng.uniform(2.05, 6.0))
    order = "angular" if rng.random() < 0.4 else "sample"
    if os.environ.get("FUZZ_RADIUS"):  # sparse large-radius models: points within ulps of the rim
        p = P.GeneratorParams(n=n, radius=float(rng.uniform(24.0, 37.0)), alpha=float(rng.uniform(0.55, 1.2)),
                              seed=int(rng.integers(1 << 30)), vertex_order=order)
    else:
        p = P.GeneratorParams(n=n, avg_degree=k, gamma=gamma, seed=int(rng.integers(1 << 30)),
                              vertex_order=order)
    try:
        model = p.resolve()
    except Exception as e:
        continue
    g, co = P.generate_with_coordinates(p)
    a = P.model_constants(model.R, model.alpha)["cosh_r_minus_1"]
    e, m, _ = O.edges_quadtree(co.phi, co.r_poincare, a, model.alpha, P.to_poincare_radius(model.R),
                               512, O.TRIG_LIBM)
    ok = g.m == m and np.array_equal(g.edge_array(), e)
    cls = None
    if not ok:
        # the only accepted difference: pairs hrgen's quadtree prunes at the rim
        # although its predicate accepts them (oracle.classify_mismatches)
        d = O.compare_edge_sets(g.edge_array(), e, co.phi, co.r_poincare, model.R)
        cls = O.classify_mismatches(d, co.phi, co.r_poincare, a)
        ok = cls["unexplained"] == 0 and cls["band"] == 0 and d["only_want"] == 0
    shard_ok = True
    if ok and order == "sample" and rng.random() < 0.5:
        cnt = int(rng.integers(2, 9))
        rows = 0
        ind = [None] * n
        for s in range(cnt):
            gs, _ = P.generate_with_stats(p, shard=P.Shard(s, cnt))
            deg = np.diff(gs.indptr)
            rows += int((deg > 0).sum())
            shard_ok &= bool(np.all((deg == 0) | (deg == np.diff(g.indptr))))
            nz = np.nonzero(deg)[0]
            for v in nz[:50]:
                shard_ok &= bool(np.array_equal(gs.indices[gs.indptr[v]:gs.indptr[v + 1]],
                                                g.indices[g.indptr[v]:g.indptr[v + 1]]))
    if not (ok and shard_ok):
        bad += 1
    print(json.dumps(dict(n=n, k=round(k, 2), gamma=round(gamma, 3), order=order, R=round(model.R, 3),
                          m=int(g.m), m_ref=int(m), ok=bool(ok), shard_ok=bool(shard_ok),
                          **({"classified": cls} if cls else {}))), flush=True)
print("cases", cases, "bad", bad)
sys.exit(1 if bad else 0)
