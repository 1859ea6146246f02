"""Median phase times of REPS generations (after 2 warm-ups) for the library
HRGEN_B200_LIB points at; one JSON line."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1501_03545_b200 as P
kw = dict(n=int(float(os.environ.get("N", "1e7"))), avg_degree=float(os.environ.get("K", "32")),
          gamma=float(os.environ.get("G", "2.5")), seed=int(os.environ.get("SEED", "2")),
          vertex_order=os.environ.get("ORDER", "sample"))
p = P.GeneratorParams(**kw)
m = p.resolve()
eng = P.get_engine(0)
order = P.generator.VERTEX_ORDERS[p.vertex_order]
keys = ("t_sample_ms", "t_sort_ms", "t_build_ms", "t_light_ms", "t_heavy_ms", "t_compact_ms",
        "t_rowsort_ms", "t_edges_ms")
res = {k: [] for k in keys}
for i in range(2 + int(os.environ.get("REPS", "7"))):
    st = eng.generate(m, p.seed, order)
    if i >= 2:
        for k in keys:
            res[k].append(getattr(st, k))
med = {k: round(sorted(v)[len(v) // 2], 4) for k, v in res.items()}
med["total_ms"] = round(med["t_sample_ms"] + med["t_build_ms"] + med["t_edges_ms"], 4)
print(json.dumps({"lib": os.path.basename(os.environ.get("HRGEN_B200_LIB", "default")),
                  "cfg": kw, "m": st.m, "tests": st.candidates, "heavy": st.heavy_queries, **med}))
