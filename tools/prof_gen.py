"""One warm + one profiled generation (config 2 by default) for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1501_03545_b200 as P
kw = dict(n=int(float(os.environ.get("N", "1e7"))), avg_degree=float(os.environ.get("K", "32")),
          gamma=float(os.environ.get("G", "2.5")), seed=int(os.environ.get("SEED", "2")),
          vertex_order=os.environ.get("ORDER", "sample"))
p = P.GeneratorParams(**kw)
m = p.resolve()
eng = P.get_engine(0)
order = P.generator.VERTEX_ORDERS[p.vertex_order]
for _ in range(int(os.environ.get("REPS", "2"))):
    st = eng.generate(m, p.seed, order)
print("m", st.m, "tests", st.candidates, "light", st.t_light_ms, "heavy", st.t_heavy_ms,
      "write", st.t_compact_ms, "rowsort", st.t_rowsort_ms)
