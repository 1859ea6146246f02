"""Warm + one generation of shard K of N (config via env) -- for launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1501_03545_b200 as P
kw = dict(n=int(float(os.environ.get("N", "1e7"))), avg_degree=float(os.environ.get("K", "32")),
          gamma=float(os.environ.get("G", "2.5")), seed=int(os.environ.get("SEED", "2")))
p = P.GeneratorParams(**kw); m = p.resolve(); eng = P.get_engine(0)
sh = P.Shard(int(os.environ.get("SK", "0")), int(os.environ.get("SN", "8")))
for _ in range(int(os.environ.get("REPS", "2"))):
    st = eng.generate(m, p.seed, 0, sh)
print({k: round(getattr(st, k), 4) for k in ("t_sample_ms", "t_build_ms", "t_light_ms", "t_heavy_ms",
                                              "t_compact_ms", "t_rowsort_ms", "t_edges_ms")},
      "launches", st.kernel_launches, "nnz", st.nnz)
