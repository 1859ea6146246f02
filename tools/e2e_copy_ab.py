"""Result copy of config 2 into pinned int64 host arrays: time per copy for
several device-widened fractions, libraries alternating (HRGEN_B200_LIB is read
at import, so each measurement is its own process; see e2e_copy_ab.sh)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1501_03545_b200 as P
p = P.GeneratorParams(n=10_000_000, avg_degree=32.0, gamma=2.5, seed=2); m = p.resolve()
eng = P.get_engine(0)
eng.generate(m, p.seed)
n, nnz = eng.sizes()
ip = torch.empty(n + 1, dtype=torch.int64, pin_memory=True).numpy()
ix = torch.empty(nnz, dtype=torch.int64, pin_memory=True).numpy()
res = {"lib": os.path.basename(os.environ.get("HRGEN_B200_LIB", "") or "default")}
for f in sys.argv[1:]:
    os.environ["HRG_WIDEN_DEVICE_FRAC"] = f
    eng.copy_result_into(indptr=ip, indices=ix)
    ts = []
    for _ in range(5):
        t = time.perf_counter(); eng.copy_result_into(indptr=ip, indices=ix); ts.append(time.perf_counter() - t)
    res[f"f{f}"] = round(sorted(ts)[2] * 1e3, 2)
print(json.dumps(res))
