
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
ixp = np.empty(nnz, np.int64); ixp[:] = 0
res = {}
for mode in ("0", "1"):
    os.environ["HRG_HOST_WIDEN"] = mode
    for buf, name in ((ix, "pinned"), (ixp, "pageable")):
        eng.copy_result_into(indptr=ip, indices=buf)
        t = time.perf_counter()
        for _ in range(3):
            eng.copy_result_into(indptr=ip, indices=buf)
        res[f"widen{mode}_{name}_ms"] = (time.perf_counter() - t) / 3 * 1e3
    ref = ix.copy() if mode == "0" else ref
    if mode == "1": res["equal"] = bool(np.array_equal(ix, ref))
print(json.dumps(res))
