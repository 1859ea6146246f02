"""Result copy of config 2 into pinned / pageable int64 host arrays for several
device-widened fractions (HRG_WIDEN_DEVICE_FRAC), and the two-context e2e
pipeline of bench.py for each fraction."""
import os, sys, time, json, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1501_03545_b200 as P
p = P.GeneratorParams(n=10_000_000, avg_degree=32.0, gamma=2.5, seed=2); m = p.resolve()
eng = P.get_engine(0)
eng.generate(m, p.seed)
n, nnz = eng.sizes()
ip = torch.empty(n + 1, dtype=torch.int64, pin_memory=True).numpy()
ix = torch.empty(nnz, dtype=torch.int64, pin_memory=True).numpy()
ref = None
res = {}
for f in ("1", "0.6", "0.45", "0.35", "0.25", "0"):
    os.environ["HRG_WIDEN_DEVICE_FRAC"] = f
    eng.copy_result_into(indptr=ip, indices=ix)
    t = time.perf_counter()
    for _ in range(3):
        eng.copy_result_into(indptr=ip, indices=ix)
    res[f"copy_pinned_f{f}_ms"] = (time.perf_counter() - t) / 3 * 1e3
    if ref is None: ref = ix.copy()
    else: res[f"equal_f{f}"] = bool(np.array_equal(ix, ref))
    # two contexts alternating generate + copy (bench.py's e2e)
    streams = [torch.cuda.Stream() for _ in range(2)]
    engines = [P.Engine(0, stream=s.cuda_stream) for s in streams]
    bufs = [(torch.empty(n + 1, dtype=torch.int64, pin_memory=True).numpy(),
             torch.empty(nnz, dtype=torch.int64, pin_memory=True).numpy()) for _ in range(2)]
    for w in range(2):
        engines[w].generate(m, p.seed); engines[w].copy_result_into(indptr=bufs[w][0], indices=bufs[w][1])
    started = threading.Event()
    def worker(w, k):
        if w == 1: started.wait()
        for i in range(k):
            engines[w].generate(m, p.seed)
            if w == 0 and i == 0: started.set()
            engines[w].copy_result_into(indptr=bufs[w][0], indices=bufs[w][1])
    torch.cuda.synchronize(); t = time.perf_counter()
    ths = [threading.Thread(target=worker, args=(w, 4)) for w in range(2)]
    [th.start() for th in ths]; [th.join() for th in ths]
    torch.cuda.synchronize()
    res[f"e2e_f{f}_ms_per_step"] = (time.perf_counter() - t) / 8 * 1e3
    del engines, bufs
print(json.dumps(res))
