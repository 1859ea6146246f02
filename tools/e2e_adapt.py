"""The result copy's adaptive device-widened share: config 2, repeated copies
into pinned int64 arrays (HRG_WIDEN_TRACE=1 prints each copy's observation),
then bench.py's two-context pipeline."""
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
ts = []
for _ in range(int(os.environ.get("COPIES", "14"))):
    t = time.perf_counter(); eng.copy_result_into(indptr=ip, indices=ix); ts.append(round((time.perf_counter() - t) * 1e3, 1))
print("copy ms:", ts)
ref = ix.copy()
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
for rnd in range(3):
    started.clear()
    torch.cuda.synchronize(); t = time.perf_counter()
    ths = [threading.Thread(target=worker, args=(w, 4)) for w in range(2)]
    [th.start() for th in ths]; [th.join() for th in ths]
    torch.cuda.synchronize()
    print("two-context e2e ms/step:", round((time.perf_counter() - t) / 8 * 1e3, 2),
          "equal:", bool(np.array_equal(bufs[0][1], ref) and np.array_equal(bufs[1][1], ref)))
