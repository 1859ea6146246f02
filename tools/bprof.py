"""Per-band block-query counters (library built with -DHRG_BLOCK_PROFILE)."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1501_03545_b200 as P
from paper_1501_03545_b200 import _lib
kw = dict(n=int(float(os.environ.get("N", "1e7"))), avg_degree=float(os.environ.get("K", "32")),
          gamma=float(os.environ.get("G", "2.5")), seed=int(os.environ.get("SEED", "2")))
p = P.GeneratorParams(**kw); m = p.resolve(); eng = P.get_engine(0)
L = _lib.load()
buf = (ctypes.c_ulonglong * (2 * 32 * 8))()
eng.generate(m, p.seed)
L.hrg_debug_block_profile(eng._ctx, buf)
st = eng.generate(m, p.seed)
L.hrg_debug_block_profile(eng._ctx, buf)
a = np.array(buf, dtype=np.float64).reshape(2, 32, 8)
print(json.dumps({"light_ms": st.t_light_ms, "write_ms": st.t_compact_ms, "tests": st.candidates}))
for ps, name in ((0, "count"), (1, "write")):
    tot = a[ps, :, 0].sum()
    print(name, "band  clk%   tiles  subtiles chunks  iters  rounds  q/chunk")
    for b in range(32):
        r = a[ps, b]
        if r[1] == 0: continue
        print(f"{name} {b:3d} {100*r[0]/tot:6.2f} {r[1]:8.0f} {r[2]:9.0f} {r[3]:9.0f} {r[4]:10.0f} {r[6]:8.0f} {r[4]/max(r[3],1):6.2f}")
