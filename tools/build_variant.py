"""Build libhrgen_b200.so variants with -D knobs into exp/lib_<name>.so (A/B runs
select one with HRGEN_B200_LIB)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1501_03545_b200 import build as B
from concurrent.futures import ThreadPoolExecutor
variants = {}
for spec in sys.argv[1:]:
    name, _, defs = spec.partition("=")
    variants[name] = [f"-D{d}" for d in defs.split(",") if d]
def one(item):
    name, defs = item
    out = os.path.join(B.ROOT, "exp", f"lib_{name}.so")
    cmd = [B.NVCC, *B.FLAGS, *defs, "-I", os.path.join(B.ROOT, "include"), "-o", out, *B.SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return name, r.returncode, (r.stderr[-500:] if r.returncode else "")
with ThreadPoolExecutor(4) as ex:
    for name, rc, err in ex.map(one, variants.items()):
        print(name, "ok" if rc == 0 else "FAILED " + err)
