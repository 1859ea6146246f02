"""Golden fixture for hrgen's quadtree pruning drop (run in the build container
only; imports hrgen from /root/reference/pkg/src, read-only, never copied):

    python tests/golden/make_prune_golden.py

At n = 1e5, R = 37, alpha = 0.6, seed 3 (hrgen's own sample_points), hrgen's
generate() returns 811 edges while its own leaf predicate (quadtree.py:611-613,
circle of the smaller id, generator.py:182-187) accepts 812 pairs: its
quadtree pruning drops one pair whose second vertex sits 1 ulp below the rim
(r_p = 1 - 2^-52).  The leaf window that drops it (quadtree.py:573-590) is an
arccos of a ratio that cancels catastrophically at the rim, evaluated with
numpy's arccos -- on AVX-512 hosts numpy dispatches float64 arccos to its
SIMD (SVML) kernels, which differ from libm's acos -- so which rim pairs the
reference drops depends on its host.  The GPU evaluates the predicate on every
pair of its conservative windows, i.e. it returns the 812.

Writes prune_drop.npz: phi, r_poincare, hrgen's edge array, and the all-pairs
predicate's edge array (as the oracle computes it, libm trig).
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from hrgen.generator import GeneratorParams, generate, sample_points  # noqa: E402

from oracle import oracle as O  # noqa: E402

N, R, ALPHA, SEED = 100_000, 37.0, 0.6, 3


def main():
    p = GeneratorParams(n=N, radius=R, alpha=ALPHA, seed=SEED)
    model = p.resolve()
    co = sample_points(N, model.alpha, model.R, SEED)
    ref = generate(p).edge_array()
    a = float(2.0 * np.sinh(np.asarray(model.R) / 2.0) ** 2)
    allpairs = O.edges_brute(co.phi, co.r_poincare, a, O.TRIG_LIBM)
    np.savez_compressed(os.path.join(HERE, "prune_drop.npz"), phi=co.phi,
                        r_poincare=co.r_poincare, hrgen_edges=ref, allpairs_edges=allpairs,
                        n=N, R=model.R, alpha=model.alpha, seed=SEED)
    print(f"hrgen m={len(ref)} all-pairs m={len(allpairs)}")


if __name__ == "__main__":
    main()
