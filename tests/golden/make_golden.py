"""Generate golden fixtures by running the reference implementation.

Run in the build container only (the reference is not present on GPU boxes):

    python tests/golden/make_golden.py

It imports hrgen from /root/reference/pkg/src (read-only, never copied) and
writes, next to this script:

  target_radius.json  -- hrgen.target_radius over a grid of (n, k, gamma)
  runs.npz            -- r_poincare of every run below, concatenated (offsets
                         per run).  phi is not stored: it is TWO_PI times the
                         first column of numpy default_rng(seed).random((n,2))
                         (generator.py:168-170), integer-exact on any host, and
                         runs.json keeps its sha256 to prove the regeneration
  runs.json           -- per run: n, alpha, R, seed, a = cosh(R)-1 and the
                         Poincare clamp as hrgen computes them, edge count m
                         and sha256 of hrgen's sorted edge array
  config0_edges.npz   -- full edge array of config 0 (n=1e4, k=6, gamma=3,
                         seed 0) for mismatch diagnostics
  long_range.json     -- hrgen.add_long_range_edges result hashes

The runs cover: the acceptance grid of hrgen tests/test_acceptance.py:59-90
(n in {100,500,2000} x k in {4,16,64} x gamma in {2.2,3,7} x seeds 0..4, with
its explicit-radius fallback), the parametrized cases of
tests/test_generator.py:128-144, the explicit-radius case :147-151, the
single-vertex case, BASELINE config 0, and large-radius stress cases where
the Poincare coordinates of the rim are only a few ulps below 1.
"""

import hashlib
import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

import hrgen  # noqa: E402
from hrgen import GeneratorParams, generate, sample_points  # noqa: E402
from hrgen.geometry import to_poincare_radius  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def edge_hash(graph):
    arr = np.ascontiguousarray(graph.edge_array(), dtype="<i8")
    return hashlib.sha256(arr.tobytes()).hexdigest()


def model_constants(R):
    # exactly the expressions hrgen evaluates (geometry.py:150, generator.py:176-178)
    a = float(2.0 * np.sinh(np.asarray(R, dtype=np.float64) / 2.0) ** 2)
    max_r = float(to_poincare_radius(R))
    rp_cap = float(np.nextafter(to_poincare_radius(R), 0.0))
    return a, max_r, rp_cap


def run_cases():
    cases = []
    for n in (100, 500, 2000):
        for kbar in (4.0, 16.0, 64.0):
            for gamma in (2.2, 3.0, 7.0):
                for seed in range(5):
                    try:
                        p = GeneratorParams(n=n, avg_degree=kbar, gamma=gamma, seed=seed)
                        p.resolve()
                    except ValueError:
                        p = GeneratorParams(n=n, radius=1.0, gamma=gamma, seed=seed)
                    cases.append(("accept", p))
    for n, kbar, gamma, seed in ((300, 6.0, 2.4, 0), (700, 10.0, 3.0, 1), (1200, 4.0, 5.0, 2)):
        cases.append(("testgen", GeneratorParams(n=n, avg_degree=kbar, gamma=gamma, seed=seed)))
    cases.append(("radius", GeneratorParams(n=500, radius=9.0, alpha=1.0, seed=0)))
    cases.append(("single", GeneratorParams(n=1, radius=5.0, alpha=1.0, seed=0)))
    cases.append(("config0", GeneratorParams(n=10_000, avg_degree=6.0, gamma=3.0, seed=0)))
    cases.append(("mid", GeneratorParams(n=50_000, avg_degree=10.0, gamma=3.0, seed=1)))
    cases.append(("mid25", GeneratorParams(n=30_000, avg_degree=32.0, gamma=2.5, seed=2)))
    # stress: rim radii within a few ulps of 1 in the Poincare disk
    cases.append(("bigR", GeneratorParams(n=4000, radius=33.0, alpha=1.0, seed=5)))
    cases.append(("bigR2", GeneratorParams(n=4000, radius=35.5, alpha=0.6, seed=6)))
    cases.append(("bigR3", GeneratorParams(n=20_000, radius=30.0, alpha=0.75, seed=7)))
    cases.append(("cfg2R", GeneratorParams(n=100_000, radius=28.789361743909193, alpha=0.75,
                                           seed=9)))
    cases.append(("cfg3R", GeneratorParams(n=100_000, radius=33.165607448498854, alpha=1.0,
                                           seed=10)))
    cases.append(("cfg4R", GeneratorParams(n=100_000, radius=35.50799080982715, alpha=0.6,
                                           seed=11)))
    cases.append(("dense", GeneratorParams(n=3000, avg_degree=256.0, gamma=5.0, seed=8)))
    # base graphs of the long-range augmentation fixtures below
    cases.append(("lr1", GeneratorParams(n=3000, avg_degree=6.0, gamma=3.0, seed=2)))
    cases.append(("lr2", GeneratorParams(n=2000, avg_degree=16.0, gamma=2.5, seed=3)))
    return cases


def main():
    # 1. target radius grid (geometry.py:197-232)
    tr = []
    for n in (100, 1000, 10_000, 100_000, 1_000_000, 10_000_000, 100_000_000):
        for k in (4.0, 6.0, 10.0, 16.0, 32.0, 64.0, 256.0):
            for gamma in (2.2, 2.5, 3.0, 5.0, 7.0):
                alpha = (gamma - 1.0) / 2.0
                try:
                    R = hrgen.target_radius(n, k, alpha)
                    tr.append({"n": n, "k": k, "gamma": gamma, "R": R.hex()})
                except ValueError as e:
                    tr.append({"n": n, "k": k, "gamma": gamma, "error": type(e).__name__})
    with open(os.path.join(HERE, "target_radius.json"), "w") as fh:
        json.dump(tr, fh, indent=0)

    # 2. generator runs
    meta = []
    rps = []
    offset = 0
    for tag, p in run_cases():
        model = p.resolve()
        t0 = time.perf_counter()
        g = generate(p)
        dt = time.perf_counter() - t0
        coords = sample_points(model.n, model.alpha, model.R, p.seed)
        a, max_r, rp_cap = model_constants(model.R)
        meta.append({
            "tag": tag, "n": model.n, "alpha": model.alpha.hex() if isinstance(model.alpha, float)
            else float(model.alpha).hex(), "R": float(model.R).hex(), "seed": p.seed,
            "avg_degree": p.avg_degree, "gamma": p.gamma,
            "a": a.hex(), "max_r": max_r.hex(), "rp_cap": rp_cap.hex(),
            "m": int(g.m), "edge_sha256": edge_hash(g), "offset": offset,
            "phi_sha256": hashlib.sha256(np.ascontiguousarray(coords.phi, "<f8").tobytes())
            .hexdigest(),
            "ref_seconds": dt,
        })
        rps.append(coords.r_poincare)
        offset += model.n
        if tag == "config0":
            np.savez_compressed(os.path.join(HERE, "config0_edges.npz"),
                                edges=g.edge_array().astype(np.int32))
        print(f"{tag:8s} n={model.n:6d} R={model.R:.4f} m={g.m} ({dt:.2f}s)", flush=True)
    np.savez_compressed(os.path.join(HERE, "runs.npz"), r_poincare=np.concatenate(rps))
    with open(os.path.join(HERE, "runs.json"), "w") as fh:
        json.dump(meta, fh, indent=0)

    # 3. long-range augmentation (generator.py:277-316)
    lr = []
    for n, kbar, gamma, seed, frac in ((3000, 6.0, 3.0, 2, 0.01), (2000, 16.0, 2.5, 3, 0.05)):
        g = generate(GeneratorParams(n=n, avg_degree=kbar, gamma=gamma, seed=seed))
        aug = hrgen.add_long_range_edges(g, frac, seed=seed)
        lr.append({"n": n, "avg_degree": kbar, "gamma": gamma, "seed": seed, "fraction": frac,
                   "m_base": int(g.m), "base_sha256": edge_hash(g),
                   "m": int(aug.m), "edge_sha256": edge_hash(aug)})
    with open(os.path.join(HERE, "long_range.json"), "w") as fh:
        json.dump(lr, fh, indent=0)


if __name__ == "__main__":
    main()
