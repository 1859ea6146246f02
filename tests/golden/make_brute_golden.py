"""Fixtures for the all-pairs reference (hrgen generate_brute_force,
generator.py:249-274), made by running hrgen itself on the coordinates of the
golden runs (tests/golden/runs.*).  Build container only (the reference is
not present on GPU boxes):

    python tests/golden/make_brute_golden.py

writes brute.json: per run (by index into runs.json), the edge count and the
sha256 of hrgen.generate_brute_force(coords, R).edge_array(), and whether it
equals hrgen.generate's edge set on the same run.
"""

import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import hrgen  # noqa: E402
import golden_data as gd  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    out = []
    for k, run in enumerate(gd.runs()):
        if run.n > 12_000:
            continue
        coords = hrgen.VertexCoordinates(phi=run.phi, r_native=2.0 * np.arctanh(run.r_poincare),
                                         r_poincare=run.r_poincare)
        g = hrgen.generate_brute_force(coords, run.R)
        e = np.ascontiguousarray(g.edge_array(), dtype="<i8")
        sha = hashlib.sha256(e.tobytes()).hexdigest()
        out.append({"run": k, "tag": run.tag, "n": run.n, "m": int(g.m), "edge_sha256": sha,
                    "equals_generate": sha == run.edge_sha256})
    with open(os.path.join(HERE, "brute.json"), "w") as fh:
        json.dump(out, fh, indent=0)
    print(len(out), "runs;", sum(not r["equals_generate"] for r in out), "differ from generate")


if __name__ == "__main__":
    main()
