"""Loader for the reference-generated fixtures in tests/golden/ (see
tests/golden/make_golden.py for how they were produced)."""

from __future__ import annotations

import functools
import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TWO_PI = 2.0 * np.pi


@functools.lru_cache(maxsize=None)
def _runs():
    with open(os.path.join(GOLDEN, "runs.json")) as fh:
        meta = json.load(fh)
    rp = np.load(os.path.join(GOLDEN, "runs.npz"))["r_poincare"]
    return meta, rp


class Run:
    """One reference generator run: coordinates + the reference's edge set
    fingerprint (sha256 of hrgen Graph.edge_array())."""

    def __init__(self, meta, rp_all):
        self.tag = meta["tag"]
        self.n = meta["n"]
        self.seed = meta["seed"]
        self.alpha = float.fromhex(meta["alpha"])
        self.R = float.fromhex(meta["R"])
        self.a = float.fromhex(meta["a"])
        self.max_r = float.fromhex(meta["max_r"])
        self.rp_cap = float.fromhex(meta["rp_cap"])
        self.m = meta["m"]
        self.edge_sha256 = meta["edge_sha256"]
        self.avg_degree = meta.get("avg_degree")
        self.gamma = meta.get("gamma")
        off = meta["offset"]
        self.r_poincare = np.ascontiguousarray(rp_all[off:off + self.n])
        # hrgen generator.py:168-170: phi = TWO_PI * draws[:, 0]
        draws = np.random.default_rng(self.seed).random((self.n, 2))
        self.phi = TWO_PI * draws[:, 0]
        got = hashlib.sha256(np.ascontiguousarray(self.phi, "<f8").tobytes()).hexdigest()
        assert got == meta["phi_sha256"], "phi regeneration does not match the reference"

    def __repr__(self):
        return f"Run({self.tag}, n={self.n}, seed={self.seed}, R={self.R:.4f}, m={self.m})"


def runs(tags=None):
    meta, rp = _runs()
    out = [Run(m, rp) for m in meta]
    if tags is not None:
        out = [r for r in out if r.tag in tags]
    return out


def target_radius_table():
    with open(os.path.join(GOLDEN, "target_radius.json")) as fh:
        return json.load(fh)


def long_range_table():
    with open(os.path.join(GOLDEN, "long_range.json")) as fh:
        return json.load(fh)


def config0_edges():
    return np.load(os.path.join(GOLDEN, "config0_edges.npz"))["edges"].astype(np.int64)
