"""ctypes wrapper over oracle/libhrg_oracle.so.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg, never by the product package.
Each wrapper names the reference function (hrgen file:line) it restates.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhrg_oracle.so")

TRIG_LIBM = 0
TRIG_CR = 1

_lib = None

_d = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)


class QtTiming(ctypes.Structure):
    _fields_ = [("t_build_s", ctypes.c_double), ("t_query_s", ctypes.c_double),
                ("t_csr_s", ctypes.c_double)]


def build():
    subprocess.check_call(["sh", os.path.join(HERE, "build.sh")])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        _u32p = ctypes.POINTER(ctypes.c_uint32)
        L.orc_philox_raw.argtypes = [_u32p, _u32p, _u32p]
        L.orc_philox_uniforms.argtypes = [ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, _d, _d]
        L.orc_sample_from_uniforms.argtypes = [ctypes.c_int64, _d, _d, ctypes.c_double,
                                               ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                               _d, _d, _d]
        L.orc_circle_params.argtypes = [ctypes.c_int64, _d, ctypes.c_double, _d, _d]
        L.orc_xy.argtypes = [ctypes.c_int64, _d, _d, ctypes.c_int, _d, _d]
        L.orc_sincos_cr.argtypes = [ctypes.c_int64, _d, _d, _d]
        L.orc_edges_brute.argtypes = [ctypes.c_int64, _d, _d, ctypes.c_double, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int64, _i64p, _i64p]
        L.orc_edges_brute.restype = ctypes.c_int64
        L.orc_edges_quadtree.argtypes = [ctypes.c_int64, _d, _d, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _i64p,
                                         _i64p, ctypes.POINTER(QtTiming)]
        L.orc_edges_quadtree.restype = ctypes.c_int64
        L.orc_rows_brute.argtypes = [ctypes.c_int64, _d, _d, ctypes.c_double, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int64, _i64p, ctypes.c_int64, _i64p,
                                     _i64p]
        L.orc_rows_brute.restype = ctypes.c_int64
        L.orc_csr_from_pairs.argtypes = [ctypes.c_int64, ctypes.c_int64, _i64p, _i64p, _i64p, _i64p]
        L.orc_cosh_gap.argtypes = [ctypes.c_int64, _i64p, _i64p, _d, _d, ctypes.c_double, _d]
        _lib = L
    return _lib


def _p(a, t=_d):
    return a.ctypes.data_as(t)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def philox_raw(ctr, key):
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    lib().orc_philox_raw(c, k, o)
    return list(o)


def philox_uniforms(n, seed, offset=0):
    u1 = np.empty(n, np.float64)
    u2 = np.empty(n, np.float64)
    lib().orc_philox_uniforms(n, seed, offset, _p(u1), _p(u2))
    return u1, u2


def sample_from_uniforms(u1, u2, two_over_alpha, sinh_half, r_cap, rp_cap):
    """hrgen generator.py:160-179 on the given uniforms (libm asinh/tanh)."""
    u1, u2 = _f64(u1), _f64(u2)
    n = u1.size
    phi, rn, rp = (np.empty(n, np.float64) for _ in range(3))
    lib().orc_sample_from_uniforms(n, _p(u1), _p(u2), two_over_alpha, sinh_half, r_cap, rp_cap,
                                   _p(phi), _p(rn), _p(rp))
    return phi, rn, rp


def circle_params(rp, a):
    """hrgen geometry.py:141-157."""
    rp = _f64(rp)
    cr = np.empty_like(rp)
    rad = np.empty_like(rp)
    lib().orc_circle_params(rp.size, _p(rp), a, _p(cr), _p(rad))
    return cr, rad


def sincos_cr(x):
    x = _f64(x)
    s = np.empty_like(x)
    c = np.empty_like(x)
    lib().orc_sincos_cr(x.size, _p(x), _p(s), _p(c))
    return s, c


def edges_brute(phi, rp, a, trig=TRIG_LIBM, nthreads=0):
    """Reference edge set {(v,w): v<w, pred(v->w)} by all-pairs tests
    (hrgen generator.py:182-187 with the quadtree.py:611-613 predicate).
    Returns an (m, 2) int64 array sorted lexicographically."""
    phi, rp = _f64(phi), _f64(rp)
    n = phi.size
    m = lib().orc_edges_brute(n, _p(phi), _p(rp), a, trig, nthreads, 0, None, None)
    u = np.empty(m, np.int64)
    v = np.empty(m, np.int64)
    lib().orc_edges_brute(n, _p(phi), _p(rp), a, trig, nthreads, m, _p(u, _i64p), _p(v, _i64p))
    return np.column_stack((u, v))


def edges_quadtree(phi, rp, a, alpha, max_r, capacity=512, trig=TRIG_LIBM, nthreads=0,
                   query_lo=0, query_hi=-1, want_pairs=True):
    """Reference edge set through the restated polar quadtree
    (hrgen quadtree.py build/pack/query_many + generator.py:190-225).
    Returns (pairs (m,2) or None, m, QtTiming)."""
    phi, rp = _f64(phi), _f64(rp)
    n = phi.size
    tm = QtTiming()
    if not want_pairs:
        m = lib().orc_edges_quadtree(n, _p(phi), _p(rp), a, alpha, max_r, capacity, trig,
                                     nthreads, query_lo, query_hi, 0, None, None,
                                     ctypes.byref(tm))
        if m < 0:
            raise ValueError("point outside the tree region")
        return None, m, tm
    # single pass with a generous buffer, retry if it was too small
    cap = max(1024, 64 * n)
    while True:
        u = np.empty(cap, np.int64)
        v = np.empty(cap, np.int64)
        m = lib().orc_edges_quadtree(n, _p(phi), _p(rp), a, alpha, max_r, capacity, trig,
                                     nthreads, query_lo, query_hi, cap, _p(u, _i64p),
                                     _p(v, _i64p), ctypes.byref(tm))
        if m < 0:
            raise ValueError("point outside the tree region")
        if m <= cap:
            return np.column_stack((u[:m], v[:m])), m, tm
        cap = m


def rows_brute(phi, rp, a, qids, trig=TRIG_LIBM, nthreads=0):
    """Full rows (ascending neighbour ids) of the vertices qids, by all-pairs
    tests against every point (hrgen generator.py:182-187 edge rule with the
    quadtree.py:611-613 predicate, circle of the smaller id).  For sampled-row
    parity at sizes where the whole edge set is out of the oracle's reach.
    Returns (indptr (len(qids)+1,), indices) int64."""
    phi, rp = _f64(phi), _f64(rp)
    q = np.ascontiguousarray(qids, dtype=np.int64)
    n = phi.size
    total = lib().orc_rows_brute(n, _p(phi), _p(rp), a, trig, nthreads, q.size, _p(q, _i64p),
                                 0, None, None)
    indptr = np.empty(q.size + 1, np.int64)
    indices = np.empty(total, np.int64)
    lib().orc_rows_brute(n, _p(phi), _p(rp), a, trig, nthreads, q.size, _p(q, _i64p), total,
                         _p(indptr, _i64p), _p(indices, _i64p))
    return indptr, indices


def csr_from_pairs(n, pairs):
    """hrgen graph.py:52-77 (rows sorted) for u<v pairs."""
    pairs = np.ascontiguousarray(pairs, dtype=np.int64).reshape(-1, 2)
    u = np.ascontiguousarray(pairs[:, 0])
    v = np.ascontiguousarray(pairs[:, 1])
    m = u.size
    indptr = np.empty(n + 1, np.int64)
    indices = np.empty(2 * m, np.int64)
    lib().orc_csr_from_pairs(n, m, _p(u, _i64p), _p(v, _i64p), _p(indptr, _i64p),
                             _p(indices, _i64p))
    return indptr, indices


def cosh_gap(pairs, phi, rp, R):
    """|cosh d - cosh R| / cosh R of each (u, v) pair, in __float128."""
    pairs = np.ascontiguousarray(pairs, dtype=np.int64).reshape(-1, 2)
    u = np.ascontiguousarray(pairs[:, 0])
    v = np.ascontiguousarray(pairs[:, 1])
    phi, rp = _f64(phi), _f64(rp)
    gap = np.empty(u.size, np.float64)
    if u.size:
        lib().orc_cosh_gap(u.size, _p(u, _i64p), _p(v, _i64p), _p(phi), _p(rp), float(R), _p(gap))
    return gap


def compare_edge_sets(got, want, phi, rp, R, band=1e-12):
    """Exact comparison of two lexicographically sorted (m, 2) u<v edge
    arrays.  Returns a dict: m of each, the pairs only in one of them, and
    their largest cosh-distance gap (the north star allows differences only
    where |cosh d - cosh R| <= band * cosh R)."""
    got = np.ascontiguousarray(got, dtype=np.int64).reshape(-1, 2)
    want = np.ascontiguousarray(want, dtype=np.int64).reshape(-1, 2)
    n = int(max(got.max(initial=-1), want.max(initial=-1))) + 1
    if got.shape == want.shape and np.array_equal(got, want):
        return dict(m_got=len(got), m_want=len(want), only_got=0, only_want=0, max_gap=0.0,
                    outside_band=0, pairs=np.empty((0, 2), np.int64), gaps=np.empty(0))
    kg = got[:, 0] * n + got[:, 1]   # both ascending (lexicographic order)
    kw = want[:, 0] * n + want[:, 1]

    def missing(a, b):  # elements of sorted a absent from sorted b
        if b.size == 0:
            return a
        i = np.minimum(np.searchsorted(b, a), b.size - 1)
        return a[b[i] != a]

    only_g = missing(kg, kw)
    only_w = missing(kw, kg)
    diff = np.concatenate([only_g, only_w])
    pairs = np.column_stack((diff // n, diff % n))
    gap = cosh_gap(pairs, phi, rp, R)
    return dict(m_got=len(got), m_want=len(want), only_got=int(only_g.size),
                only_want=int(only_w.size), max_gap=float(gap.max(initial=0.0)),
                outside_band=int(np.count_nonzero(gap > band)), pairs=pairs, gaps=gap)


RIM_ULPS = 2.0 ** -46   # 1 - r_p below this: a point within ~64 ulps of the disk's rim


def classify_mismatches(d, phi, rp, a, band=1e-12):
    """Sort the pairs of a compare_edge_sets result into
      band      -- |cosh d - cosh R| <= band cosh R (the north star's exception);
      ref_drop  -- present only in the GPU set, accepted by the reference's own
                   leaf predicate (quadtree.py:611-613, circle of the smaller id;
                   checked here by all-pairs rows), with an endpoint at the rim
                   (1 - r_p < 2^-46): pairs hrgen's quadtree prunes although its
                   predicate accepts them -- its leaf window (quadtree.py:573-590)
                   and the predicate round differently where fp64 Poincare
                   coordinates cannot resolve the hyperbolic distance;
      unexplained -- everything else (a real disagreement).
    Returns the counts."""
    pairs = d["pairs"]
    out = {"band": 0, "ref_drop": 0, "unexplained": 0}
    if pairs.size == 0:
        return out
    n_got = d["only_got"]
    got_only = pairs[:n_got]
    gaps = d["gaps"]
    inband = gaps <= band
    out["band"] = int(inband.sum())
    # GPU-only pairs outside the band: the reference predicate on all pairs
    cand = got_only[~inband[:n_got]]
    if cand.size:
        q = np.unique(cand[:, 0])
        ip, ix = rows_brute(phi, rp, a, q)
        row = {int(v): ix[ip[k]:ip[k + 1]] for k, v in enumerate(q)}
        for u, v in cand.tolist():
            rim = max(rp[u], rp[v]) >= 1.0 - RIM_ULPS
            if rim and np.isin(v, row[u]).item():
                out["ref_drop"] += 1
            else:
                out["unexplained"] += 1
    out["unexplained"] += int((~inband[n_got:]).sum())
    return out


def edge_hash(pairs):
    """sha256 of the lexicographically sorted (m,2) little-endian int64 edge
    array -- the form hrgen Graph.edge_array() (graph.py:38-42) returns."""
    import hashlib
    arr = np.ascontiguousarray(pairs, dtype="<i8").reshape(-1, 2)
    return hashlib.sha256(arr.tobytes()).hexdigest()
