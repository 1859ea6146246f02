"""Multi-rank path on CPU (gloo, world_size 2): the angular-sector sharding
partitions the vertices exactly, and the union of the ranks' rows is the
whole graph.  The device is stood in for by the oracle (same Philox stream,
brute-force reference edge set), so the host logic of
generate_distributed -- ranks, shards, the edge-count all-reduce -- runs
unmodified."""

import math
import os
import socket
import types

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1501_03545_b200 as P
from paper_1501_03545_b200 import distributed as D


def test_sector_partition_is_exact():
    rng = np.random.default_rng(0)
    phi = np.concatenate([rng.random(200_000) * 2 * math.pi,
                          [0.0, np.nextafter(2 * math.pi, 0), math.pi, math.pi / 2]])
    for count in (1, 2, 3, 4, 7, 8):
        sec = D.sector_of(phi, count)
        assert sec.min() >= 0 and sec.max() < count
        q = D.angular_key(phi)
        for i in range(count):
            lo, hi = D.sector_bounds(i, count)
            mine = sec == i
            assert np.all(q[mine] >= lo) and np.all(q[mine] < hi)
        # contiguous, covering key ranges
        assert D.sector_bounds(0, count)[0] == 0
        assert D.sector_bounds(count - 1, count)[1] == 2**53
        for i in range(count - 1):
            assert D.sector_bounds(i, count)[1] == D.sector_bounds(i + 1, count)[0]


class OracleEngine:
    """CPU stand-in for Engine: same coordinates (Philox + hrgen's sampling
    formula), reference edge set by brute force, rows of one sector."""

    device = 0

    def generate(self, model, seed, order, shard):
        from oracle import oracle as O
        k = P.model_constants(model.R, model.alpha)
        u1, u2 = O.philox_uniforms(model.n, seed)
        phi, _, rp = O.sample_from_uniforms(u1, u2, k["two_over_alpha"], k["sinh_half_alpha_r"],
                                           k["r_cap"], k["rp_cap"])
        pairs = O.edges_brute(phi, rp, k["cosh_r_minus_1"])
        indptr, indices = O.csr_from_pairs(model.n, pairs)
        keep = D.sector_of(phi, shard.count) == shard.index
        deg = np.diff(indptr) * keep
        self.indptr = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
        rows = [indices[indptr[v]:indptr[v + 1]] for v in np.flatnonzero(keep)]
        self.indices = np.concatenate(rows).astype(np.int64) if rows else np.empty(0, np.int64)
        self.full = (indptr, indices)
        return types.SimpleNamespace(nnz=int(self.indices.size), m=int(self.indices.size) // 2,
                                     t_sample_ms=0.0, t_build_ms=0.0, t_edges_ms=0.0,
                                     candidates=0, kernel_launches=0)

    def copy_csr(self, index_dtype=np.int64, pinned=False):
        return self.indptr, self.indices.astype(index_dtype)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        params = P.GeneratorParams(n=3000, avg_degree=12.0, gamma=2.5, seed=11)
        eng = OracleEngine()
        g, m_total, st = D.generate_distributed(params, engine=eng)
        full_indptr, full_indices = eng.full
        # rows this rank emitted are exactly the full rows of its sector
        mine = np.flatnonzero(np.diff(g.indptr))
        for v in mine:
            assert np.array_equal(g.neighbors(v), full_indices[full_indptr[v]:full_indptr[v + 1]])
        # union over ranks == the whole graph
        deg = torch.tensor(np.diff(g.indptr), dtype=torch.int64)
        dist.all_reduce(deg)
        assert np.array_equal(deg.numpy(), np.diff(full_indptr))
        assert m_total == full_indices.size // 2
        out[rank] = m_total
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_gloo_world2_shards_cover_the_graph():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert len(out) == world and len(set(out.values())) == 1 and out[0] > 0
