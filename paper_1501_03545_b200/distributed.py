"""Multi-GPU generation: one process per GPU, angular-sector sharding.

Every rank samples the same point set (the stream is counter-based, so this
costs no communication), builds the same band index, and emits the CSR rows
of the query vertices whose angle lies in its sector
[2*pi*rank/world, 2*pi*(rank+1)/world).  The rows of all ranks together are
exactly the single-GPU graph; the only collective is one scalar all-reduce
of the row-entry counts (for the edge total).  The sector rule below is the
host mirror of the device's (hrg_api.cu build_index / k_band_setup), so
tests can check the partition without a GPU.
"""

from __future__ import annotations

import numpy as np

from .engine import Shard, get_engine
from .errors import ParameterDomainError
from .generator import VERTEX_ORDERS, GeneratorParams, _check_model_domain, _stats
from .graph import Graph

Q_BITS = 53
TWO_PI = 6.283185307179586  # == 2.0 * math.pi
Q_SCALE = float(2**Q_BITS) / TWO_PI


def angular_key(phi):
    """floor(phi * 2^53/(2 pi)) clamped to [0, 2^53) -- the device's qkey()."""
    q = np.floor(np.asarray(phi, dtype=np.float64) * Q_SCALE)
    q = np.clip(q, 0, 2**Q_BITS - 1)
    return q.astype(np.uint64)


SORT_SHIFT = Q_BITS - 27  # the device orders points to 2^-27 of a turn


def sector_bounds(index: int, count: int):
    """Half-open key range [lo, hi) of sector `index` of `count`: an even
    split of the 2^27 sort-granularity angles (hrg_api.cu build_index)."""
    span = 2**(Q_BITS - SORT_SHIFT)
    lo = (index * span + count - 1) // count
    hi = span if index + 1 == count else ((index + 1) * span + count - 1) // count
    return lo << SORT_SHIFT, hi << SORT_SHIFT


def sector_of(phi, count: int):
    """Sector index of every angle (vectorized)."""
    q = angular_key(np.atleast_1d(phi))
    starts = np.array([sector_bounds(i, count)[0] for i in range(count)], dtype=np.uint64)
    return np.searchsorted(starts, q, side="right") - 1


def shard_for_rank(rank: int, world: int) -> Shard:
    if not 0 <= rank < world:
        raise ValueError("rank must be in [0, world)")
    return Shard(rank, world)


def generate_distributed(params: GeneratorParams, *, group=None, device=None, engine=None):
    """Generate on every rank of `group` (torch.distributed).  Returns
    (local_graph, m_total, stats): local_graph holds all n rows, non-empty only
    for this rank's sector; m_total is the edge count of the whole graph."""
    import torch
    import torch.distributed as dist

    if params.long_range_fraction > 0.0:
        # hrgen adds long-range edges to the finished graph (generator.py:
        # 228-229): a rank holds only its sector's rows, so it cannot draw them
        raise ParameterDomainError(
            "long_range_fraction > 0 needs the whole graph; generate it on one rank or add "
            "the edges after gathering the rows (add_long_range_edges)")
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    model = params.resolve()
    _check_model_domain(model)
    eng = engine if engine is not None else get_engine(device)
    st = eng.generate(model, params.seed, VERTEX_ORDERS[params.vertex_order],
                      shard_for_rank(rank, world))
    indptr, indices = eng.copy_csr(np.int64, pinned=False)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", eng.device) if backend == "nccl" else torch.device("cpu")
    tot = torch.tensor([int(st.nnz)], dtype=torch.int64, device=dev)
    dist.all_reduce(tot, op=dist.ReduceOp.SUM, group=group)
    m_total = int(tot.item()) // 2
    return Graph(indptr=indptr, indices=indices), m_total, _stats(model, st)


__all__ = ["angular_key", "generate_distributed", "sector_bounds", "sector_of",
           "shard_for_rank", "Q_SCALE", "TWO_PI"]
