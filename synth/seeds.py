"""Seed vertices for sampling instances (inputs only).

Seeds are drawn uniformly with replacement from the non-isolated vertices
(reading R29 / SURVEY.md G29), using the input hash (not the
sampler's Philox stream), so walks never start on a vertex without neighbours.
"""
from __future__ import annotations

import torch

from .rmat import RmatGraph, hash_stream, stream_key


def nonisolated_vertices(g: RmatGraph) -> torch.Tensor:
    """Ascending int64 ids of vertices with degree > 0."""
    return torch.nonzero(g.degrees() > 0).flatten()


def _pick(pool: torch.Tensor, idx: torch.Tensor, key: int) -> torch.Tensor:
    h = hash_stream(idx, key)                      # uniform in [0, 2**32)
    n = pool.numel()
    if n == 0:
        raise ValueError("graph has no non-isolated vertex")
    return pool[(h * n) >> 32]                     # h*n < 2**59: no int64 overflow


def instance_seeds(g: RmatGraph, n_instances: int, graph_seed: int | None = None,
                   set_id: int = 0) -> torch.Tensor:
    """One seed per instance, int32 [n] (uint32 semantics). `set_id` selects one of
    the three seed sets the paper averages over (§6)."""
    gs = g.graph_seed if graph_seed is None else graph_seed
    pool = nonisolated_vertices(g)
    idx = torch.arange(n_instances, dtype=torch.int64, device=pool.device)
    return _pick(pool, idx, stream_key(gs, 3, set_id)).to(torch.int32)


def mdrw_seeds(g: RmatGraph, n_instances: int, pool_size: int, graph_seed: int | None = None,
               set_id: int = 0) -> torch.Tensor:
    """MDRW: pool_size seeds per instance, int32 [n, m] (PAPER.md line 466:
    "an instance has multiple source vertices")."""
    gs = g.graph_seed if graph_seed is None else graph_seed
    pool = nonisolated_vertices(g)
    idx = torch.arange(n_instances * pool_size, dtype=torch.int64, device=pool.device)
    return _pick(pool, idx, stream_key(gs, 4, set_id)).to(torch.int32).view(n_instances, pool_size)
