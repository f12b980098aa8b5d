"""Multi-GPU plumbing: instance sharding and the end-of-run output gather.

C-SAW's multi-GPU scheme (§5.4): "divides all the
sampling instances into several disjoint groups, each of which contains equal
number of instances ... no inter-GPU communication is required".  Each rank
runs the C ABI on its contiguous instance range, passing the range start as
`instance_base` so that draws (keyed by global instance id) and therefore
outputs are identical for any GPU count.  The only collective is the gather of
sampled subgraphs after sampling (NCCL over NVLink on GPUs; gloo on CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, equal (±1) instance range of `rank`: [floor(r N / W), floor((r+1) N / W))."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return (rank * n_total) // world, ((rank + 1) * n_total) // world


def _all_gather_var(t: torch.Tensor, group=None) -> list[torch.Tensor]:
    """all_gather of a 1-D/2-D tensor whose first dimension differs across ranks."""
    world = dist.get_world_size(group)
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    ns = [int(x.item()) for x in ns]
    m = max(ns) if ns else 0
    pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return [b[:k] for b, k in zip(bufs, ns)]


def gather_walks(path: torch.Tensor, group=None) -> torch.Tensor:
    """Concatenate every rank's walk rows in rank (= instance) order; returned on all ranks."""
    return torch.cat(_all_gather_var(path.contiguous(), group), dim=0)


def gather_samples(offsets: torch.Tensor, src: torch.Tensor, dst: torch.Tensor, depth: torch.Tensor, group=None):
    """Concatenate per-rank sampling outputs (offsets [n_r + 1] + edge arrays) into one
    instance-ordered result: offsets are re-based onto the concatenated edge arrays."""
    offs = _all_gather_var(offsets[:-1].contiguous(), group)
    tot = _all_gather_var(offsets[-1:].contiguous(), group)
    srcs = _all_gather_var(src.contiguous(), group)
    dsts = _all_gather_var(dst.contiguous(), group)
    deps = _all_gather_var(depth.contiguous(), group)
    base = 0
    out_offs = []
    for o, t in zip(offs, tot):
        out_offs.append(o + base)
        base += int(t[0].item())
    out_offs.append(torch.tensor([base], dtype=offsets.dtype, device=offsets.device))
    return torch.cat(out_offs), torch.cat(srcs), torch.cat(dsts), torch.cat(deps)
