"""Seeded edge weights for the EdgeBias = w(e) path (inputs only, no sampling math).

Recipe: the weight of an undirected edge {u, v} is a
function of the pair (both CSR entries (u -> v) and (v -> u) carry the same value),
built from the input hash as mantissa x power of two so every value is exact in
fp32 and identical on CPU and CUDA:
    h = hash((min(u,v) * 2654435761 + max(u,v)) mod 2^32),   # 32-bit pair key
    w = (1 + (h & 0xFFFF)) * 2^(((h >> 16) % 9) - 20)        # 2^-20 .. 2^4, 17-bit mantissa
and a fraction `zero_frac` of edges (by a second hash of the pair) get w = 0
(zero-width CTPS regions that must never be chosen, R4).
"""
from __future__ import annotations

import torch

from .rmat import RmatGraph, hash_stream, stream_key

_M32 = 0xFFFFFFFF


def edge_weights(g: RmatGraph, seed: int = 1, zero_frac: float = 0.0) -> torch.Tensor:
    """float32 [E'] aligned with g.col_idx (same device)."""
    rp, col = g.row_ptr, g.col_idx.to(torch.int64) & _M32
    src = torch.repeat_interleave(torch.arange(g.num_vertices, device=rp.device), rp[1:] - rp[:-1])
    lo, hi = torch.minimum(src, col), torch.maximum(src, col)
    pair = (lo * 2654435761 + hi) & _M32          # lo < 2^32, product < 2^64 / 2: fits int64
    h = hash_stream(pair, stream_key(seed, 6))
    mant = (1 + (h & 0xFFFF)).to(torch.float32)
    ex = ((h >> 16) % 9 - 20).to(torch.float32)
    w = mant * torch.pow(torch.full_like(mant, 2.0), ex)
    if zero_frac > 0:
        z = hash_stream(pair, stream_key(seed, 7))
        w = torch.where(z < int(zero_frac * 2**32), torch.zeros_like(w), w)
    return w.contiguous()
