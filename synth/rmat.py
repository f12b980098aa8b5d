"""R-MAT graph generator and the G_toy fixture (inputs only, no sampling math).

Recipe:
  1. Draw E/2 undirected R-MAT edges at scale ceil(log2 V) with the Graph500
     quadrant probabilities (a, b, c, d) = (0.57, 0.19, 0.19, 0.05).
  2. Reject endpoints >= V and self-loops.
  3. Scramble labels with a hash-keyed permutation of [0, V) (balances the
     equal vertex-range partitions of the out-of-memory mode, §5.1).
  4. Symmetrise, sort each row ascending and drop duplicates.
The resulting CSR has row_ptr int64[V+1], col_idx int32[E'] (values < V, read
as uint32 by the C ABI), sorted rows, no self-loops, no duplicate entries.
E' (the number of CSR entries) is reported; it is below E because of rejection
and deduplication.

All randomness is a 32-bit integer hash computed in int64 tensors with every
intermediate product < 2**63, so CPU and CUDA generation agree bit for bit.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

_M32 = 0xFFFFFFFF


def _mul32(x: torch.Tensor, c: int) -> torch.Tensor:
    """(x * c) mod 2**32 for x in [0, 2**32) held in int64, without int64 overflow."""
    ch, cl = c >> 16, c & 0xFFFF
    lo = x * cl                                   # < 2**48
    hi = ((x * ch) & 0xFFFF) << 16                # < 2**32
    return (lo + hi) & _M32


def mix32(x: torch.Tensor) -> torch.Tensor:
    """lowbias32 integer hash (C. Wellons), elementwise on int64 holding uint32."""
    x = x & _M32
    x = x ^ (x >> 16)
    x = _mul32(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32(x, 0x846CA68B)
    x = x ^ (x >> 16)
    return x


def _mix32_int(x: int) -> int:
    x &= _M32
    x ^= x >> 16
    x = (x * 0x7FEB352D) & _M32
    x ^= x >> 15
    x = (x * 0x846CA68B) & _M32
    x ^= x >> 16
    return x


def stream_key(graph_seed: int, purpose: int, level: int = 0) -> int:
    """32-bit key for one hash stream (purpose tags: 1 = R-MAT level, 2 = permutation, 3 = seeds)."""
    k = _mix32_int(graph_seed * 0x9E3779B1 + 0x632BE5AB)
    k = _mix32_int(k ^ (purpose * 0x85EBCA77))
    k = _mix32_int(k ^ (level * 0xC2B2AE3D + 0x27D4EB2F))
    return k


def hash_stream(idx: torch.Tensor, key: int) -> torch.Tensor:
    """Uniform 32-bit values for indices idx (< 2**32) under a stream key."""
    h = mix32(idx ^ key)
    return mix32(h + (key ^ 0x165667B1))


@dataclass
class RmatGraph:
    num_vertices: int
    row_ptr: torch.Tensor      # int64 [V+1]
    col_idx: torch.Tensor      # int32 [E'] (uint32 semantics)
    graph_seed: int
    target_edges: int

    @property
    def num_edges(self) -> int:
        return int(self.col_idx.numel())

    def degrees(self) -> torch.Tensor:
        return (self.row_ptr[1:] - self.row_ptr[:-1])

    def to(self, device) -> "RmatGraph":
        return RmatGraph(self.num_vertices, self.row_ptr.to(device), self.col_idx.to(device),
                         self.graph_seed, self.target_edges)


# Graph500 R-MAT quadrant probabilities.
RMAT_A, RMAT_B, RMAT_C = 0.57, 0.19, 0.19


def _rmat_edges(first: int, count: int, scale: int, graph_seed: int, device) -> tuple[torch.Tensor, torch.Tensor]:
    t1 = int(RMAT_A * 2**32)
    t2 = int((RMAT_A + RMAT_B) * 2**32)
    t3 = int((RMAT_A + RMAT_B + RMAT_C) * 2**32)
    idx = torch.arange(first, first + count, dtype=torch.int64, device=device)
    src = torch.zeros(count, dtype=torch.int64, device=device)
    dst = torch.zeros(count, dtype=torch.int64, device=device)
    for level in range(scale):
        h = hash_stream(idx, stream_key(graph_seed, 1, level))
        q = (h >= t1).to(torch.int64) + (h >= t2).to(torch.int64) + (h >= t3).to(torch.int64)
        src = (src << 1) | (q >> 1)
        dst = (dst << 1) | (q & 1)
        del h, q
    return src, dst


def rmat_csr(num_vertices: int, target_entries: int, graph_seed: int, device="cpu",
             chunk: int = 1 << 26, fill: bool = True) -> RmatGraph:
    """Symmetric, deduplicated R-MAT CSR with ~target_entries entries (see module doc).

    fill=True keeps drawing (a longer prefix of the same edge stream) until the
    deduplicated CSR has >= 97 % of target_entries, so rejection of ids >= V and
    duplicate edges do not shrink the graph below the paper's Table 2 size."""
    n_draw = target_entries // 2
    g = None
    for _ in range(4 if fill else 1):
        g = _rmat_once(num_vertices, target_entries, n_draw, graph_seed, device, chunk)
        got = g.num_edges
        if not fill or got >= 0.97 * target_entries or got == 0:
            break
        n_draw = int(n_draw * min(4.0, target_entries / got) * 1.01) + 1
    return g


def _rmat_once(num_vertices: int, target_entries: int, n_undirected: int, graph_seed: int, device,
               chunk: int) -> RmatGraph:
    V = int(num_vertices)
    if V < 2:
        raise ValueError("need at least 2 vertices")
    scale = max(1, math.ceil(math.log2(V)))
    # label permutation: sort (hash << 32 | v) -> unique, deterministic keys
    v = torch.arange(V, dtype=torch.int64, device=device)
    pkey = (hash_stream(v, stream_key(graph_seed, 2)) << 32) | v
    perm = torch.argsort(pkey)          # perm[v] = new label of old vertex v
    del pkey, v
    keys = []
    for first in range(0, n_undirected, chunk):
        cnt = min(chunk, n_undirected - first)
        s, d = _rmat_edges(first, cnt, scale, graph_seed, device)
        ok = (s < V) & (d < V) & (s != d)
        s, d = perm[s[ok]], perm[d[ok]]
        keys.append((s << 32) | d)
        keys.append((d << 32) | s)
        del s, d, ok
    key = torch.cat(keys) if keys else torch.empty(0, dtype=torch.int64, device=device)
    del keys
    key, _ = torch.sort(key)
    if key.numel() > 1:
        keep = torch.ones(key.numel(), dtype=torch.bool, device=device)
        keep[1:] = key[1:] != key[:-1]
        key = key[keep]
        del keep
    src = key >> 32
    col = (key & _M32).to(torch.int32)
    del key
    counts = torch.bincount(src, minlength=V)
    del src
    row_ptr = torch.zeros(V + 1, dtype=torch.int64, device=device)
    row_ptr[1:] = torch.cumsum(counts, 0)
    return RmatGraph(V, row_ptr, col, graph_seed, target_entries)


def gtoy_csr() -> RmatGraph:
    """G_toy: 12 vertices, 16 undirected edges.

    Consistent with every stated fact of PAPER.md Fig. 1(a) caption (line 127:
    N(v8) = {v5, v7, v9, v10, v11} with neighbour degrees 3, 6, 2, 2, 2 giving
    S = {0,3,9,11,13,15}, lines 226-229), Fig. 4 caption (line 404: pool
    {v8, v0, v3}, v8 -> v7 is an edge) and §5.2's Fig. 8 example (lines
    857-863: 0-7, 2-3, 8-5, 3-4 are edges; seeds {0,2,8} give active counts
    (2,0,1) over 3 partitions).  The figure bodies themselves are stripped, so
    this graph is a constructed fixture, not the paper's exact drawing.
    """
    row_ptr = [0, 1, 2, 4, 6, 9, 12, 15, 21, 26, 28, 30, 32]
    col = [7, 7, 3, 7, 2, 4, 3, 5, 7, 4, 6, 8, 5, 7, 11, 0, 1, 2, 4, 6, 8,
           5, 7, 9, 10, 11, 8, 10, 8, 9, 6, 8]
    return RmatGraph(12, torch.tensor(row_ptr, dtype=torch.int64),
                     torch.tensor(col, dtype=torch.int32), 0, 32)


def degree_stats(g: RmatGraph) -> dict:
    """Shape statistics printed in every run report."""
    deg = g.degrees().to(torch.float64)
    V = g.num_vertices
    E = g.num_edges
    s1 = float(deg.sum())
    s2 = float((deg * deg).sum())
    return {
        "V": V, "E_entries": E, "E_target": g.target_edges,
        "isolated_frac": float((deg == 0).sum()) / V,
        "max_deg": int(deg.max()) if V else 0,
        "mean_deg": s1 / V if V else 0.0,
        "E_pi_simple_deg": (s2 / s1) if s1 else 0.0,
    }
