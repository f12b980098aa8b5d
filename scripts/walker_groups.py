"""cfg2 per-step scan path (materialised degree bias) at 4,000 / 1,000 / 500 walkers:
the walker-group width G follows the walker count (1 / 2..8 warps per walker)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_09103_b200 as cs  # noqa: E402
from synth import CONFIGS, instance_seeds, rmat_csr  # noqa: E402

cfg = CONFIGS["cfg2"]
dev = torch.device("cuda:0")
g = rmat_csr(cfg.graph_vertices, cfg.graph_entries, cfg.graph_seed, device=dev)
G = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=0, edge_bias=True)
seeds = instance_seeds(g, 4000).to(dev)
flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)
for n in (4000, 1000, 500, 148):
    s = seeds[:n].contiguous()
    out = torch.empty((n, cfg.length + 1), dtype=torch.int32, device=dev)
    cs.csaw_walk(G, "degree", s, cfg.length, rng_seed=1, out=out)
    ts = []
    for r in range(3):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cs.csaw_walk(G, "degree", s, cfg.length, rng_seed=1 + r, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sum(ts) / len(ts)
    print(f"walkers {n:5d}: {ms:8.2f} ms/step  {n * cfg.length / ms * 1e3:.3e} SEPS")
