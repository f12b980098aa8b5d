"""Time the node2vec-index build kernels of the cfg3 graph (run under ncu --metrics gpu__time_duration.sum)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2009_09103_b200 as cs
from synth import CONFIGS, rmat_csr
cfg = CONFIGS["cfg3"]
g = rmat_csr(cfg.graph_vertices, cfg.graph_entries, cfg.graph_seed, device="cuda:0")
torch.cuda.synchronize()
t0 = time.time()
G = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=0, node2vec_index=True)
torch.cuda.synchronize()
print("create s", time.time() - t0, G.info()["cache_build_ms"])
