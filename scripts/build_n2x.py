"""Build the cfg3 graph with the node2vec intersection index (ncu target for the build kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_09103_b200 as cs  # noqa: E402
from synth import CONFIGS, rmat_csr  # noqa: E402

cfg = CONFIGS["cfg3"]
g = rmat_csr(cfg.graph_vertices, cfg.graph_entries, cfg.graph_seed, device=torch.device("cuda:0"))
torch.cuda.synchronize()
G = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=0, node2vec_index=True)
print(G.info())
