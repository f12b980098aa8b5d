import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2009_09103_b200 as cs, oracle as O
from synth import rmat_csr, instance_seeds, nonisolated_vertices, CONFIGS
from tests._parity import check_walk, graph_pair
g = rmat_csr(1 << 15, 1 << 19, 7, device='cuda').to('cpu')
G, og = graph_pair(g.row_ptr, g.col_idx)
seeds = instance_seeds(g, 256).numpy()
check_walk(G, og, "node2vec", seeds, 40, rng_seed=3, p=2.0, q=0.5)
print("medium ok", flush=True)
from tests.test_gpu_parity import hub_csr
rp, col = hub_csr()
G2, og2 = graph_pair(rp, col)
check_walk(G2, og2, "node2vec", np.array([0, 1, 0, 1, 5, 0, 1, 17], np.uint32), 12, rng_seed=9, p=2.0, q=0.5)
print("hub ok", flush=True)
cfg = CONFIGS["cfg3"]
g3 = rmat_csr(cfg.graph_vertices, cfg.graph_entries, cfg.graph_seed, device='cuda')
G3 = cs.csaw_graph_create(g3.row_ptr, g3.col_idx)
og3 = O.Graph(g3.row_ptr.cpu().numpy(), g3.col_idx.cpu().numpy().view(np.uint32))
s3 = nonisolated_vertices(g3)[:20000].to(torch.int32).cuda()
check_walk(G3, og3, "node2vec", s3.cpu().numpy(), 80, rng_seed=1, p=2.0, q=0.5, walkers=range(0, 20000, 500))
print("cfg3 subset ok", flush=True)
