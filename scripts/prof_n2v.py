"""Small node2vec launch on the cfg3 graph for ncu (the full workload is too long to replay).

    python scripts/prof_n2v.py <stride> [cache]
"""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_09103_b200 as cs
from synth import CONFIGS, rmat_csr, nonisolated_vertices
cfg = CONFIGS["cfg3"]
g = rmat_csr(cfg.graph_vertices, cfg.graph_entries, cfg.graph_seed, device="cuda")
G = cs.csaw_graph_create(g.row_ptr, g.col_idx, node2vec_tri="cache" in sys.argv[2:])  # "cache": k_node2vec_tri
seeds = nonisolated_vertices(g)[:: max(1, int(sys.argv[1]) if len(sys.argv) > 1 else 40)].to(torch.int32).cuda()
b = cs.make_bias("node2vec", p=cfg.p, q=cfg.q)
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); cs.csaw_walk(G, b, seeds, cfg.length, rng_seed=1); e1.record(); torch.cuda.synchronize()
    print("walkers", seeds.numel(), "ms", e0.elapsed_time(e1), "SEPS", seeds.numel() * cfg.length / e0.elapsed_time(e1) * 1e3)
