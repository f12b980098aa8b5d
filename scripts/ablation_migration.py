"""NEXT-2: collision-migration ablation (§6.2, Fig. 10-11).

Times csaw_sample for the four sampling algorithms of Fig. 10 (biased neighbor
sampling, forest fire, layer sampling, unbiased neighbor sampling) under the
three collision-migration modes of §4.2 -- bipartite region search (the
method), repeated sampling (Fig. 6(a)) and updated sampling (Fig. 6(b)) -- and
reports time per call and random draws per selected vertex (Fig. 11's
"#iterations").  All three modes sample the same distribution; they differ in
draws and work.  Output: one JSON document (stdout).

    python scripts/ablation_migration.py [--config cfg2] [--instances 2000] [--fanout 2 2]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2009_09103_b200 as cs  # noqa: E402
from synth import CONFIGS, instance_seeds, rmat_csr  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2", help="graph shape to use (its R-MAT graph)")
    ap.add_argument("--instances", type=int, default=2000)
    ap.add_argument("--fanout", type=int, nargs="+", default=[2, 2])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cache", action="store_true", help="use the static-bias CTPS cache")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    dev = torch.device("cuda:0")
    g = rmat_csr(cfg.graph_vertices, cfg.graph_entries, cfg.graph_seed, device=dev)
    seeds = instance_seeds(g, args.instances).to(dev)
    out = {"graph": args.config, "instances": args.instances, "fanout": args.fanout, "cache": args.cache,
           "batched_driver": True, "results": []}
    # the batched driver is the paper's structure (one queue of all instances)
    G = cs.csaw_graph_create(g.row_ptr, g.col_idx, ctps_cache=args.cache, batched_only=True)
    algos = [("biased NS", "degree", {}), ("forest fire", "forest_fire", {"pf": 0.7}),
             ("layer", "layer", {}), ("unbiased NS", "uniform", {})]
    for name, kind, kw in algos:
        row = {"algorithm": name}
        ref = None
        for mode in ("brs", "repeated", "updated"):
            b = cs.make_bias(kind, migration=mode, **kw)
            fan = args.fanout if kind != "forest_fire" else []
            depth = len(args.fanout)
            r = cs.csaw_sample(G, b, seeds, fanout=fan, depth=depth, rng_seed=1)   # warm-up
            times = []
            for _ in range(args.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                r = cs.csaw_sample(G, b, seeds, fanout=fan, depth=depth, rng_seed=1)
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
            st = cs.csaw_stats(G)
            edges = int(r[1].numel())
            row[mode] = {"ms": sorted(times)[len(times) // 2], "hot_kernel_ms": st["hot_kernel_ms"],
                         "draws": st["draws"], "edges": edges,
                         "draws_per_pick": st["draws"] / max(edges, 1)}
            if ref is None:
                ref = r[1].numel()
        row["brs_speedup_vs_repeated"] = row["repeated"]["hot_kernel_ms"] / max(row["brs"]["hot_kernel_ms"], 1e-9)
        row["brs_speedup_vs_updated"] = row["updated"]["hot_kernel_ms"] / max(row["brs"]["hot_kernel_ms"], 1e-9)
        row["draw_reduction_vs_repeated"] = row["repeated"]["draws_per_pick"] / max(row["brs"]["draws_per_pick"], 1e-9)
        out["results"].append(row)
    print(json.dumps(out, indent=1))
    G.close()


if __name__ == "__main__":
    main()
