"""Per-rank work of bench.py's strong-scaling split, timed on ONE GPU (a prediction, not the
SCALE measurement): for N = 1, 2, 4, 8 every rank r runs the same kernels on its contiguous share
bench.make_seeds(cfg, g, r, N, "strong") with no communication in the timed region, so a rank's
time on its own GPU is the time of its share alone.  Predicted SEPS(N) = all edges / the slowest
share's time.  CUDA events on the launching stream, L2 flushed before each timed call.

    python scripts/strong_shares.py cfg3 cfg2 > profiles/r02d_strong_shares.md
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2009_09103_b200 as cs  # noqa: E402
from synth import CONFIGS, rmat_csr  # noqa: E402


def time_call(fn, flush, reps=3):
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


def main(names):
    dev = torch.device("cuda:0")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    print("# Strong-scaling shares timed on one B200 (prediction; `scripts/strong_shares.py`)\n")
    print("Each rank of `bench.py --gpus N` runs its contiguous share of the config's instances with no "
          "communication in the timed region; this times every share alone on one GPU (min of 3, L2 flushed).  "
          "Predicted SEPS(N) = all edges / the slowest share.  The driver's SCALE run measures the real thing.\n")
    print("| config | N | slowest share (ms) | shares (ms) | predicted SEPS | predicted efficiency |")
    print("|---|---|---|---|---|---|")
    for name in names:
        cfg = CONFIGS[name]
        g = rmat_csr(cfg.graph_vertices, cfg.graph_entries, cfg.graph_seed, device=dev)
        if cfg.workload == "node2vec":
            G = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=0, node2vec_index=True)
            bias = cs.make_bias("node2vec", p=cfg.p, q=cfg.q)
        else:
            G = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=0, ctps_cache=True, walk_buckets=True)
            bias = cs.make_bias(cfg.bias)
        seps1 = None
        for N in (1, 2, 4, 8):
            ts = []
            edges = 0
            for r in range(N):
                base, seeds, _ = bench.make_seeds(cfg, g, r, N, "strong")
                seeds = seeds.to(dev)
                out = torch.empty((seeds.numel(), cfg.length + 1), dtype=torch.int32, device=dev)
                fn = lambda: cs.csaw_walk(G, bias, seeds, cfg.length, instance_base=base, rng_seed=1, out=out)  # noqa: E731
                fn()
                torch.cuda.synchronize()
                ts.append(time_call(fn, flush))
                edges += seeds.numel() * cfg.length
                del out
            seps = edges / (max(ts) / 1e3)
            if N == 1:
                seps1 = seps
            shares = ", ".join(f"{t:.3f}" for t in ts)
            print(f"| {name} | {N} | {max(ts):.3f} | {shares} | {seps:.3g} | {seps / (N * seps1):.2f} |")
        G.close()
        del g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg3", "cfg2"])
