"""NEXT-4(iii): out-of-memory ablation (§6 Fig. 13-15).

The paper measures, with 4 partitions, 2 resident and 2 streams, the effect of
multi-instance batched sampling (BA), workload-aware partition scheduling (WS)
and thread-block workload balancing (BAL) on biased neighbor sampling, biased
random walk, forest fire and unbiased neighbor sampling, "pretending" graphs do
not fit.  Here the same four applications run on a synthetic
R-MAT graph under an imposed device budget, in four schedules:

  full      BA + WS + BAL (the method)
  -BAL      CTAs split evenly between a wave's partition kernels
  -WS       partitions taken round-robin by id, FIFO eviction
  -BA       instances sampled in separate calls of --group instances each
            (no cross-instance batching: every group re-walks the partitions)

and reports time per run, partition transfers (Fig. 15's metric) and
hot-kernel time.  All schedules produce identical outputs (checked).
Output: one JSON document on stdout.

    python scripts/ablation_oom.py [--config cfg2] [--instances 4096] [--walk-length 200]
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


def budget(g, P, R):
    V = g.row_ptr.numel() - 1
    rp = g.row_ptr.numpy()
    b = [p * (V // P) + min(p, V % P) for p in range(P + 1)]   # equal ranges, remainder to the lowest
    maxpe = max(int(rp[b[p + 1]] - rp[b[p]]) for p in range(P))
    return 8 * (V + 1) + 4 * V + R * maxpe * 4 + (64 << 20)


def timed(G, app, seeds, args, group=0):
    """(ms, partition loads, hot kernel ms, outputs) of one run (group > 0: -BA)."""
    chunks = [(0, seeds)] if group <= 0 else [(i, seeds[i:i + group]) for i in range(0, seeds.numel(), group)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    loads, hot = 0, 0.0
    outs = []
    e0.record()
    for base, s in chunks:
        if app == "biased RW":
            outs.append(cs.csaw_walk(G, "degree", s, args.walk_length, rng_seed=1, instance_base=base))
        else:
            kind = {"biased NS": "degree", "forest fire": "forest_fire", "unbiased NS": "uniform"}[app]
            fan = [] if kind == "forest_fire" else [2, 2]
            outs.append(cs.csaw_sample(G, cs.make_bias(kind, pf=0.7), s, fanout=fan, depth=2, rng_seed=1,
                                       instance_base=base))
        st = cs.csaw_stats(G)
        loads += st["partition_loads"]
        hot += st["hot_kernel_ms"]
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), loads, hot, outs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2", help="graph shape (its R-MAT graph)")
    ap.add_argument("--instances", type=int, default=4096)
    ap.add_argument("--walk-length", type=int, default=200)
    ap.add_argument("--partitions", type=int, default=4)
    ap.add_argument("--resident", type=int, default=2)
    ap.add_argument("--group", type=int, default=256, help="-BA: instances per separate call")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    dev = torch.device("cuda:0")
    g = rmat_csr(cfg.graph_vertices, cfg.graph_entries, cfg.graph_seed, device=dev).to("cpu")
    seeds = instance_seeds(g, args.instances).to(dev)
    P, R = args.partitions, args.resident
    bud = budget(g, P, R)
    out = {"graph": args.config, "V": g.row_ptr.numel() - 1, "E": g.col_idx.numel(), "instances": args.instances,
           "walk_length": args.walk_length, "partitions": P, "resident": R, "streams": 2, "budget_bytes": bud,
           "group_without_BA": args.group, "results": []}
    graphs = {
        "full": cs.csaw_graph_create(g.row_ptr, g.col_idx, budget_bytes=bud, num_partitions=P, max_resident=R,
                                     num_streams=2),
        "-BAL": cs.csaw_graph_create(g.row_ptr, g.col_idx, budget_bytes=bud, num_partitions=P, max_resident=R,
                                     num_streams=2, oom_bal=False),
        "-WS": cs.csaw_graph_create(g.row_ptr, g.col_idx, budget_bytes=bud, num_partitions=P, max_resident=R,
                                    num_streams=2, oom_ws=False),
    }
    for app in ("biased NS", "biased RW", "forest fire", "unbiased NS"):
        row = {"application": app}
        ref = None
        for name in ("full", "-BAL", "-WS", "-BA"):
            G = graphs["full" if name == "-BA" else name]
            group = args.group if name == "-BA" else 0
            timed(G, app, seeds, args, group)   # warm-up (residency from a previous run is kept: fair to all)
            best = None
            for _ in range(args.reps):
                ms, loads, hot, outs = timed(G, app, seeds, args, group)
                if best is None or ms < best[0]:
                    best = (ms, loads, hot)
            if name != "-BA":
                flat = outs[0] if app != "biased RW" else (outs[0],)
                if ref is None:
                    ref = flat
                same = all(torch.equal(a.cpu(), b.cpu()) for a, b in zip(ref, flat))
            elif app == "biased RW":
                same = bool(torch.equal(torch.cat(outs), ref[0]))
            else:
                same = int(sum(o[1].numel() for o in outs)) == int(ref[1].numel())   # same edge count
            row[name] = {"ms": best[0], "partition_loads": best[1], "hot_kernel_ms": best[2], "identical": same}
        f = row["full"]["ms"]
        row["speedup_BA"] = row["-BA"]["ms"] / f
        row["speedup_WS"] = row["-WS"]["ms"] / f
        row["speedup_BAL"] = row["-BAL"]["ms"] / f
        row["transfer_reduction_WS"] = row["-WS"]["partition_loads"] / max(row["full"]["partition_loads"], 1)
        out["results"].append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
    for G in graphs.values():
        G.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
