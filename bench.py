#!/usr/bin/env python
"""bench.py — C-SAW hot path on B200: sampled edges per second (SEPS) + roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--scaling strong|weak]
                    [--impl ours|reference]

A "step" is one pass of the whole hot path over one batch of synthetic input.
The default workload is cfg3 (BASELINE.json configs[2]): the node2vec walk
(p = 2, q = 0.5, length 80) of one walker per non-isolated vertex (~1.89M) on
the Orkut-shaped R-MAT graph -- the largest config that BASELINE.json does not
tag as multi-GPU (DESIGN.md §6 "Which config is the bench line").  Inputs are
synthetic (synth/, seeded) and resident in HBM when the timed region starts; L2
is flushed (256 MB write) before every timed step; each step is timed with CUDA
events on the launching stream.  Timed steps cycle through the rng seeds 1, 2, 3
(the mean over three seed sets).

Multi-GPU (§8(e)): one process per GPU.  `--gpus N` without a torchrun
environment re-launches itself under torch.distributed.run.  Default is STRONG
scaling: the config's fixed instance set is split into contiguous ranges, one
per rank (Fig. 17), instance ids stay global (Philox
counter), so the union of the ranks' outputs is bit-identical to N = 1.
`--scaling weak` gives every rank the full workload on its own id range.  No
collective on the data path; max-over-ranks device time; NCCL only for the
optional output gather after timing.  The oracle (oracle/) runs only in the
cpu_baseline leg and in --impl reference.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from synth import (CONFIGS, degree_stats, edge_weights, instance_seeds, mdrw_seeds, nonisolated_vertices,  # noqa: E402
                   rmat_csr)

METRIC = "sampled edges/sec (SEPS) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "sampled_edges/s"
L2_FLUSH_BYTES = 256 << 20
DEFAULT_CONFIG = "cfg3"


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong (default): the config's instance set split across ranks; weak: every rank runs "
                         "the whole config on its own instance-id range")
    ap.add_argument("--rng-seeds", default="1,2,3", help="timed steps cycle through these Philox seeds (P:968)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="oracle CPU-baseline budget (wall s)")
    ap.add_argument("--gather", action="store_true", help="NCCL-gather outputs after timing (reported apart)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--in-memory", action="store_true", help="cfg5: ignore the OOM budget (in-memory MDRW)")
    ap.add_argument("--no-cache", action="store_true",
                    help="disable the static-bias CTPS cache / node2vec triangle counts (scan every pool)")
    ap.add_argument("--gather-bias", action="store_true",
                    help="with --no-cache: degree walks gather deg[u] per neighbour instead of streaming the "
                         "materialised per-edge bias (CSAW_GRAPH_EDGE_BIAS)")
    ap.add_argument("--scan-path-steps", type=int, default=1,
                    help="detail.scan_path: time this many steps of the config's per-step scan path (no caches; "
                         "0 = skip)")
    ap.add_argument("--no-zerocopy", action="store_true", help="OOM configs: skip the zero-copy OOM variant")
    ap.add_argument("--oom-budget-gb", type=float, default=0.0,
                    help="OOM configs: override the device budget (1e9 B) -- experiments only, the config names 8 GB")
    ap.add_argument("--oom-store", default="host", choices=["host", "peer"],
                    help="OOM configs: partition store in pinned host memory (the paper) or in a peer GPU's HBM "
                         "(NEXT-4(i), CSAW_GRAPH_OOM_PEER_STORE; with one GPU a same-device stand-in)")
    ap.add_argument("--oom-variant", default="partition", choices=["partition", "zerocopy"],
                    help="OOM configs: time the paper's partition scheduling (default) or the zero-copy mode")
    ap.add_argument("--no-walk-buckets", action="store_true",
                    help="degree walks: the vertex-head walk index (k_walk_head) instead of the bucketed index "
                         "(CSAW_GRAPH_WALK_BUCKETS, k_walk_gb) (A/B)")
    ap.add_argument("--mdrw-alt-records", action="store_true",
                    help="MDRW: the other slot-record layout (CSAW_GRAPH_MDRW_ALT_RECORDS: packed 8 B {row, degree} "
                         "+ vertex ids instead of 16 B {v, degree, row} records) (A/B)")
    ap.add_argument("--next-meta", action="store_true",
                    help="MDRW: 8 B next-vertex metadata + col (CSAW_GRAPH_NEXT_META) instead of the 16 B "
                         "next-vertex records (CSAW_GRAPH_NEXT_RECORD) (A/B)")
    return ap.parse_args(argv)


# ------------------------------------------------------------------ self-launch (--gpus N)
def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_spawn(args) -> int | None:
    """`--gpus N` (N > 1) outside torchrun: re-launch this script as N ranks under
    torch.distributed.run on 127.0.0.1 and return its exit code (None = run here)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


# ------------------------------------------------------------------ workload description
def workload_of(cfg):
    return {"walk": "walk", "node2vec": "walk", "mdrw": "walk",
            "neighbor": "sample", "layer": "sample", "forest_fire": "sample"}[cfg.workload]


def make_graph(cfg, device):
    t0 = time.perf_counter()
    g = rmat_csr(cfg.graph_vertices, cfg.graph_entries, cfg.graph_seed, device=device)
    if device.type == "cuda":
        torch.cuda.synchronize(device)
    return g, time.perf_counter() - t0


def total_instances(cfg, g):
    if cfg.workload == "node2vec" and cfg.n_instances == 0:
        return int(nonisolated_vertices(g).numel())
    return cfg.n_instances


def make_seeds(cfg, g, rank, world, scaling):
    """(instance_base, seeds, n_total) of this rank.  strong: the config's instances split
    into contiguous ranges [floor(rN/W), floor((r+1)N/W)); weak: N instances per rank
    with global ids [rN, (r+1)N)."""
    N = total_instances(cfg, g)
    if scaling == "strong":
        lo, hi, total = rank * N // world, (rank + 1) * N // world, N
    else:
        lo, hi, total = rank * N, (rank + 1) * N, N * world
    if cfg.workload == "node2vec":
        verts = nonisolated_vertices(g)
        idx = torch.arange(lo, hi, device=verts.device) % verts.numel()   # one walker per non-isolated vertex
        return lo, verts[idx].to(torch.int32), total
    if cfg.workload == "mdrw":
        s = mdrw_seeds(g, hi, cfg.pool_size)
        return lo, s[lo:hi].contiguous(), total
    s = instance_seeds(g, hi)
    return lo, s[lo:hi].contiguous(), total


def bias_of(cs, cfg):
    return {"walk": cs.make_bias(cfg.bias), "node2vec": cs.make_bias("node2vec", p=cfg.p, q=cfg.q),
            "mdrw": cs.make_bias("mdrw", pool_size=cfg.pool_size), "neighbor": cs.make_bias(cfg.bias),
            "layer": cs.make_bias("layer"), "forest_fire": cs.make_bias("forest_fire", pf=cfg.pf)}[cfg.workload]


# ------------------------------------------------------------------ §8(d) algorithmic bytes
def _bit_length(x: torch.Tensor) -> torch.Tensor:
    """bit length of non-negative int64 x (exact: frexp of the float64 value), so
    ceil(log2 d) = bit_length(d - 1)."""
    _, e = torch.frexp(x.to(torch.float64))
    return torch.where(x > 0, e.to(torch.int64), torch.zeros_like(x))


BYTES_MODEL = {
    "walk_degree_scan": "SURVEY §8(d) degree-biased pool: 16 (row_ptr pair) + 8 d(v) (col + deg) per step + 4 (path)",
    "walk_degree_stream": "per-step scan of the materialised degree bias (CSAW_GRAPH_EDGE_BIAS): 16 (row_ptr "
                          "pair) + 4 d(v) (the pool's biases, streamed) + 4 (the pick's col) + 4 (path)",
    "walk_degree_cached": "SURVEY §8(f) NEXT-1 cached CTPS: 32 B sectors x (row_ptr pair + ceil(log2 d(v)) probes "
                          "+ col) per step + 4 (path)",
    "walk_uniform": "16 (row_ptr pair) + 4 (one col entry) + 4 (path) per step",
    "walk_weight_cached": "SURVEY §8(f) NEXT-1 cached CTPS of the edge weights (fp64 prefix): 32 B sectors x (row_ptr "
                          "pair + ceil(log2 d(v)) probes + col) per step + 4 (path)",
    "walk_weight_stream": "per-step scan of the fp32 edge weights (float path): 16 (row_ptr pair) + 4 d(v) (the pool's "
                          "weights, streamed) + 4 (the pick's col) + 4 (path)",
    "node2vec": "SURVEY §8(d) node2vec step: 16 + 4 d(v) + 4 (N(prev) carried from the previous step); "
                "step 0 uniform: 16 + 4 + 4",
    "node2vec_index": "NEXT-1-style sector model of the node2vec intersection index: 32 B sectors x (the 128 B "
                      "record of the entry the walker arrived by (4 sectors) + the binary-search probes between its "
                      "splitters) per step + 4 (path); probes counted in the kernel",
    "mdrw": "SURVEY §8(d) MDRW step: 16 (row_ptr v) + 4 (col) + 4 (deg u) + 8 (edge out) = 32",
    "sample_degree": "SURVEY §8(d) degree-biased pool: 16 + 8 d(v) per expanded vertex + 9 per emitted edge",
    "sample_layer": "SURVEY §8(d) layer: sum over levels and frontier vertices of 16 + 8 d(v) + 9 per edge",
    "sample_ff": "SURVEY §8(d) uniform / FF expanded vertex: 16 + 4 x + 9 x (x = its emitted edges)",
    "sample_cached": "NEXT-1 sector model of the cached degree / layer pools: 16 (row_ptr pair) per expanded vertex + "
                     "32 B x (2 + ceil(log2 d(src))) + 9 per emitted edge",
    "oom_host": "host link: partition / zero-copy bytes moved H2D per step (library counters)",
}


def walk_alg_bytes(cfg, deg, out, cached, stream=False):
    """§8(d) bytes of one walk launch, from its output (device tensors)."""
    if cfg.workload == "mdrw":
        return 32 * out.shape[0] * out.shape[1], "mdrw"
    p = out.to(torch.int64) & 0xFFFFFFFF
    v = p[:, :-1]
    valid = v != 0xFFFFFFFF
    d = torch.where(valid, deg[torch.where(valid, v, torch.zeros_like(v))], torch.zeros_like(v))
    nsteps = int(valid.sum())
    if cfg.workload == "node2vec":
        first = int(valid[:, 0].sum())
        return int(16 * nsteps + 4 * d[:, 1:].sum() + 4 * first + 4 * nsteps), "node2vec"
    if cfg.bias == "uniform":
        return 24 * nsteps, "walk_uniform"
    if cfg.bias == "weight" and not cached:
        return int(16 * nsteps + 4 * d.sum() + 8 * nsteps), "walk_weight_stream"
    if cfg.bias == "weight":
        probes = _bit_length(torch.clamp(d - 1, min=0))
        return int(32 * (2 * nsteps + probes[valid].sum()) + 4 * nsteps), "walk_weight_cached"
    if cached:
        probes = _bit_length(torch.clamp(d - 1, min=0))
        return int(32 * (2 * nsteps + probes[valid].sum()) + 4 * nsteps), "walk_degree_cached"
    if stream:
        return int(16 * nsteps + 4 * d.sum() + 8 * nsteps), "walk_degree_stream"
    return int(16 * nsteps + 8 * d.sum() + 4 * nsteps), "walk_degree_scan"


def sample_alg_bytes(cfg, deg, seeds, offs, src, dst, dep, cached=False):
    """§8(d) bytes of one sampling launch: the expanded vertices of every level are the
    seed (level 0) and the new vertices of the previous level (UPDATE's post-filter)."""
    n = seeds.numel()
    V = deg.numel()
    m = src.numel()
    inst = torch.repeat_interleave(torch.arange(n, device=offs.device), (offs[1:] - offs[:-1]).to(torch.int64))
    s64 = src.to(torch.int64) & 0xFFFFFFFF
    d64 = dst.to(torch.int64) & 0xFFFFFFFF
    dp = dep.to(torch.int64)
    seeds64 = seeds.to(torch.int64) & 0xFFFFFFFF
    if cfg.workload == "forest_fire":
        # every expanded vertex: 16 + 4 x + 9 x; vertices that burned nothing still cost 16
        exp = [torch.ones(n, dtype=torch.int64, device=offs.device)]
        visited = inst * V + seeds64[inst]
        for lvl in range(1, cfg.depth):
            key = torch.unique((inst * V + d64)[dp == lvl])
            key = key[~torch.isin(key, torch.unique(visited))]
            exp.append(torch.ones(key.numel(), dtype=torch.int64, device=offs.device))
            visited = torch.cat([visited, key])
        npools = sum(int(e.numel()) for e in exp)
        return 16 * npools + 13 * m, "sample_ff"
    # degree / layer: every expanded vertex's whole neighbour list (16 + 8 d)
    level_keys = [torch.arange(n, device=offs.device) * V + seeds64]
    visited = level_keys[0]
    for lvl in range(1, cfg.depth):
        key = torch.unique((inst * V + d64)[dp == lvl])
        key = key[~torch.isin(key, visited)]
        level_keys.append(key)
        visited = torch.cat([visited, key])
    tot = 0
    if cached:   # NEXT-1 sector model: 16 B row_ptr pair per expanded vertex, 32 B x (2 + ceil(log2 d)) per pick
        for key in level_keys:
            tot += 16 * int(key.numel())
        ds = deg[s64]
        probes = _bit_length(torch.clamp(ds - 1, min=0))
        tot += int(32 * (2 * m + probes.sum())) + 9 * m
        return tot, "sample_cached"
    for key in level_keys:
        dv = deg[key % V]
        tot += int(16 * key.numel() + 8 * dv.sum())
    return tot + 9 * m, ("sample_layer" if cfg.workload == "layer" else "sample_degree")


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                power.append(float(parts[6]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "power_w_max": max(power) if power else None}


# ------------------------------------------------------------------ oracle CPU baseline
def _oracle_job(args):
    import oracle as O
    cfg_name, lo, hi, base, seeds, rng_seed = args
    cfg = CONFIGS[cfg_name]
    g = O._G
    edges = 0
    for j, i in enumerate(range(lo, hi)):
        gi = base + i
        s = seeds[j]
        if cfg.workload == "walk" and cfg.bias == "weight":
            O.weight_walk(g, cfg.length, int(s), gi, rng_seed)
            edges += cfg.length
        elif cfg.workload == "walk":
            O.walk(g, O.KIND_DEGREE if cfg.bias == "degree" else O.KIND_UNIFORM, cfg.length, int(s), gi, rng_seed)
            edges += cfg.length
        elif cfg.workload == "node2vec":
            O.node2vec(g, cfg.p, cfg.q, cfg.length, int(s), gi, rng_seed)
            edges += cfg.length
        elif cfg.workload == "mdrw":
            O.mdrw(g, s, cfg.length, gi, rng_seed)
            edges += cfg.length
        elif cfg.workload == "layer":
            edges += O.layer_sample(g, list(cfg.fanout), cfg.depth, int(s), gi, rng_seed)[0].size
        elif cfg.workload == "forest_fire":
            edges += O.neighbor_sample(g, O.KIND_FF, [], cfg.depth, int(s), gi, rng_seed, cfg.pf)[0].size
        else:
            edges += O.neighbor_sample(g, O.KIND_DEGREE if cfg.bias == "degree" else O.KIND_UNIFORM,
                                       list(cfg.fanout), cfg.depth, int(s), gi, rng_seed)[0].size
    return edges


def oracle_timed_sample(cfg, og, seeds_np, base, rng_seed, budget_s, workers=None):
    """Time the oracle (as it stands) over a bounded prefix of this config's instances on
    all host cores (independent instances).  Returns (SEPS, cores, sample text)."""
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor

    import oracle as O
    workers = workers or os.cpu_count() or 1
    n = len(seeds_np)
    O._G = og
    t0 = time.perf_counter()
    _oracle_job((cfg.name, 0, 1, base, seeds_np[:1], rng_seed))
    t1 = max(time.perf_counter() - t0, 1e-4)
    per_worker = max(1, int(budget_s / t1))
    m = int(min(n, per_worker * workers))
    m = max(m, min(n, workers))
    passes = max(1, min(1000, int(budget_s * workers / max(t1 * n, 1e-9)))) if m == n else 1
    chunks = np.array_split(np.arange(m), workers * 2)
    jobs = [(cfg.name, int(c[0]), int(c[-1]) + 1, base, seeds_np[int(c[0]):int(c[-1]) + 1], rng_seed)
            for c in chunks if c.size] * passes
    t0 = time.perf_counter()
    with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("fork")) as ex:
        edges = sum(ex.map(_oracle_job, jobs))
    wall = time.perf_counter() - t0
    sample = (f"{m} of {n} instances of {cfg.name} (full length/depth each)"
              + (f" x {passes} passes" if passes > 1 else "") + f", {workers} processes")
    return edges / wall, workers, sample, edges, wall


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    """The oracle, as it stands, on the box's host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    import oracle as O
    O.build()
    dev = torch.device("cuda:0") if torch.cuda.is_available() else torch.device("cpu")
    g, _ = make_graph(cfg, dev)
    base, seeds, _ = make_seeds(cfg, g, 0, 1, "strong")
    og = O.Graph.from_torch(g, edge_weights(g, cfg.graph_seed) if cfg.bias == "weight" else None)
    seeds_np = seeds.cpu().numpy().view(np.uint32)
    del g
    if dev.type == "cuda":
        torch.cuda.empty_cache()
    rng = [int(s) for s in args.rng_seeds.split(",")]
    per_step = max(2.0, 120.0 / max(1, args.steps + args.warmup))
    for i in range(args.warmup):
        oracle_timed_sample(cfg, og, seeds_np, base, rng[i % len(rng)], min(per_step, 3.0))
    vals, walls, samples = [], [], []
    for i in range(args.steps):
        v, cores, sample, edges, wall = oracle_timed_sample(cfg, og, seeds_np, base, rng[i % len(rng)], per_step)
        vals.append(v)
        walls.append(wall)
        samples.append(sample)
    value = statistics.mean(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * statistics.mean(walls),
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (seeded R-MAT, synth/)",
            "config": config_block(cfg, args.gpus, None, args.scaling, total_instances_cfg(cfg)),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": samples[-1]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def total_instances_cfg(cfg):
    return cfg.n_instances or "one walker per non-isolated vertex"


def config_block(cfg, world, stats_g, scaling, n_total, oom_mode=None, colc=None):
    c = {"workload": f"{cfg.name}: {cfg.description}", "instances_total": n_total,
         "graph": {"V": cfg.graph_vertices, "E_target": cfg.graph_entries,
                   "generator": "R-MAT Graph500 (0.57,0.19,0.19,0.05), symmetrised, dedup"},
         "parallelism": (f"strong scaling: the {n_total} instances split into {world} contiguous ranges, one per GPU; "
                         "CSR replicated" if scaling == "strong" else
                         f"weak scaling: every one of {world} GPU(s) runs the whole config on its own instance-id "
                         "range; CSR replicated"),
         "l2": "flushed (256 MB write) before every timed step; CSR also larger than L2"}
    if cfg.workload in ("walk", "node2vec", "mdrw"):
        c["length"] = cfg.length
    if cfg.fanout:
        c["fanout"] = list(cfg.fanout)
    if cfg.depth:
        c["depth"] = cfg.depth
    if cfg.workload == "node2vec":
        c["p"], c["q"] = cfg.p, cfg.q
    if cfg.workload == "forest_fire":
        c["pf"] = cfg.pf
    if cfg.workload == "mdrw":
        c["pool_size"] = cfg.pool_size
    if cfg.oom_budget_bytes:
        c["oom"] = {"device_budget_bytes": cfg.oom_budget_bytes, "partitions": cfg.oom_partitions,
                    "resident": cfg.oom_resident, "streams": cfg.oom_resident}
        if oom_mode == "zerocopy":
            c["oom"] = {"device_budget_bytes": cfg.oom_budget_bytes, "mode": "zero-copy: a col_idx prefix resident "
                        "within the budget, the rest read in place from pinned host memory",
                        "graph_device_bytes": colc}
        elif oom_mode:
            c["oom"]["mode"] = "partition scheduling (paper §5)"
    if stats_g:
        c["graph_stats"] = stats_g
    return c


def measure_h2d_peak(dev, nbytes=1 << 30, reps=5, store=None) -> float:
    """Pinned host -> device cudaMemcpyAsync bandwidth (GB/s, best of reps): the
    roofline of the OOM configs.  store = a GPU index: the
    store -> device copy of the peer partition store instead (NEXT-4(i))."""
    h = (torch.empty(nbytes, dtype=torch.uint8).pin_memory() if store is None
         else torch.empty(nbytes, dtype=torch.uint8, device=torch.device("cuda", store)))
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    best = 0.0
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = max(best, nbytes / (e0.elapsed_time(e1) / 1000.0) / 1e9)
    del h, d
    return best


# ------------------------------------------------------------------ our arm
def main():
    args = parse_args()
    rc = maybe_spawn(args)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference(args)
    import paper_2009_09103_b200 as cs
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        print(json.dumps({"metric": METRIC, "error": "no CUDA device: the library has no CPU fallback"}))
        return 1
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    cfg = CONFIGS[args.config]
    if args.oom_budget_gb > 0 and cfg.oom_budget_bytes:   # experiments only
        import dataclasses
        cfg = dataclasses.replace(cfg, oom_budget_bytes=int(args.oom_budget_gb * 1e9))
    kind = workload_of(cfg)
    rng_seeds = [int(s) for s in args.rng_seeds.split(",")]

    g, gen_s = make_graph(cfg, dev)
    gstats = degree_stats(g)
    deg = (g.row_ptr[1:] - g.row_ptr[:-1]).to(torch.int64)
    base, seeds, n_total = make_seeds(cfg, g, rank, world, args.scaling)
    seeds = seeds.to(dev).contiguous()
    n = seeds.shape[0]
    oom = cfg.oom_budget_bytes > 0 and not args.in_memory
    torch.cuda.empty_cache()   # return the generator's transient buffers: the library allocates with cudaMalloc
    if oom:
        # out-of-memory mode (§5): the device holds only what the imposed budget allows
        del deg
        g = g.to("cpu")
        torch.cuda.empty_cache()
        zc_main = args.oom_variant == "zerocopy"
        store = None
        if args.oom_store == "peer":
            ndev = torch.cuda.device_count()
            store = (local + 1) % ndev if ndev > 1 else local
        G = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=local, budget_bytes=cfg.oom_budget_bytes,
                                 num_partitions=cfg.oom_partitions, max_resident=1 if zc_main else cfg.oom_resident,
                                 num_streams=cfg.oom_resident, zerocopy=zc_main, store_device=store)
    else:
        use_cache = (not args.no_cache) and cfg.bias in ("degree", "layer")
        use_tri = (not args.no_cache) and cfg.workload == "node2vec"
        use_meta = (not args.no_cache) and cfg.workload == "mdrw"
        use_eb = args.no_cache and not args.gather_bias and cfg.workload == "walk" and cfg.bias == "degree"
        wts = edge_weights(g, cfg.graph_seed) if cfg.bias == "weight" else None
        # (the narrow walk index + vertex heads stay built beside the buckets: without them the bucket
        # build measured 222 vs 20-54 ms and the walk 1.233 vs 1.209 ms on cfg2)
        use_buckets = ((use_cache or cfg.bias == "weight") and cfg.workload == "walk" and not args.no_walk_buckets
                       and not args.no_cache)
        G = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=local, ctps_cache=use_cache, node2vec_tri=use_tri,
                                 next_meta=use_meta and args.next_meta, next_record=use_meta and not args.next_meta,
                                 walk_index=use_cache, node2vec_index=use_tri, edge_bias=use_eb,
                                 weights=wts, walk_buckets=use_buckets,
                                 flags=cs.CSAW_GRAPH_MDRW_ALT_RECORDS if args.mdrw_alt_records else 0)
    ginfo = G.info()
    bias = bias_of(cs, cfg)
    stream = torch.cuda.current_stream(dev)

    if kind == "walk":
        shape = (n, cfg.length, 2) if cfg.workload == "mdrw" else (n, cfg.length + 1)
        out_dev = torch.empty(shape, dtype=torch.int32, device=dev)

        def step(seed):
            cs.csaw_walk(G, bias, seeds, cfg.length, instance_base=base, rng_seed=seed, out=out_dev, stream=stream)
            return n * cfg.length
    else:
        cap = cs.csaw_sample_capacity(bias, list(cfg.fanout), cfg.depth, n)
        bufs = [torch.empty(n + 1, dtype=torch.int64, device=dev), torch.empty(cap, dtype=torch.int32, device=dev),
                torch.empty(cap, dtype=torch.int32, device=dev), torch.empty(cap, dtype=torch.uint8, device=dev)]
        last = {}

        def step(seed):
            nonlocal bufs, cap
            try:
                r = cs.csaw_sample(G, bias, seeds, fanout=list(cfg.fanout), depth=cfg.depth, instance_base=base,
                                   rng_seed=seed, out=bufs, stream=stream)
            except cs.CsawError as e:
                if e.status != 5:
                    raise
                cap = int(cap * 2)
                bufs = [bufs[0]] + [torch.empty(cap, dtype=t.dtype, device=dev) for t in bufs[1:]]
                r = cs.csaw_sample(G, bias, seeds, fanout=list(cfg.fanout), depth=cfg.depth, instance_base=base,
                                   rng_seed=seed, out=bufs, stream=stream)
            last["r"] = r
            return int(r[1].numel())

    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.15)
    for i in range(max(args.warmup, 0)):       # the timed sequence exactly (flush, step, stats read)
        flush.fill_(1)
        w0 = torch.cuda.Event(enable_timing=True)
        w1 = torch.cuda.Event(enable_timing=True)
        w0.record(stream)
        torch.cuda.nvtx.range_push("csaw_warmup")
        step(rng_seeds[i % len(rng_seeds)])
        torch.cuda.nvtx.range_pop()
        w1.record(stream)
        cs.csaw_stats(G)
    torch.cuda.synchronize(dev)

    # ---------------- timed region (device-resident inputs)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.lines.clear()
    evs = []
    edges = 0
    launches = 0
    hot_ms, hot_launches = 0.0, 0
    kbytes = 0
    h2d_bytes, transfer_ms = 0, 0.0
    st_last = None
    for i in range(args.steps):
        flush.fill_(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        torch.cuda.nvtx.range_push("csaw_step")   # ncu: --nvtx --nvtx-include csaw_step/
        edges += step(rng_seeds[i % len(rng_seeds)])
        torch.cuda.nvtx.range_pop()
        e1.record(stream)
        evs.append((e0, e1))
        st = cs.csaw_stats(G)
        st_last = st
        launches += st["kernel_launches"]
        hot_ms += st["hot_kernel_ms"]
        hot_launches += st["hot_launches"]
        kbytes += st["index_bytes"]
        h2d_bytes += st["h2d_bytes"]
        transfer_ms += st["transfer_ms"]
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        e = torch.tensor([edges], dtype=torch.int64, device=dev)
        dist.all_reduce(e, op=dist.ReduceOp.SUM)
        edges_all = int(e.item())
    else:
        edges_all = edges
    value = edges_all / (total_ms / 1000.0)
    steps_per_seed = {s: sum(1 for i in range(args.steps) if rng_seeds[i % len(rng_seeds)] == s) for s in rng_seeds}

    # ---------------- §8(d) algorithmic bytes of the timed launches (from the outputs, untimed re-runs)
    alg_bytes, model = 0, "oom_host"
    if not oom:
        cached = bool(ginfo.get("ctps_cache")) or (cfg.bias == "weight" and bool(ginfo.get("walk_buckets", 0) & 2))
        for s, k in steps_per_seed.items():
            if k == 0:
                continue
            step(s)
            torch.cuda.synchronize(dev)
            if kind == "walk" and ginfo.get("node2vec_index") and cfg.workload == "node2vec":
                b, model = cs.csaw_stats(G)["index_bytes"], "node2vec_index"
            elif kind == "walk":
                b, model = walk_alg_bytes(cfg, deg, out_dev, cached, bool(ginfo.get("edge_bias")))
            else:
                b, model = sample_alg_bytes(cfg, deg, seeds, *last["r"], cached=cached)
            alg_bytes += b * k

    # ---------------- optional NCCL gather of the sampled outputs (not on the SEPS clock, G31)
    gather_ms = None
    if args.gather and world > 1:
        from paper_2009_09103_b200 import dist as cdist
        t0 = time.perf_counter()
        if kind == "walk":
            cdist.gather_walks(out_dev)
        else:
            cdist.gather_samples(*last["r"])
        torch.cuda.synchronize(dev)
        gather_ms = 1000 * (time.perf_counter() - t0)

    # ---------------- OOM configs: measured host-link peak + the zero-copy variant (NEXT-4)
    store_dev = None
    if oom and args.oom_store == "peer":
        ndev = torch.cuda.device_count()
        store_dev = (local + 1) % ndev if ndev > 1 else local
    h2d_peak = measure_h2d_peak(dev, store=store_dev) if oom else None
    zc = None
    if oom and not args.no_zerocopy and args.oom_variant != "zerocopy":
        zc = run_zerocopy(cs, g, cfg, bias, seeds, base, rng_seeds[0], kind, n, dev, local, stream, flush,
                          out_dev if kind == "walk" else None, last.get("r"), G, args)

    # ---------------- the config's per-step scan path (no caches), reported apart
    scan_path = None
    if args.scan_path_steps > 0 and not oom and not args.no_cache and rank == 0:
        scan_path = run_scan_path(cs, g, cfg, deg, seeds, base, rng_seeds, n, dev, local, stream, flush, args,
                                  wts if cfg.bias == "weight" else None)

    # ---------------- end-to-end through the C ABI with host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(cs, G, bias, seeds, cfg, base, rng_seeds, args, kind, n, dev, world, flush, oom)

    # ---------------- roofline of the hot kernel
    peaks = load_peaks()
    hot_avg_ms = hot_ms / max(hot_launches, 1)
    variant = cfg.name + ("_inmem" if cfg.oom_budget_bytes and args.in_memory else "")
    if not oom and not ginfo.get("ctps_cache") and cfg.bias in ("degree", "layer"):
        variant += "_stream" if ginfo.get("edge_bias") else "_scan"
    if cfg.workload == "node2vec" and not ginfo.get("node2vec_tri") and not ginfo.get("node2vec_index"):
        variant += "_merge"
    kname = hot_kernel_name(cfg, bool(ginfo.get("node2vec_tri") if cfg.workload == "node2vec" else ginfo.get("ctps_cache")),
                            oom and args.oom_variant != "zerocopy", int(ginfo.get("walk_index_leaf") or 0),
                            int(ginfo.get("walk_index_group") or 0), bool(ginfo.get("walk_index_heads")),
                            bool(ginfo.get("node2vec_index")), bool(ginfo.get("edge_bias")),
                            buckets=bool(ginfo.get("walk_buckets", 0) & (2 if cfg.bias == "weight" else 1)))
    ncu = load_ncu(variant, kname)
    if oom:
        ach = (h2d_bytes / (total_ms / 1000.0) / 1e9) if h2d_bytes else None
        roof = {"bound": "host-link" if store_dev is None else ("nvlink" if store_dev != local else "d2d-standin"),
                "achieved": ach, "peak": h2d_peak, "unit": "GB/s",
                "frac": (ach / h2d_peak) if ach and h2d_peak else None, "traffic": None,
                "kernel": kname, "bytes_model": BYTES_MODEL["oom_host"],
                "h2d_bytes_per_step": h2d_bytes / max(args.steps, 1),
                "transfer_ms_per_step": transfer_ms / max(args.steps, 1),
                "peak_source": ("pinned cudaMemcpyAsync H2D, 1 GiB, best of 5, measured in this run"
                                if store_dev is None else
                                f"cudaMemcpyAsync cuda:{store_dev} -> cuda:{local}, 1 GiB, best of 5, measured in this run"
                                + (" (same-device stand-in: one GPU)" if store_dev == local else " (NVLink)")),
                "host_link_peak_gbs": h2d_peak if store_dev is None else None,
                "store": "host" if store_dev is None else f"cuda:{store_dev}" + (" (stand-in)" if store_dev == local else "")}
    else:
        bytes_per_launch = alg_bytes / max(hot_launches, 1)
        achieved = bytes_per_launch / (hot_avg_ms / 1000.0) / 1e9 if hot_avg_ms > 0 else None
        peak = peaks.get("hbm_gbs", 7672.0)
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None,
                "traffic": ncu.get("dram_bytes_per_launch"),
                "f_dram": ncu.get("f_dram"), "l2_sector_eff": ncu.get("l2_sector_eff"),
                "ncu_round": ncu.get("round"),
                "kernel": kname, "bytes_model": BYTES_MODEL[model], "alg_bytes_per_launch": bytes_per_launch,
                "kernel_requested_bytes_per_launch": (kbytes / max(hot_launches, 1)) if kbytes else None,
                "hot_ms_per_launch": hot_avg_ms, "hot_share_of_step": (hot_ms / total_ms) if total_ms else None,
                **random_gather_context(achieved, ncu.get("dram_bytes_per_launch"), hot_avg_ms),
                "peak_source": ("MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)" if "hbm_gbs" in peaks
                                else "fallback: B200_PROFILING.md")}

    # ---------------- oracle CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import oracle as O
            O.build()
            og = O.Graph.from_torch(g, edge_weights(g, cfg.graph_seed) if cfg.bias == "weight" else None)
            sv = seeds.cpu().numpy()
            sv = sv.view(np.uint32) if sv.dtype == np.int32 else sv.astype(np.uint32)
            v, cores, sample, _, _ = oracle_timed_sample(cfg, og, sv, base, rng_seeds[0], args.cpu_seconds)
            cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample}
        except Exception as ex:  # report, never hide
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle", "sample": f"failed: {ex}"}

    if rank == 0:
        ms_step = total_ms / max(args.steps, 1)
        build_ms = float(ginfo.get("cache_build_ms") or 0.0)
        eps = edges_all / max(args.steps, 1)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": args.scaling, "vs_baseline": None, "dtype": "u32",
                "data": "synthetic (seeded R-MAT + seeds from synth/; no datasets)",
                "config": config_block(cfg, world, gstats, args.scaling, n_total,
                                       oom_mode=(args.oom_variant if oom else None), colc=ginfo.get("device_bytes")),
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
                "detail": {"edges_per_step": eps, "edges_per_step_rank0": edges / max(args.steps, 1),
                           "step_ms": step_ms, "rng_seeds": rng_seeds, "graph_gen_s": gen_s, "gather_ms": gather_ms,
                           "cache": {"ctps_cache": bool(ginfo.get("ctps_cache")),
                                     "node2vec_tri": bool(ginfo.get("node2vec_tri")),
                                     "node2vec_index": bool(ginfo.get("node2vec_index")),
                                     "graph_device_bytes": ginfo.get("device_bytes"),
                                     "build_ms": build_ms,
                                     "one_call_seps": eps / ((ms_step + build_ms) / 1000.0),
                                     "calls_to_amortise_build": (build_ms / ms_step) if ms_step else None,
                                     "note": "one_call_seps = edges of one step / (step time + the graph's cache "
                                             "build, P:784-786 computes its cache during sampling)"},
                           "scan_path": scan_path,
                           "oom": bool(ginfo.get("oom_mode")),
                           "partition_loads_per_step": st_last["partition_loads"] if st_last else None,
                           "oom_zerocopy": zc,
                           "neighbours_scanned_per_step": st_last["neighbours_scanned"] if st_last else None,
                           "pools_per_step": st_last["pools"] if st_last else None}}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    G.close()
    return 0


def run_scan_path(cs, g, cfg, deg, seeds, base, rng_seeds, n, dev, local, stream, flush, args, wts=None):
    """detail.scan_path: the same workload through the per-step scan path -- no CTPS cache, no
    walk index, no node2vec index: every step evaluates its pool's biases and scans them
    (the north star's literal hot path, §4.1).  Degree walks stream the materialised per-edge
    bias (CSAW_GRAPH_EDGE_BIAS) unless --gather-bias.  Timed like `value` (L2 flushed before
    each step, CUDA events on the launching stream)."""
    try:
        eb = cfg.workload == "walk" and cfg.bias == "degree" and not args.gather_bias
        Gs = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=local, edge_bias=eb, weights=wts)
        info = Gs.info()
        bias = bias_of(cs, cfg)
        kind = workload_of(cfg)
        if kind == "walk":
            shape = (n, cfg.length, 2) if cfg.workload == "mdrw" else (n, cfg.length + 1)
            out = torch.empty(shape, dtype=torch.int32, device=dev)
            res = {}

            def sstep(seed):
                cs.csaw_walk(Gs, bias, seeds, cfg.length, instance_base=base, rng_seed=seed, out=out, stream=stream)
                return n * cfg.length
        else:
            res = {}
            out = None

            def sstep(seed):
                res["r"] = cs.csaw_sample(Gs, bias, seeds, fanout=list(cfg.fanout), depth=cfg.depth,
                                          instance_base=base, rng_seed=seed, stream=stream)
                return int(res["r"][1].numel())
        sstep(rng_seeds[0])            # warm-up
        torch.cuda.synchronize(dev)
        ts, edges, hot, hl = [], 0, 0.0, 0
        for i in range(args.scan_path_steps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            edges += sstep(rng_seeds[i % len(rng_seeds)])
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ts.append(e0.elapsed_time(e1))
            st = cs.csaw_stats(Gs)
            hot += st["hot_kernel_ms"]
            hl += st["hot_launches"]
        if kind == "walk":
            b, model = walk_alg_bytes(cfg, deg, out, False, eb)
        else:
            b, model = sample_alg_bytes(cfg, deg, seeds, *res["r"])
        peak = load_peaks().get("hbm_gbs", 7672.0)
        hot_avg = hot / max(hl, 1)
        ach = b / (hot_avg / 1000.0) / 1e9 if hot_avg > 0 else None
        kname = hot_kernel_name(cfg, False, False, 0, 0, False, False, eb)
        Gs.close()
        del out, res
        torch.cuda.empty_cache()
        return {"kernel": kname, "ms_per_step": sum(ts) / len(ts), "value": edges / (sum(ts) / 1000.0), "unit": UNIT,
                "steps": len(ts), "alg_bytes_per_launch": b, "bytes_model": BYTES_MODEL[model],
                "achieved_gbs": ach, "frac": (ach / peak) if ach else None, "hot_ms_per_launch": hot_avg,
                "edge_bias": bool(info.get("edge_bias")),
                "what": "per-step bias evaluation + warp-scan CTPS + ITS (no static-bias cache / index)"}
    except Exception as ex:  # report, never hide
        return {"error": str(ex)}


def run_zerocopy(cs, g, cfg, bias, seeds, base, seed, kind, n, dev, local, stream, flush, out_ref, r_ref, G, args):
    """cfg5: the zero-copy OOM variant under the same budget, reported apart (NEXT-4)."""
    try:
        Gz = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=local, budget_bytes=cfg.oom_budget_bytes,
                                  num_partitions=cfg.oom_partitions, max_resident=1, zerocopy=True)
        if kind == "walk":
            outz = torch.empty(out_ref.shape, dtype=torch.int32, device=dev)

            def zstep():
                cs.csaw_walk(Gz, bias, seeds, cfg.length, instance_base=base, rng_seed=seed, out=outz, stream=stream)
                return n * cfg.length

            def zsame():
                cs.csaw_walk(G, bias, seeds, cfg.length, instance_base=base, rng_seed=seed, out=out_ref, stream=stream)
                return bool(torch.equal(outz, out_ref))
        else:
            zr = []

            def zstep():
                zr[:] = cs.csaw_sample(Gz, bias, seeds, fanout=list(cfg.fanout), depth=cfg.depth,
                                       instance_base=base, rng_seed=seed, stream=stream)
                return int(zr[1].numel())

            def zsame():
                ref = cs.csaw_sample(G, bias, seeds, fanout=list(cfg.fanout), depth=cfg.depth, instance_base=base,
                                     rng_seed=seed, stream=stream)
                return all(bool(torch.equal(a, b)) for a, b in zip(ref, zr))
        zstep()
        torch.cuda.synchronize(dev)
        zt, ze, zh = [], 0, 0
        for _ in range(max(1, args.steps)):
            flush.fill_(1)
            z0 = torch.cuda.Event(enable_timing=True)
            z1 = torch.cuda.Event(enable_timing=True)
            z0.record(stream)
            ze += zstep()
            z1.record(stream)
            torch.cuda.synchronize(dev)
            zt.append(z0.elapsed_time(z1))
            zh += cs.csaw_stats(Gz)["h2d_bytes"]
        res = {"value": ze / (sum(zt) / 1000.0), "unit": UNIT, "ms_per_step": sum(zt) / len(zt),
               "device_bytes": Gz.info()["device_bytes"], "h2d_bytes_per_step": zh / len(zt),
               "identical_to_partitioned": zsame(),
               "what": "OOM zero-copy: col_idx prefix resident, the rest read in place from pinned host memory, "
                       "same 8 GB budget (NEXT-4)"}
        Gz.close()
        return res
    except Exception as ex:
        return {"error": str(ex)}


def run_e2e(cs, G, bias, seeds, cfg, base, rng_seeds, args, kind, n, dev, world, flush, oom):
    """Same metric through the C ABI with pinned HOST buffers: the library copies the
    step's seeds host->device and writes the step's result into host memory inside the
    call.  Timed like `value`: L2 flushed before every step, same step count (OOM
    partition mode: at most 2 steps), host wall clock around the synchronous call."""
    seeds_h = seeds.cpu().pin_memory()
    steps = max(1, min(args.steps, 2) if oom else args.steps)
    times = []
    edges = 0
    if kind == "walk":
        shape = (n, cfg.length, 2) if cfg.workload == "mdrw" else (n, cfg.length + 1)
        out_h = torch.empty(shape, dtype=torch.int32).pin_memory()
        cs.csaw_walk(G, bias, seeds_h, cfg.length, instance_base=base, rng_seed=rng_seeds[0], out=out_h)
        for i in range(steps):
            flush.fill_(1)
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            cs.csaw_walk(G, bias, seeds_h, cfg.length, instance_base=base, rng_seed=rng_seeds[i % len(rng_seeds)],
                         out=out_h)
            times.append(time.perf_counter() - t0)
            edges += n * cfg.length
        h2d = seeds_h.numel() * 4
        d2h = out_h.numel() * 4
    else:
        cap = cs.csaw_sample_capacity(bias, list(cfg.fanout), cfg.depth, n) * 2
        out_h = [torch.empty(n + 1, dtype=torch.int64).pin_memory(), torch.empty(cap, dtype=torch.int32).pin_memory(),
                 torch.empty(cap, dtype=torch.int32).pin_memory(), torch.empty(cap, dtype=torch.uint8).pin_memory()]
        r = cs.csaw_sample(G, bias, seeds_h, fanout=list(cfg.fanout), depth=cfg.depth, instance_base=base,
                           rng_seed=rng_seeds[0], out=out_h)
        m = 0
        for i in range(steps):
            flush.fill_(1)
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            r = cs.csaw_sample(G, bias, seeds_h, fanout=list(cfg.fanout), depth=cfg.depth, instance_base=base,
                               rng_seed=rng_seeds[i % len(rng_seeds)], out=out_h)
            times.append(time.perf_counter() - t0)
            edges += r[1].numel()
            m += r[1].numel()
        h2d = seeds_h.numel() * 4
        d2h = (n + 1) * 8 + (m / steps) * 9
    t = sum(times)
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ee = torch.tensor([edges], dtype=torch.int64, device=dev)
        dist.all_reduce(ee, op=dist.ReduceOp.SUM)
        t, edges = float(tt.item()), int(ee.item())
    return {"value": edges / t, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "steps": steps, "timing": "host wall clock around the synchronous C-ABI call, L2 flushed before each "
                                      "step (max over ranks)"}


def hot_kernel_name(cfg, cached=False, oom=False, wix_leaf=0, wix_group=0, heads=False, n2x=False, eb=False,
                    buckets=False):
    if cfg.workload == "walk":
        if cfg.bias == "weight":
            return "k_walk_gbw" if buckets else "k_walk_vscan<float>"
        if cfg.bias == "degree" and not cached and eb:
            return "k_walk_vscan<uint32>"
        if cfg.bias == "degree" and cached and buckets:
            return "k_walk_gb"
        if cfg.bias == "degree" and wix_leaf and heads and wix_group == 32:
            return f"k_walk_head<{wix_leaf}>"
        if cfg.bias == "degree" and wix_leaf:
            return f"k_walk_wix<{wix_leaf}>" if wix_group == 32 else f"k_walk_wixg<{wix_group}, {wix_leaf}>"
        return "k_walk_cached" if (cfg.bias == "degree" and cached) else f"k_walk<{cfg.bias}>"
    if cfg.workload == "mdrw":
        return "k_mdrw_oom_part" if oom else ("k_mdrw_fast" if cfg.pool_size <= 2048 else "k_mdrw")
    if cfg.workload == "node2vec":
        if n2x:
            return "k_node2vec_tma"
        return "k_node2vec_tri" if cached else "k_node2vec<int>"
    if oom:
        return "k_ns_select<1>" if cfg.bias == "degree" else "k_ns_select<0>"
    mode = {"neighbor": 2 if cached else 1, "forest_fire": 3, "layer": 5 if cached else 4}[cfg.workload]
    if cfg.workload == "neighbor" and cfg.bias == "uniform":
        mode = 0
    return f"k_sample_fused<{mode}>"


def random_gather_context(achieved, traffic=None, hot_ms=None) -> dict:
    """The measured random-access ceiling (profiles/random_gather_peaks.json, scripts/random_roofline.cu):
    64 B records at uniformly random offsets of a 64 GiB buffer -- the access pattern of the pointer-chasing
    walk kernels -- reach ~0.95 TB/s of requested bytes, far below the streaming copy peak.  Context for
    `frac` (which stays against the copy peak): a dependent-gather kernel near this figure is at its
    practical roofline."""
    try:
        with open(os.path.join(ROOT, "profiles", "random_gather_peaks.json")) as f:
            pk = json.load(f)
        rg = pk["by_footprint_gib"]["64"]["64B"]
        line = pk.get("random_line", {}).get("dram_gbs")
    except Exception:
        return {}
    out = {"random_gather_peak_gbs": rg, "frac_of_random_gather_peak": (achieved / rg) if achieved else None}
    if line:
        # the kernel's DRAM traffic (ncu) against the measured random-line ceiling: every random read moves a
        # 128 B line, ~34 G lines/s = 4.35 TB/s (profiles/random_gather_peaks.json "random_line")
        dram = traffic / (hot_ms / 1000.0) / 1e9 if traffic and hot_ms else None
        out.update({"random_line_ceiling_gbs": line, "dram_gbs_ncu": dram,
                    "dram_frac_of_random_line_ceiling": (dram / line) if dram else None})
    return out


def load_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def load_ncu(cfg_name, kernel) -> dict:
    """DRAM bytes per launch, f_dram and L2 sector efficiency of the hot kernel from the
    committed ncu --set full capture summary (profiles/ncu_traffic.json, written by
    scripts/ncu_summary.py); {} unless the capture is of the same kernel."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        v = d.get(cfg_name)
        if not isinstance(v, dict):
            return {}
        norm = lambda k: k.replace("void ", "").replace("csaw::", "").replace(" ", "")
        a, b = norm(v.get("kernel", "")), norm(kernel)
        if a.split("<")[0] != b.split("<")[0] or ("<" in a and "<" in b and a != b):
            return {}
        return v
    except Exception:
        return {}


if __name__ == "__main__":
    sys.exit(main())
