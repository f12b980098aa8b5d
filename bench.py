#!/usr/bin/env python
"""bench.py — C-SAW hot path on B200: sampled edges per second (SEPS) + roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]

A "step" is one pass of the whole hot path over one batch: for the default
config (cfg2, BASELINE.json configs[1]) every walker of the 4,000-walker,
2,000-step degree-biased random walk on the LJ-shaped R-MAT graph.  Inputs are
synthetic (synth/, seeded), resident in HBM when the timed region starts; L2 is
flushed (256 MB write) before every timed step, and each step is timed with
CUDA events on the launching stream.  Multi-GPU: one process per GPU
(torchrun), weak scaling (each rank runs the config's workload on its own
disjoint instance-id range), max-over-ranks time, NCCL used only for the
optional output gather after timing.  The oracle (oracle/) is executed only by
the cpu_baseline leg and by --impl reference.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from synth import CONFIGS, degree_stats, instance_seeds, mdrw_seeds, nonisolated_vertices, rmat_csr  # noqa: E402

METRIC = "sampled edges/sec (SEPS) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "sampled_edges/s"
L2_FLUSH_BYTES = 256 << 20


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rng-seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="oracle CPU-baseline budget (wall s)")
    ap.add_argument("--gather", action="store_true", help="NCCL-gather outputs after timing (reported apart)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--in-memory", action="store_true", help="cfg5: ignore the OOM budget (in-memory MDRW)")
    ap.add_argument("--no-cache", action="store_true",
                    help="disable the static-bias CTPS cache / node2vec triangle counts (scan every pool)")
    ap.add_argument("--no-zerocopy", action="store_true", help="cfg5: skip the zero-copy OOM variant")
    ap.add_argument("--oom-budget-gb", type=float, default=0.0,
                    help="OOM configs: override the device budget (GiB) -- experiments only, the config names 8 GB")
    ap.add_argument("--oom-variant", default="partition", choices=["partition", "zerocopy"],
                    help="OOM configs: time the paper's partition scheduling (default) or the zero-copy mode "
                         "(col_idx prefix resident within the budget, the rest read in place from pinned host memory)")
    return ap.parse_args()


# ------------------------------------------------------------------ workload description
def workload_of(cfg):
    """(kind, bias name, csaw entry) for a config."""
    return {"walk": "walk", "node2vec": "walk", "mdrw": "walk",
            "neighbor": "sample", "layer": "sample", "forest_fire": "sample"}[cfg.workload]


def make_graph(cfg, device):
    t0 = time.perf_counter()
    g = rmat_csr(cfg.graph_vertices, cfg.graph_entries, cfg.graph_seed, device=device)
    torch.cuda.synchronize(device) if device.type == "cuda" else None
    return g, time.perf_counter() - t0


def make_seeds(cfg, g, rank, world):
    """This rank's instance ids [base, base+n) and seeds (weak scaling: n per rank)."""
    if cfg.workload == "node2vec":
        verts = nonisolated_vertices(g)
        n = verts.numel() if cfg.n_instances == 0 else cfg.n_instances
        return rank * n, verts[:n].to(torch.int32)
    n = cfg.n_instances
    if cfg.workload == "mdrw":
        s = mdrw_seeds(g, n * world, cfg.pool_size)
        return rank * n, s[rank * n:(rank + 1) * n].contiguous()
    s = instance_seeds(g, n * world)
    return rank * n, s[rank * n:(rank + 1) * n].contiguous()


def bias_of(cs, cfg):
    return {"walk": cs.make_bias(cfg.bias), "node2vec": cs.make_bias("node2vec", p=cfg.p, q=cfg.q),
            "mdrw": cs.make_bias("mdrw", pool_size=cfg.pool_size), "neighbor": cs.make_bias(cfg.bias),
            "layer": cs.make_bias("layer"), "forest_fire": cs.make_bias("forest_fire", pf=cfg.pf)}[cfg.workload]


def algorithmic_bytes(cfg, st, n, edges):
    """Bytes the method must move (element granularity), DESIGN.md §6:
    degree pool: 16 (row_ptr pair) + 8 d (col + deg) per pool, + output;
    uniform: 16 + 4 per step; node2vec: 16 + 4 d(v) + 4 d(prev); MDRW: 32 per step;
    sampling select kernel: 16 per pool + 8 per scanned candidate + 12 per staged edge."""
    scanned, pools = st["neighbours_scanned"], st["pools"]
    probes = st.get("cache_probes", 0)
    if st.get("index_bytes") and cfg.workload in ("walk", "node2vec"):
        # bytes the kernel read, counted in the kernel (narrow walk index: record + nodes + leaf
        # and col entries; node2vec with triangle counts: row_ptr pairs, tri, list entries), + path
        return st["index_bytes"] + 4 * n * (cfg.length + 1) + 4 * n
    if probes and cfg.workload == "walk":
        # cached CTPS: row_ptr pair 16 + T 8 + col 4 per step, 8 per cache probe, + path
        return 28 * pools + 8 * probes + 4 * n * (cfg.length + 1) + 4 * n
    if probes:
        return 24 * pools + 8 * probes + 12 * edges
    if cfg.workload == "walk":
        out = 4 * n * (cfg.length + 1) + 4 * n
        if cfg.bias == "degree":
            return 16 * pools + 8 * scanned + out
        return 20 * pools + out
    if cfg.workload == "node2vec":
        return 16 * pools + 8 * scanned + 4 * n * (cfg.length + 1) + 4 * n
    if cfg.workload == "mdrw":
        return 32 * n * cfg.length + 16 * n * cfg.pool_size
    if cfg.workload == "forest_fire":
        return 16 * pools + 16 * edges
    return 16 * pools + 8 * scanned + 12 * edges


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
        if cfg.workload == "walk":
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
    # calibrate single-instance cost
    t0 = time.perf_counter()
    _oracle_job((cfg.name, 0, 1, base, seeds_np[:1], rng_seed))
    t1 = max(time.perf_counter() - t0, 1e-4)
    per_worker = max(1, int(budget_s / t1))
    m = int(min(n, per_worker * workers))
    m = max(m, min(n, workers))
    # tiny workloads (e.g. cfg1): repeat whole passes so the sample is ~budget_s of CPU work
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
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    import oracle as O
    O.build()
    dev = torch.device("cuda:0") if torch.cuda.is_available() else torch.device("cpu")
    g, _ = make_graph(cfg, dev)
    base, seeds = make_seeds(cfg, g, 0, 1)
    og = O.Graph.from_torch(g)
    seeds_np = seeds.cpu().numpy().view(np.uint32)
    del g
    if dev.type == "cuda":
        torch.cuda.empty_cache()
    per_step = max(2.0, 120.0 / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        oracle_timed_sample(cfg, og, seeds_np, base, args.rng_seed, min(per_step, 3.0))
    vals, walls, samples = [], [], []
    for _ in range(args.steps):
        v, cores, sample, edges, wall = oracle_timed_sample(cfg, og, seeds_np, base, args.rng_seed, per_step)
        vals.append(v)
        walls.append(wall)
        samples.append(sample)
    value = statistics.mean(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * statistics.mean(walls),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (seeded R-MAT, synth/)",
            "config": config_block(cfg, 1, None),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": samples[-1]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def config_block(cfg, world, stats_g, oom_mode=None, colc=None):
    c = {"workload": f"{cfg.name}: {cfg.description}", "instances_per_gpu": cfg.n_instances or "all non-isolated",
         "graph": {"V": cfg.graph_vertices, "E_target": cfg.graph_entries, "generator": "R-MAT Graph500 (0.57,0.19,0.19,0.05), symmetrised, dedup"},
         "parallelism": f"instances sharded over {world} GPU(s), CSR replicated",
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


# ------------------------------------------------------------------ our arm
def main():
    args = parse_args()
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
        cfg = dataclasses.replace(cfg, oom_budget_bytes=int(args.oom_budget_gb * (1 << 30)))
    kind = workload_of(cfg)

    g, gen_s = make_graph(cfg, dev)
    gstats = degree_stats(g)
    base, seeds = make_seeds(cfg, g, rank, world)
    seeds = seeds.to(dev).contiguous()
    n = seeds.shape[0]
    oom = cfg.oom_budget_bytes > 0 and not args.in_memory
    if oom:
        # out-of-memory mode (§5): the device holds only what the imposed budget
        # allows -- move the generated graph to host memory first
        g = g.to("cpu")
        torch.cuda.empty_cache()
        zc_main = args.oom_variant == "zerocopy"
        G = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=local, budget_bytes=cfg.oom_budget_bytes,
                                 num_partitions=cfg.oom_partitions, max_resident=1 if zc_main else cfg.oom_resident,
                                 num_streams=cfg.oom_resident, zerocopy=zc_main)
    else:
        # static-bias CTPS cache (§8(f) NEXT-1, bit-identical) for degree-biased selections
        use_cache = (not args.no_cache) and cfg.bias in ("degree", "layer")
        use_tri = (not args.no_cache) and cfg.workload == "node2vec"   # node2vec edge triangle counts
        use_meta = (not args.no_cache) and cfg.workload == "mdrw"   # next-vertex metadata per entry
        G = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=local, ctps_cache=use_cache, node2vec_tri=use_tri,
                                 next_meta=use_meta, walk_index=use_cache)   # walk index + vertex heads
    ginfo = G.info()
    bias = bias_of(cs, cfg)
    stream = torch.cuda.current_stream(dev)

    # output buffers (device) for the device-resident timed region
    if kind == "walk":
        shape = (n, cfg.length, 2) if cfg.workload == "mdrw" else (n, cfg.length + 1)
        out_dev = torch.empty(shape, dtype=torch.int32, device=dev)

        def step():
            cs.csaw_walk(G, bias, seeds, cfg.length, instance_base=base, rng_seed=args.rng_seed, out=out_dev,
                         stream=stream)
            return n * cfg.length
    else:
        cap = cs.csaw_sample_capacity(bias, list(cfg.fanout), cfg.depth, n)
        bufs = [torch.empty(n + 1, dtype=torch.int64, device=dev), torch.empty(cap, dtype=torch.int32, device=dev),
                torch.empty(cap, dtype=torch.int32, device=dev), torch.empty(cap, dtype=torch.uint8, device=dev)]

        def step():
            nonlocal bufs, cap
            try:
                r = cs.csaw_sample(G, bias, seeds, fanout=list(cfg.fanout), depth=cfg.depth, instance_base=base,
                                   rng_seed=args.rng_seed, out=bufs, stream=stream)
            except cs.CsawError as e:
                if e.status != 5:
                    raise
                cap = int(cap * 2)
                bufs = [bufs[0]] + [torch.empty(cap, dtype=t.dtype, device=dev) for t in bufs[1:]]
                r = cs.csaw_sample(G, bias, seeds, fanout=list(cfg.fanout), depth=cfg.depth, instance_base=base,
                                   rng_seed=args.rng_seed, out=bufs, stream=stream)
            return int(r[1].numel())

    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    # the clock sampler starts before the warm-up, and warm-up steps are the timed steps'
    # exact sequence (flush + step), so the first timed step is not a cold-host outlier
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.15)
    for _ in range(max(args.warmup, 0)):
        flush.fill_(1)
        w0 = torch.cuda.Event(enable_timing=True)
        w1 = torch.cuda.Event(enable_timing=True)
        w0.record(stream)
        torch.cuda.nvtx.range_push("csaw_warmup")   # NVTX initialises on first use: not inside a timed step
        step()
        torch.cuda.nvtx.range_pop()
        w1.record(stream)
        cs.csaw_stats(G)
    torch.cuda.synchronize(dev)

    # ---------------- timed region (device-resident inputs)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.lines.clear()   # keep only samples taken during the timed region
    evs = []
    edges = 0
    launches = 0
    hot_ms, hot_launches = 0.0, 0
    alg_bytes = 0
    st_last = None
    for _ in range(args.steps):
        flush.fill_(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        torch.cuda.nvtx.range_push("csaw_step")   # lets ncu select the timed launches (--nvtx-include csaw_step/)
        edges += step()
        torch.cuda.nvtx.range_pop()
        e1.record(stream)
        evs.append((e0, e1))
        st = cs.csaw_stats(G)
        st_last = st
        launches += st["kernel_launches"]
        hot_ms += st["hot_kernel_ms"]
        hot_launches += st["hot_launches"]
        alg_bytes += algorithmic_bytes(cfg, st, n, st["sampled_edges"])
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

    # ---------------- optional NCCL gather of the sampled outputs (not on the SEPS clock, G31)
    gather_ms = None
    if args.gather and world > 1:
        from paper_2009_09103_b200 import dist as cdist
        t0 = time.perf_counter()
        if kind == "walk":
            cdist.gather_walks(out_dev)
        else:
            cdist.gather_samples(*r_last(cs, G, bias, seeds, cfg, base, args, stream))
        torch.cuda.synchronize(dev)
        gather_ms = 1000 * (time.perf_counter() - t0)

    # ---------------- cfg5: the B200-native zero-copy OOM variant (NEXT-4), reported apart
    zc = None
    if oom and not args.no_zerocopy and args.oom_variant != "zerocopy":
        try:
            Gz = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=local, budget_bytes=cfg.oom_budget_bytes,
                                      num_partitions=cfg.oom_partitions, max_resident=1, zerocopy=True)
            if kind == "walk":
                outz = torch.empty((n, cfg.length, 2), dtype=torch.int32, device=dev)

                def zstep():
                    cs.csaw_walk(Gz, bias, seeds, cfg.length, instance_base=base, rng_seed=args.rng_seed, out=outz,
                                 stream=stream)
                    return n * cfg.length

                def zsame():
                    return bool(torch.equal(outz, out_dev))
            else:
                zr = []

                def zstep():
                    zr[:] = cs.csaw_sample(Gz, bias, seeds, fanout=list(cfg.fanout), depth=cfg.depth,
                                           instance_base=base, rng_seed=args.rng_seed, stream=stream)
                    return int(zr[1].numel())

                def zsame():
                    ref = r_last(cs, G, bias, seeds, cfg, base, args, stream)
                    return all(bool(torch.equal(a, b)) for a, b in zip(ref, zr))
            zstep()
            torch.cuda.synchronize(dev)
            zt, ze = [], 0
            for _ in range(max(1, args.steps)):
                flush.fill_(1)
                z0 = torch.cuda.Event(enable_timing=True)
                z1 = torch.cuda.Event(enable_timing=True)
                z0.record(stream)
                ze += zstep()
                z1.record(stream)
                torch.cuda.synchronize(dev)
                zt.append(z0.elapsed_time(z1))
            zc = {"value": ze / (sum(zt) / 1000.0), "unit": UNIT, "ms_per_step": sum(zt) / len(zt),
                  "identical_to_partitioned": zsame(),
                  "what": "OOM zero-copy: col_idx read in place from pinned host memory, same 8 GB budget (NEXT-4)"}
            Gz.close()
        except Exception as ex:
            zc = {"error": str(ex)}

    # ---------------- end-to-end through the C ABI with host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(cs, G, bias, seeds, cfg, base, args, kind, n, dev, world)

    # ---------------- roofline of the hot kernel
    peaks = load_peaks()
    hot_avg_ms = hot_ms / max(hot_launches, 1)
    bytes_per_launch = alg_bytes / max(hot_launches, 1)
    achieved = bytes_per_launch / (hot_avg_ms / 1000.0) / 1e9 if hot_avg_ms > 0 else None
    peak = peaks.get("hbm_gbs", 6650.0)
    variant = cfg.name
    if cfg.oom_budget_bytes and args.in_memory:
        variant += "_inmem"
    elif not ginfo.get("ctps_cache") and cfg.bias in ("degree", "layer") and not ginfo.get("oom_mode"):
        variant += "_scan"
    kname = hot_kernel_name(cfg, bool(ginfo.get("node2vec_tri") if cfg.workload == "node2vec" else ginfo.get("ctps_cache")),
                            bool(ginfo.get("oom_mode")) and args.oom_variant != "zerocopy",
                            int(ginfo.get("walk_index_leaf") or 0), int(ginfo.get("walk_index_group") or 0),
                            bool(ginfo.get("walk_index_heads")))
    traffic = load_traffic(variant, kname)
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": (achieved / peak) if achieved else None, "traffic": traffic,
            "kernel": kname, "alg_bytes_per_launch": bytes_per_launch,
            "hot_ms_per_launch": hot_avg_ms, "hot_share_of_step": (hot_ms / total_ms) if total_ms else None,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (of measured)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s"}

    # ---------------- oracle CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import oracle as O
            O.build()
            og = O.Graph.from_torch(g)
            sv = seeds.cpu().numpy()
            sv = sv.view(np.uint32) if sv.dtype == np.int32 else sv.astype(np.uint32)
            v, cores, sample, _, _ = oracle_timed_sample(cfg, og, sv, base, args.rng_seed, args.cpu_seconds)
            cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample}
        except Exception as ex:  # report, never hide
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle", "sample": f"failed: {ex}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total_ms / max(args.steps, 1), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "u32",
                "data": "synthetic (seeded R-MAT + seeds from synth/; no datasets)",
                "config": config_block(cfg, world, gstats, oom_mode=(args.oom_variant if oom else None),
                                       colc=ginfo.get("device_bytes")), "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk,
                "detail": {"edges_per_step_per_gpu": edges / max(args.steps, 1), "step_ms": step_ms,
                           "graph_gen_s": gen_s, "gather_ms": gather_ms,
                           "ctps_cache": bool(ginfo.get("ctps_cache")), "cache_build_ms": ginfo.get("cache_build_ms"),
                           "oom": bool(ginfo.get("oom_mode")),
                           "partition_loads_per_step": st_last["partition_loads"] if st_last else None,
                           "h2d_bytes_per_step": st_last["h2d_bytes"] if st_last else None,
                           "transfer_ms_per_step": st_last["transfer_ms"] if st_last else None,
                           "host_link_gbs": (st_last["h2d_bytes"] / st_last["transfer_ms"] / 1e6)
                           if st_last and st_last["transfer_ms"] else None,
                           "cache_probes_per_step": st_last["cache_probes"] if st_last else None,
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


def r_last(cs, G, bias, seeds, cfg, base, args, stream):
    return cs.csaw_sample(G, bias, seeds, fanout=list(cfg.fanout), depth=cfg.depth, instance_base=base,
                          rng_seed=args.rng_seed, stream=stream)


def run_e2e(cs, G, bias, seeds, cfg, base, args, kind, n, dev, world):
    """Same metric through the C ABI with pinned HOST buffers: the library copies the
    step's seeds host->device and the step's result device->host inside the call."""
    seeds_h = seeds.cpu().pin_memory()
    steps = max(1, min(args.steps, 3))
    times = []
    edges = 0
    if kind == "walk":
        shape = (n, cfg.length, 2) if cfg.workload == "mdrw" else (n, cfg.length + 1)
        out_h = torch.empty(shape, dtype=torch.int32).pin_memory()
        cs.csaw_walk(G, bias, seeds_h, cfg.length, instance_base=base, rng_seed=args.rng_seed, out=out_h)
        for _ in range(steps):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            cs.csaw_walk(G, bias, seeds_h, cfg.length, instance_base=base, rng_seed=args.rng_seed, out=out_h)
            times.append(time.perf_counter() - t0)
            edges += n * cfg.length
        h2d = seeds_h.numel() * 4
        d2h = out_h.numel() * 4
    else:
        cap = cs.csaw_sample_capacity(bias, list(cfg.fanout), cfg.depth, n) * 2
        out_h = [torch.empty(n + 1, dtype=torch.int64).pin_memory(), torch.empty(cap, dtype=torch.int32).pin_memory(),
                 torch.empty(cap, dtype=torch.int32).pin_memory(), torch.empty(cap, dtype=torch.uint8).pin_memory()]
        r = cs.csaw_sample(G, bias, seeds_h, fanout=list(cfg.fanout), depth=cfg.depth, instance_base=base,
                           rng_seed=args.rng_seed, out=out_h)
        m = r[1].numel()
        for _ in range(steps):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            r = cs.csaw_sample(G, bias, seeds_h, fanout=list(cfg.fanout), depth=cfg.depth, instance_base=base,
                               rng_seed=args.rng_seed, out=out_h)
            times.append(time.perf_counter() - t0)
            edges += r[1].numel()
        h2d = seeds_h.numel() * 4
        d2h = (n + 1) * 8 + m * 9
    t = sum(times)
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ee = torch.tensor([edges], dtype=torch.int64, device=dev)
        dist.all_reduce(ee, op=dist.ReduceOp.SUM)
        t, edges = float(tt.item()), int(ee.item())
    return {"value": edges / t, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "steps": steps, "timing": "host wall clock around the synchronous C-ABI call (max over ranks)"}


def hot_kernel_name(cfg, cached=False, oom=False, wix_leaf=0, wix_group=0, heads=False):
    if cfg.workload == "walk":
        if cfg.bias == "degree" and wix_leaf and heads and wix_group == 32:
            return f"k_walk_head<{wix_leaf}>"
        if cfg.bias == "degree" and wix_leaf:
            return f"k_walk_wix<{wix_leaf}>" if wix_group == 32 else f"k_walk_wixg<{wix_group}, {wix_leaf}>"
        return "k_walk_cached" if (cfg.bias == "degree" and cached) else f"k_walk<{cfg.bias}>"
    if cfg.workload == "mdrw":
        return "k_mdrw_oom_part" if oom else ("k_mdrw_fast" if cfg.pool_size <= 2048 else "k_mdrw")
    if cfg.workload == "node2vec":
        return "k_node2vec_tri" if cached else "k_node2vec<int>"
    if oom:
        # OOM traversal sampling runs the batched level driver, one select launch per resident partition
        return "k_ns_select<1>" if cfg.bias == "degree" else "k_ns_select<0>"
    # sampling: the fused one-warp-per-instance kernel (small per-instance frontiers)
    mode = {"neighbor": 2 if cached else 1, "forest_fire": 3, "layer": 5 if cached else 4}[cfg.workload]
    if cfg.workload == "neighbor" and cfg.bias == "uniform":
        mode = 0
    return f"k_sample_fused<{mode}>"


def load_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def load_traffic(cfg_name, kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the hot kernel, from the
    committed ncu --set full capture summary (profiles/ncu_traffic.json), else null.  Only
    a capture of the same kernel counts (a stale entry for another variant is ignored)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        v = d.get(cfg_name)
        if not isinstance(v, dict):
            return None
        norm = lambda k: k.replace("void ", "").replace("csaw::", "").replace(" ", "")
        a, b = norm(v.get("kernel", "")), norm(kernel)
        # same kernel; template arguments must agree when both names carry them
        if a.split("<")[0] != b.split("<")[0] or ("<" in a and "<" in b and a != b):
            return None
        return v.get("dram_bytes_per_launch")
    except Exception:
        return None


if __name__ == "__main__":
    sys.exit(main())
