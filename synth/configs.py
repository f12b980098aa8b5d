"""The five BASELINE.json configs as concrete synthetic workloads.

Workload parameters follow PAPER.md §6 "Test Setup" (lines 972-974):
NeighborSize = Depth = 2 for sampling, forest fire P_f = 0.7, walk length
2,000, MDRW FrontierSize (pool) 2,000; graph shapes follow Table 2 (lines
945-955; FR/TW edge counts read as billions, reading R13).
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace


@dataclass(frozen=True)
class WorkloadConfig:
    name: str
    graph_vertices: int
    graph_entries: int          # target CSR entries (directed, after symmetrisation)
    graph_seed: int
    workload: str               # "neighbor" | "walk" | "node2vec" | "layer" | "forest_fire" | "mdrw"
    bias: str                   # "degree" | "uniform" | "node2vec" | "layer" | "forest_fire" | "mdrw"
    n_instances: int            # instances / walkers (0 = one walker per non-isolated vertex)
    fanout: tuple = ()
    depth: int = 0
    length: int = 0
    p: float = 1.0
    q: float = 1.0
    pf: float = 0.0
    pool_size: int = 0
    oom_budget_bytes: int = 0
    oom_partitions: int = 0
    oom_resident: int = 0
    description: str = ""


CONFIGS = {
    "cfg1": WorkloadConfig(
        "cfg1", 1024, 16384, 1, "neighbor", "degree", 64, fanout=(2, 2), depth=2,
        description="degree-biased neighbor sampling, 2 hops, fanout 2, 64 instances, R-MAT 1,024 V / 16K E"),
    "cfg2": WorkloadConfig(
        "cfg2", 4_800_000, 69_000_000, 2, "walk", "degree", 4000, length=2000,
        description="degree-biased random walk, length 2,000, 4,000 walkers, LJ-shaped R-MAT 4.8M V / 69M E"),
    "cfg3": WorkloadConfig(
        "cfg3", 3_000_000, 117_000_000, 3, "node2vec", "node2vec", 0, length=80, p=2.0, q=0.5,
        description="node2vec p=2 q=0.5, length 80, one walker per non-isolated vertex, OR-shaped R-MAT 3M V / 117M E"),
    "cfg4_layer": WorkloadConfig(
        "cfg4_layer", 41_600_000, 1_470_000_000, 4, "layer", "layer", 8192, fanout=(2, 2), depth=2,
        description="layer sampling fanout 2/layer, depth 2, 8,192 instances, TW-shaped R-MAT 41.6M V / 1.47B E"),
    "cfg4_ff": WorkloadConfig(
        "cfg4_ff", 41_600_000, 1_470_000_000, 4, "forest_fire", "forest_fire", 8192, depth=2, pf=0.7,
        description="forest fire pf=0.7, depth 2, 8,192 instances, TW-shaped R-MAT 41.6M V / 1.47B E"),
    "cfg5": WorkloadConfig(
        "cfg5", 65_600_000, 1_800_000_000, 5, "mdrw", "mdrw", 4000, length=2000, pool_size=2000,
        oom_budget_bytes=8_000_000_000, oom_partitions=4, oom_resident=2,
        description="MDRW pool 2,000, 2,000 steps, 4,000 instances, FR-shaped R-MAT 65.6M V / 1.8B E, OOM 8 GB budget"),
    # the float path (R28/R32) at config-2 scale: the same LJ-shaped graph with seeded fp32 edge
    # weights (synth/weights.py) and EdgeBias = w(e) -- not a BASELINE config, a measurement of
    # the per-step weight scan
    "cfg2_weight": WorkloadConfig(
        "cfg2_weight", 4_800_000, 69_000_000, 2, "walk", "weight", 4000, length=2000,
        description="edge-weight walk (EdgeBias = w(e), fp32 weights summed in fp64), length 2,000, 4,000 walkers, "
                    "LJ-shaped R-MAT 4.8M V / 69M E with seeded weights"),
    # config 5's second half: batched multi-instance traversal sampling under the same budget (§5.2-5.3)
    "cfg5_ns": WorkloadConfig(
        "cfg5_ns", 65_600_000, 1_800_000_000, 5, "neighbor", "degree", 8192, fanout=(2, 2), depth=2,
        oom_budget_bytes=8_000_000_000, oom_partitions=4, oom_resident=2,
        description="degree-biased neighbor sampling fanout 2, depth 2, 8,192 instances, batched, "
                    "FR-shaped R-MAT 65.6M V / 1.8B E, OOM 8 GB budget"),
}


def small_config(name: str, vertices: int, entries: int, **over) -> WorkloadConfig:
    """Same workload as CONFIGS[name] on a smaller graph (parity-test sizes)."""
    return replace(CONFIGS[name], graph_vertices=vertices, graph_entries=entries, **over)
