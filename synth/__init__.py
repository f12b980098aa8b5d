"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This package holds ONLY input generation (graphs, seed vertices, workload
parameters).  It contains none of C-SAW's selection arithmetic: no Philox, no
CTPS, no inverse-transform search, no bipartite region search.  Both sides of a
parity test receive the same bytes from here and nothing else in common.

The randomness used to *build* inputs is a 32-bit integer hash (lowbias32-style
mix) evaluated with int64 torch ops, so the same seed gives bit-identical graphs
on CPU and on a CUDA device.  The sampler's own random numbers (Philox4x32-10)
are implemented separately in `oracle/` and in the CUDA library.
"""
from .rmat import RmatGraph, rmat_csr, gtoy_csr, degree_stats
from .seeds import instance_seeds, nonisolated_vertices, mdrw_seeds
from .configs import CONFIGS, WorkloadConfig, small_config
from .weights import edge_weights

__all__ = [
    "RmatGraph", "rmat_csr", "gtoy_csr", "degree_stats",
    "instance_seeds", "nonisolated_vertices", "mdrw_seeds",
    "CONFIGS", "WorkloadConfig", "small_config", "edge_weights",
]
