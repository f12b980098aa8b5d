"""Host logic of bench.py (no GPU): the §8(d) algorithmic-byte model computed from a
launch's output, the strong / weak instance split and the --gpus self-launch rule.
Expected byte counts are hand-computed from SURVEY.md §8(d)'s per-unit figures."""
import os

import numpy as np
import torch

import bench
from synth import CONFIGS, gtoy_csr


def _deg(rp):
    rp = torch.as_tensor(rp, dtype=torch.int64)
    return rp[1:] - rp[:-1]


def test_walk_bytes_degree_scan_cached_and_node2vec():
    # degrees: v0:3, v1:1, v2:2, v3:5
    deg = torch.tensor([3, 1, 2, 5], dtype=torch.int64)
    path = torch.tensor([[0, 1, 0, 3], [2, 0, 2, 0]], dtype=torch.int32)     # 2 walkers, 3 steps each
    # ★ scan: per step 16 + 8 d(v) + 4, v = path[:, :3] -> d = 3,1,3 and 2,3,2 -> sum d = 14
    b, m = bench.walk_alg_bytes(CONFIGS["cfg2"], deg, path, cached=False)
    assert m == "walk_degree_scan" and b == 6 * 16 + 8 * 14 + 6 * 4
    # NEXT-1: 32 (2 + ceil(log2 d)) + 4; ceil(log2 .) of 3,1,3,2,3,2 = 2,0,2,1,2,1 -> 8
    b, m = bench.walk_alg_bytes(CONFIGS["cfg2"], deg, path, cached=True)
    assert m == "walk_degree_cached" and b == 32 * (2 * 6 + 8) + 6 * 4
    # node2vec: step 0 16 + 4 + 4; later steps 16 + 4 d(v) + 4: d(v) at t=1,2 = 1,3 and 3,2 -> 9
    b, m = bench.walk_alg_bytes(CONFIGS["cfg3"], deg, path, cached=False)
    assert m == "node2vec" and b == 6 * 16 + 2 * 4 + 4 * 9 + 6 * 4
    # a walk that ended (0xFFFFFFFF padding, R20) counts the pools it evaluated: at v0 and
    # at v1 (whose step produced the end marker), none after
    path2 = torch.tensor([[0, 1, -1, -1]], dtype=torch.int32)
    b, _ = bench.walk_alg_bytes(CONFIGS["cfg2"], deg, path2, cached=False)
    assert b == 2 * 16 + 8 * (3 + 1) + 2 * 4


def test_sample_bytes_degree_and_layer():
    deg = torch.tensor([2, 4, 1, 3, 2], dtype=torch.int64)
    seeds = torch.tensor([1, 3], dtype=torch.int32)
    # instance 0 (seed 1): depth 1 -> 0, 2; depth 2 -> (0,1) back to the seed, (2,4)
    # instance 1 (seed 3): depth 1 -> 4; depth 2 -> (4,3)
    offs = torch.tensor([0, 4, 6], dtype=torch.int64)
    src = torch.tensor([1, 1, 0, 2, 3, 4], dtype=torch.int32)
    dst = torch.tensor([0, 2, 1, 4, 4, 3], dtype=torch.int32)
    dep = torch.tensor([1, 1, 2, 2, 1, 2], dtype=torch.uint8)
    cfg = CONFIGS["cfg1"]
    # expanded: level 0 seeds {1, 3} (d 4, 3); level 1: inst0 {0, 2} (d 2, 1), inst1 {4} (d 2)
    exp_d = [4, 3, 2, 1, 2]
    b, m = bench.sample_alg_bytes(cfg, deg, seeds, offs, src, dst, dep)
    assert m == "sample_degree" and b == 16 * 5 + 8 * sum(exp_d) + 9 * 6
    b, m = bench.sample_alg_bytes(CONFIGS["cfg4_layer"], deg, seeds, offs, src, dst, dep)
    assert m == "sample_layer" and b == 16 * 5 + 8 * sum(exp_d) + 9 * 6
    # forest fire: 16 per expanded vertex + 13 per edge
    b, m = bench.sample_alg_bytes(CONFIGS["cfg4_ff"], deg, seeds, offs, src, dst, dep)
    assert m == "sample_ff" and b == 16 * 5 + 13 * 6


def test_sample_bytes_visited_vertices_are_not_expanded_twice():
    deg = torch.tensor([2, 2, 2], dtype=torch.int64)
    seeds = torch.tensor([0], dtype=torch.int32)
    # depth 1: 0 -> 1 and 0 -> 1 again cannot happen (distinct picks), but 1 picked from the
    # seed and the seed itself reached at depth 1 through a self-loop-free graph: 0 -> 1, 0 -> 2
    offs = torch.tensor([0, 2], dtype=torch.int64)
    src = torch.tensor([0, 0], dtype=torch.int32)
    dst = torch.tensor([1, 2], dtype=torch.int32)
    dep = torch.tensor([1, 1], dtype=torch.uint8)
    b, _ = bench.sample_alg_bytes(CONFIGS["cfg1"], deg, seeds, offs, src, dst, dep)
    assert b == 16 * 3 + 8 * 6 + 9 * 2
    # an edge back to the seed at depth 1 does not expand the seed again
    dst2 = torch.tensor([1, 0], dtype=torch.int32)
    b, _ = bench.sample_alg_bytes(CONFIGS["cfg1"], deg, seeds, offs, src, dst2, dep)
    assert b == 16 * 2 + 8 * 4 + 9 * 2


def test_strong_split_covers_every_instance_once():
    g = gtoy_csr()
    cfg = CONFIGS["cfg1"]
    N = cfg.n_instances
    parts = [bench.make_seeds(cfg, g, r, 3, "strong") for r in range(3)]
    bases = [p[0] for p in parts]
    assert bases == [0, N // 3, 2 * N // 3] and all(p[2] == N for p in parts)
    whole = torch.cat([p[1] for p in parts])
    assert torch.equal(whole, bench.make_seeds(cfg, g, 0, 1, "strong")[1])
    w = [bench.make_seeds(cfg, g, r, 2, "weak") for r in range(2)]
    assert [x[0] for x in w] == [0, N] and all(x[1].numel() == N for x in w)


def test_self_launch_only_outside_torchrun(monkeypatch):
    args = bench.parse_args(["--gpus", "1"])
    assert bench.maybe_spawn(args) is None
    monkeypatch.setenv("WORLD_SIZE", "2")
    assert bench.maybe_spawn(bench.parse_args(["--gpus", "2"])) is None
    assert bench.parse_args([]).config == "cfg3" and bench.parse_args([]).scaling == "strong"


def test_walk_bytes_stream_model_and_scan_path_names():
    # materialised degree-bias stream: 16 + 4 d(v) + 4 (the pick's col) + 4 (path) per step
    deg = torch.tensor([3, 1, 2, 5], dtype=torch.int64)
    path = torch.tensor([[0, 1, 0, 3], [2, 0, 2, 0]], dtype=torch.int32)
    b, m = bench.walk_alg_bytes(CONFIGS["cfg2"], deg, path, cached=False, stream=True)
    assert m == "walk_degree_stream" and b == 6 * 16 + 4 * 14 + 6 * 8
    assert bench.hot_kernel_name(CONFIGS["cfg2"], cached=False, eb=True) == "k_walk_vscan<uint32>"
    assert bench.hot_kernel_name(CONFIGS["cfg2"], cached=False) == "k_walk<degree>"
    assert bench.hot_kernel_name(CONFIGS["cfg3"], n2x=True) == "k_node2vec_tma"


def test_random_gather_context_reads_the_committed_measurement():
    c = bench.random_gather_context(500.0)
    assert c["random_gather_peak_gbs"] > 0
    assert abs(c["frac_of_random_gather_peak"] - 500.0 / c["random_gather_peak_gbs"]) < 1e-12


def test_sample_bytes_cached_sector_model():
    deg = torch.tensor([2, 4, 1, 3, 2], dtype=torch.int64)
    seeds = torch.tensor([1, 3], dtype=torch.int32)
    offs = torch.tensor([0, 4, 6], dtype=torch.int64)
    src = torch.tensor([1, 1, 0, 2, 3, 4], dtype=torch.int32)
    dst = torch.tensor([0, 2, 1, 4, 4, 3], dtype=torch.int32)
    dep = torch.tensor([1, 1, 2, 2, 1, 2], dtype=torch.uint8)
    # expanded vertices: 5 (as in the scan model); per pick ceil(log2 d(src)): src degrees
    # 4, 4, 2, 1, 3, 2 -> 2, 2, 1, 0, 2, 1 = 8
    b, m = bench.sample_alg_bytes(CONFIGS["cfg4_layer"], deg, seeds, offs, src, dst, dep, cached=True)
    assert m == "sample_cached" and b == 16 * 5 + 32 * (2 * 6 + 8) + 9 * 6


def test_bucketed_walk_names_and_weight_models():
    """The bucketed walk kernels are named in the roofline; the cached edge-weight walk uses the
    NEXT-1 sector model (same formula as the cached degree walk), the per-step scan the stream model."""
    assert bench.hot_kernel_name(CONFIGS["cfg2"], cached=True, wix_leaf=128, wix_group=32, heads=True,
                                 buckets=True) == "k_walk_gb"
    assert bench.hot_kernel_name(CONFIGS["cfg2"], cached=True, wix_leaf=128, wix_group=32,
                                 heads=True) == "k_walk_head<128>"
    assert bench.hot_kernel_name(CONFIGS["cfg2_weight"], buckets=True) == "k_walk_gbw"
    assert bench.hot_kernel_name(CONFIGS["cfg2_weight"]) == "k_walk_vscan<float>"
    deg = torch.tensor([3, 1, 2, 5], dtype=torch.int64)
    path = torch.tensor([[0, 1, 0, 3], [2, 0, 2, 0]], dtype=torch.int32)
    bc, mc = bench.walk_alg_bytes(CONFIGS["cfg2_weight"], deg, path, cached=True)
    bd, _ = bench.walk_alg_bytes(CONFIGS["cfg2"], deg, path, cached=True)
    assert mc == "walk_weight_cached" and bc == bd == 32 * (2 * 6 + 8) + 6 * 4
    bs, ms = bench.walk_alg_bytes(CONFIGS["cfg2_weight"], deg, path, cached=False)
    assert ms == "walk_weight_stream" and bs == 6 * 16 + 4 * 14 + 6 * 8


def test_random_line_context():
    """dram_frac_of_random_line_ceiling = ncu DRAM bytes / launch time / the measured random-line rate."""
    c = bench.random_gather_context(500.0, traffic=4.35e9, hot_ms=1.0)
    assert c["random_line_ceiling_gbs"] > 0
    assert abs(c["dram_gbs_ncu"] - 4350.0) < 1e-6
    assert abs(c["dram_frac_of_random_line_ceiling"] - 4350.0 / c["random_line_ceiling_gbs"]) < 1e-12
    assert bench.random_gather_context(500.0)["dram_frac_of_random_line_ceiling"] is None


def test_new_bench_options_parse():
    a = bench.parse_args(["--no-walk-buckets", "--next-meta", "--mdrw-alt-records", "--config", "cfg5"])
    assert a.no_walk_buckets and a.next_meta and a.mdrw_alt_records and a.config == "cfg5"
    d = bench.parse_args([])
    assert d.config == "cfg3" and not d.no_walk_buckets and d.gpus == 1
