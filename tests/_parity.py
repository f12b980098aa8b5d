"""Helpers comparing the CUDA path (through the C ABI) with the CPU oracle."""
from __future__ import annotations

import numpy as np
import torch

import oracle as O
import paper_2009_09103_b200 as cs

DEV = "cuda:0"


def u32(t) -> np.ndarray:
    a = t.cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)
    return a.view(np.uint32) if a.dtype == np.int32 else a.astype(np.uint32)


def graph_pair(row_ptr, col):
    """(device csaw graph, oracle graph) for a CSR given as torch/numpy arrays."""
    rp = torch.as_tensor(np.asarray(row_ptr, dtype=np.int64))
    c = torch.as_tensor(np.asarray(col).astype(np.uint32).view(np.int32))
    G = cs.csaw_graph_create(rp.to(DEV), c.to(DEV), device=0)
    return G, O.Graph(rp.numpy(), c.numpy().view(np.uint32))


def check_sample(G, og, workload, seeds, fanout=(), depth=None, rng_seed=1, instance_base=0, pf=0.0,
                 a_max=0, instances=None, migration="brs"):
    """Run csaw_sample and compare every instance (or `instances`) with the oracle, element by element."""
    depth = len(fanout) if depth is None else depth
    kind = {"degree": "degree", "uniform": "uniform", "forest_fire": "forest_fire", "layer": "layer",
            "snowball": "snowball"}[workload]
    seeds_t = torch.as_tensor(np.asarray(seeds).astype(np.uint32).view(np.int32)).to(DEV)
    b = cs.make_bias(kind, pf=pf, a_max=a_max, migration=migration)
    offs, src, dst, dep = cs.csaw_sample(G, b, seeds_t, fanout=fanout, depth=depth, rng_seed=rng_seed,
                                         instance_base=instance_base)
    offs = offs.cpu().numpy().astype(np.int64)
    src, dst, dep = u32(src), u32(dst), dep.cpu().numpy()
    am = a_max or O.A_MAX_DEFAULT
    ids = range(len(seeds)) if instances is None else instances
    total = 0
    O.set_migration(migration)
    try:
        total = _compare_instances(og, workload, seeds, fanout, depth, rng_seed, instance_base, pf, am, ids,
                                   offs, src, dst, dep)
    finally:
        O.set_migration("brs")
    return offs, total


def _compare_instances(og, workload, seeds, fanout, depth, rng_seed, instance_base, pf, am, ids, offs, src, dst, dep):
    total = 0
    for i in ids:
        gi = instance_base + i
        if workload == "layer":
            es, ed, ee = O.layer_sample(og, fanout, depth, int(seeds[i]), gi, rng_seed, am)
        else:
            k = {"degree": O.KIND_DEGREE, "uniform": O.KIND_UNIFORM, "forest_fire": O.KIND_FF,
                 "snowball": O.KIND_SNOWBALL}[workload]
            es, ed, ee = O.neighbor_sample(og, k, fanout, depth, int(seeds[i]), gi, rng_seed, pf, am)
        a, bnd = int(offs[i]), int(offs[i + 1])
        assert bnd - a == es.size, f"instance {i}: {bnd - a} edges vs oracle {es.size}"
        assert np.array_equal(src[a:bnd], es), f"instance {i}: src differs"
        assert np.array_equal(dst[a:bnd], ed), f"instance {i}: dst differs"
        assert np.array_equal(dep[a:bnd], ee), f"instance {i}: depth differs"
        total += es.size
    return total


def check_walk(G, og, kind, seeds, length, rng_seed=1, instance_base=0, walkers=None, p=1.0, q=1.0):
    seeds_t = torch.as_tensor(np.asarray(seeds).astype(np.uint32).view(np.int32)).to(DEV)
    path = u32(cs.csaw_walk(G, cs.make_bias(kind, p=p, q=q), seeds_t, length, rng_seed=rng_seed,
                            instance_base=instance_base))
    ids = range(len(seeds)) if walkers is None else walkers
    for w in ids:
        gi = instance_base + w
        if kind == "node2vec":
            ref = O.node2vec(og, p, q, length, int(seeds[w]), gi, rng_seed)
        else:
            ref = O.walk(og, O.KIND_DEGREE if kind == "degree" else O.KIND_UNIFORM, length, int(seeds[w]), gi,
                         rng_seed)
        if not np.array_equal(path[w], ref):
            t = int(np.argmax(path[w] != ref))
            raise AssertionError(f"walker {w}: first divergence at path index {t}: gpu {path[w][t]} oracle {ref[t]}")
    return path


def check_node2vec_float(G, og, seeds, length, p, q, rng_seed=1, walkers=None, tol=1e-6):
    """Float path: teacher-forced per-step check; a pick may differ from the oracle's
    only where the oracle's draw lies within tol*T of a CTPS boundary (north star)."""
    seeds_t = torch.as_tensor(np.asarray(seeds).astype(np.uint32).view(np.int32)).to(DEV)
    path = u32(cs.csaw_walk(G, cs.make_bias("node2vec", p=p, q=q), seeds_t, length, rng_seed=rng_seed))
    ids = range(len(seeds)) if walkers is None else walkers
    excused = 0
    for w in ids:
        assert path[w][0] == seeds[w]
        for t in range(length):
            prev = O.NONE32 if t == 0 else int(path[w][t - 1])
            ref, margin = O.node2vec_step(og, p, q, prev, int(path[w][t]), w, t, rng_seed)
            if int(path[w][t + 1]) != ref:
                assert margin <= tol, f"walker {w} step {t}: gpu {path[w][t+1]} oracle {ref} margin {margin}"
                excused += 1
    return excused


def check_mdrw(G, og, seeds2d, steps, rng_seed=1, instances=None):
    s = torch.as_tensor(np.asarray(seeds2d).astype(np.uint32).view(np.int32)).to(DEV)
    edges = u32(cs.csaw_walk(G, cs.make_bias("mdrw"), s, steps, rng_seed=rng_seed))
    ids = range(seeds2d.shape[0]) if instances is None else instances
    for i in ids:
        ref = O.mdrw(og, seeds2d[i], steps, i, rng_seed)
        if not np.array_equal(edges[i], ref):
            t = int(np.argmax((edges[i] != ref).any(axis=1)))
            raise AssertionError(f"instance {i}: first divergence at step {t}: gpu {edges[i][t]} oracle {ref[t]}")
    return edges
