"""ctypes wrapper of the C-SAW CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE, NOT PRODUCT CODE: only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this package.  It
never imports the CUDA library package and the CUDA library never imports it.

Every function restates a passage of the paper; see oracle.c for citations.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from concurrent.futures import ProcessPoolExecutor

import numpy as np

_DIR = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_DIR, "oracle.c")
_LIB = os.path.join(_DIR, "liboracle.so")

NONE32 = 0xFFFFFFFF
A_MAX_DEFAULT = 64


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (plain -O2, no threads, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fvisibility=hidden",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        P = C.c_void_p
        i64, i32, u32, u64, f64 = C.c_int64, C.c_int32, C.c_uint32, C.c_uint64, C.c_double
        sig = {
            "oracle_philox4x32_10": (None, [P, P, P]),
            "oracle_below": (u64, [u64, u64]),
            "oracle_prefix": (None, [P, i64, P]),
            "oracle_its": (i64, [P, i64, u64]),
            "oracle_brs_step": (i64, [P, P, i64, i64, u64]),
            "oracle_select_wor": (i64, [P, i64, i64, u64, u32, u32, u32, i32, P, P]),
            "oracle_set_migration": (None, [i32]),
            "oracle_ff_theta": (u64, [f64]),
            "oracle_ff_burn": (i64, [u64, u32, u32, u32, i64, f64]),
            "oracle_neighbor_sample": (i64, [P, P, i64, i32, P, i32, f64, u32, u32, u64, i32, P, P, P, i64, P]),
            "oracle_layer_sample": (i64, [P, P, i64, P, i32, u32, u32, u64, i32, P, P, P, i64, P]),
            "oracle_walk_step": (u32, [P, P, i64, i32, u32, u32, u32, u64]),
            "oracle_walk": (None, [P, P, i64, i32, i32, u32, u32, u64, P]),
            "oracle_walk_variant_step": (u32, [P, P, i64, i32, f64, u32, u32, u32, u32, u64]),
            "oracle_walk_variant": (None, [P, P, i64, i32, f64, i32, u32, u32, u64, P]),
            "oracle_n2v_scale": (u32, [f64, f64]),
            "oracle_select_float": (i64, [P, i64, u64, P]),
            "oracle_node2vec_step": (u32, [P, P, i64, f64, f64, u32, u32, u32, u32, u64, P]),
            "oracle_node2vec": (None, [P, P, i64, f64, f64, i32, u32, u32, u64, P, P]),
            "oracle_mdrw": (None, [P, P, i64, P, i32, i32, u32, u64, P]),
            "oracle_select_wor_float": (i64, [P, i64, i64, u64, u32, u32, u32, i32, P, P]),
            "oracle_weight_walk_step": (u32, [P, P, P, i64, u32, u32, u32, u64, P]),
            "oracle_weight_walk": (None, [P, P, P, i64, i32, u32, u32, u64, P, P]),
            "oracle_weight_sample": (i64, [P, P, P, i64, P, i32, u32, u32, u64, i32, P, P, P, i64, P]),
            "oracle_node2vec_w_step": (u32, [P, P, P, i64, f64, f64, u32, u32, u32, u32, u64, P]),
            "oracle_node2vec_w": (None, [P, P, P, i64, f64, f64, i32, u32, u32, u64, P, P]),
            "oracle_partition_bounds": (None, [i64, i32, P]),
            "oracle_active_counts": (None, [P, i32, P, i64, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class Graph:
    """Host CSR handed to the oracle: row_ptr int64[V+1], col uint32[E] (sorted rows),
    optional edge weights w float32[E] (EdgeBias = w(e))."""

    def __init__(self, row_ptr, col_idx, weights=None):
        self.row_ptr = np.ascontiguousarray(np.asarray(row_ptr, dtype=np.int64))
        self.col = np.ascontiguousarray(np.asarray(col_idx).astype(np.uint32, copy=False))
        self.V = self.row_ptr.size - 1
        self.w = None if weights is None else np.ascontiguousarray(np.asarray(weights, dtype=np.float32))

    @classmethod
    def from_torch(cls, g, weights=None):
        w = None if weights is None else weights.cpu().numpy().astype(np.float32, copy=False)
        return cls(g.row_ptr.cpu().numpy(), g.col_idx.cpu().numpy().view(np.uint32), w)

    def deg(self, v):
        return int(self.row_ptr[v + 1] - self.row_ptr[v])

    def nbrs(self, v):
        return self.col[self.row_ptr[v]:self.row_ptr[v + 1]]


# ---------------------------------------------------------------- primitives
def philox4x32_10(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_p(c), _p(k), _p(o))
    return [int(x) for x in o]


def below(U: int, M: int) -> int:
    return int(lib().oracle_below(U, M))


def prefix(b) -> np.ndarray:
    b = np.ascontiguousarray(np.asarray(b, dtype=np.uint32))
    S = np.zeros(b.size + 1, dtype=np.uint64)
    lib().oracle_prefix(_p(b), b.size, _p(S))
    return S


def its(S, x: int) -> int:
    S = np.ascontiguousarray(np.asarray(S, dtype=np.uint64))
    return int(lib().oracle_its(_p(S), S.size - 1, x))


def brs_step(b, s, x2) -> int:
    b = np.ascontiguousarray(np.asarray(b, dtype=np.uint32))
    S = prefix(b)
    return int(lib().oracle_brs_step(_p(S), _p(b), b.size, s, x2))


def select_wor(b, k, seed, inst, t, slot, a_max=A_MAX_DEFAULT, with_attempts=False):
    b = np.ascontiguousarray(np.asarray(b, dtype=np.uint32))
    picks = np.zeros(max(b.size, 1), dtype=np.int64)
    att = np.zeros(1, dtype=np.int64)
    n = lib().oracle_select_wor(_p(b), b.size, k, seed, inst, t, slot, a_max, _p(picks), _p(att))
    r = [int(x) for x in picks[:n]]
    return (r, int(att[0])) if with_attempts else r


MIGRATION = {"brs": 0, "repeated": 1, "updated": 2}


def set_migration(mode) -> None:
    """Collision-migration mode of every later selection in this process (0 BRS, 1 repeated, 2 updated)."""
    lib().oracle_set_migration(MIGRATION[mode] if isinstance(mode, str) else int(mode))


def ff_theta(pf: float) -> int:
    return int(lib().oracle_ff_theta(pf))


def ff_burn(seed, inst, depth, v, deg, pf) -> int:
    return int(lib().oracle_ff_burn(seed, inst, depth, v, deg, pf))


def select_float(b, U: int):
    """Float-bias ITS (R28): -> (s, margin); s = -1 if the pool total is 0."""
    b = np.ascontiguousarray(np.asarray(b, dtype=np.float32))
    m = np.zeros(1, dtype=np.float64)
    s = lib().oracle_select_float(_p(b), b.size, U, _p(m))
    return int(s), float(m[0])


def select_wor_float(b, k, seed, inst, t, slot, a_max=A_MAX_DEFAULT):
    """Without-replacement selection over fp32 biases (float BRS, R28) -> (picks in
    pick order, minimum boundary margin over the draws)."""
    b = np.ascontiguousarray(np.asarray(b, dtype=np.float32))
    picks = np.zeros(max(b.size, 1), dtype=np.int64)
    m = np.ones(1, dtype=np.float64)
    n = lib().oracle_select_wor_float(_p(b), b.size, k, seed, inst, t, slot, a_max, _p(picks), _p(m))
    return [int(x) for x in picks[:n]], float(m[0])


def weight_walk_step(g: Graph, v, inst, t, rng_seed):
    """One edge-weight walk step at v -> (next vertex, margin)."""
    m = np.ones(1, dtype=np.float64)
    u = lib().oracle_weight_walk_step(_p(g.row_ptr), _p(g.col), _p(g.w), g.V, v, inst, t, rng_seed, _p(m))
    return int(u), float(m[0])


def weight_walk(g: Graph, length, s0, inst, rng_seed, with_margins=False):
    path = np.zeros(length + 1, dtype=np.uint32)
    mg = np.ones(max(length, 1), dtype=np.float64)
    lib().oracle_weight_walk(_p(g.row_ptr), _p(g.col), _p(g.w), g.V, length, s0, inst, rng_seed, _p(path), _p(mg))
    return (path, mg[:length]) if with_margins else path


def weight_sample(g: Graph, fanout, depth, seed_vertex, inst, rng_seed, a_max=A_MAX_DEFAULT):
    """Edge-weight neighbor sampling of one instance -> (src, dst, depth, min margin)."""
    fan = np.ascontiguousarray(np.asarray(list(fanout) + [0] * max(0, depth - len(fanout)), dtype=np.int32))
    cap = 1024
    m = np.ones(1, dtype=np.float64)
    while True:
        s = np.zeros(cap, np.uint32); d = np.zeros(cap, np.uint32); e = np.zeros(cap, np.uint8)
        n = lib().oracle_weight_sample(_p(g.row_ptr), _p(g.col), _p(g.w), g.V, _p(fan), depth, seed_vertex, inst,
                                       rng_seed, a_max, _p(s), _p(d), _p(e), cap, _p(m))
        if n >= 0:
            return s[:n], d[:n], e[:n], float(m[0])
        cap = -n


def n2v_scale(p, q) -> int:
    return int(lib().oracle_n2v_scale(p, q))


# ---------------------------------------------------------------- workloads
KIND_UNIFORM, KIND_DEGREE, KIND_FF, KIND_SNOWBALL = 0, 1, 2, 3


def neighbor_sample(g: Graph, kind, fanout, depth, seed_vertex, inst, rng_seed, pf=0.0,
                    a_max=A_MAX_DEFAULT):
    """One instance -> (src, dst, depth) uint arrays in canonical order."""
    fan = np.ascontiguousarray(np.asarray(list(fanout) + [0] * max(0, depth - len(fanout)), dtype=np.int32))
    cap = 1024
    while True:
        s = np.zeros(cap, np.uint32); d = np.zeros(cap, np.uint32); e = np.zeros(cap, np.uint8)
        n = lib().oracle_neighbor_sample(_p(g.row_ptr), _p(g.col), g.V, kind, _p(fan), depth, pf,
                                         seed_vertex, inst, rng_seed, a_max, _p(s), _p(d), _p(e), cap, None)
        if n >= 0:
            return s[:n], d[:n], e[:n]
        cap = -n


def layer_sample(g: Graph, fanout, depth, seed_vertex, inst, rng_seed, a_max=A_MAX_DEFAULT):
    fan = np.ascontiguousarray(np.asarray(fanout, dtype=np.int32))
    cap = 1024
    while True:
        s = np.zeros(cap, np.uint32); d = np.zeros(cap, np.uint32); e = np.zeros(cap, np.uint8)
        n = lib().oracle_layer_sample(_p(g.row_ptr), _p(g.col), g.V, _p(fan), depth,
                                      seed_vertex, inst, rng_seed, a_max, _p(s), _p(d), _p(e), cap, None)
        if n >= 0:
            return s[:n], d[:n], e[:n]
        cap = -n


def walk_step(g: Graph, kind, v, inst, t, rng_seed) -> int:
    return int(lib().oracle_walk_step(_p(g.row_ptr), _p(g.col), g.V, kind, v, inst, t, rng_seed))


def walk(g: Graph, kind, length, s0, inst, rng_seed) -> np.ndarray:
    path = np.zeros(length + 1, dtype=np.uint32)
    lib().oracle_walk(_p(g.row_ptr), _p(g.col), g.V, kind, length, s0, inst, rng_seed, _p(path))
    return path


KIND_MH, KIND_RESTART, KIND_JUMP = 6, 7, 8


def walk_variant(g: Graph, kind, length, s0, inst, rng_seed, pr=0.0) -> np.ndarray:
    """Metropolis-Hastings (6), restart (7) or jump (8) walk (Table 1 variants)."""
    path = np.zeros(length + 1, dtype=np.uint32)
    lib().oracle_walk_variant(_p(g.row_ptr), _p(g.col), g.V, kind, pr, length, s0, inst, rng_seed, _p(path))
    return path


def walk_variant_step(g: Graph, kind, pr, s0, v, inst, t, rng_seed) -> int:
    return int(lib().oracle_walk_variant_step(_p(g.row_ptr), _p(g.col), g.V, kind, pr, s0, v, inst, t, rng_seed))


def node2vec_step(g: Graph, p, q, prev, v, inst, t, rng_seed):
    m = np.zeros(1, dtype=np.float64)
    u = lib().oracle_node2vec_step(_p(g.row_ptr), _p(g.col), g.V, p, q, prev, v, inst, t, rng_seed, _p(m))
    return int(u), float(m[0])


def node2vec(g: Graph, p, q, length, s0, inst, rng_seed, with_margins=False):
    path = np.zeros(length + 1, dtype=np.uint32)
    mg = np.ones(max(length, 1), dtype=np.float64)
    lib().oracle_node2vec(_p(g.row_ptr), _p(g.col), g.V, p, q, length, s0, inst, rng_seed, _p(path), _p(mg))
    return (path, mg[:length]) if with_margins else path


def node2vec_w_step(g: Graph, p, q, prev, v, inst, t, rng_seed):
    """Weighted node2vec step (alpha * w, R33) -> (next vertex, margin)."""
    m = np.ones(1, dtype=np.float64)
    u = lib().oracle_node2vec_w_step(_p(g.row_ptr), _p(g.col), _p(g.w), g.V, p, q, prev, v, inst, t, rng_seed, _p(m))
    return int(u), float(m[0])


def node2vec_w(g: Graph, p, q, length, s0, inst, rng_seed, with_margins=False):
    path = np.zeros(length + 1, dtype=np.uint32)
    mg = np.ones(max(length, 1), dtype=np.float64)
    lib().oracle_node2vec_w(_p(g.row_ptr), _p(g.col), _p(g.w), g.V, p, q, length, s0, inst, rng_seed, _p(path), _p(mg))
    return (path, mg[:length]) if with_margins else path


def mdrw(g: Graph, seeds, steps, inst, rng_seed) -> np.ndarray:
    seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint32))
    edges = np.zeros((steps, 2), dtype=np.uint32)
    lib().oracle_mdrw(_p(g.row_ptr), _p(g.col), g.V, _p(seeds), seeds.size, steps, inst, rng_seed, _p(edges))
    return edges


def partition_bounds(V, P) -> list:
    b = np.zeros(P + 1, dtype=np.int64)
    lib().oracle_partition_bounds(V, P, _p(b))
    return [int(x) for x in b]


def active_counts(bounds, frontier) -> list:
    bnd = np.ascontiguousarray(np.asarray(bounds, dtype=np.int64))
    f = np.ascontiguousarray(np.asarray(frontier, dtype=np.uint32))
    c = np.zeros(bnd.size - 1, dtype=np.int64)
    lib().oracle_active_counts(_p(bnd), bnd.size - 1, _p(f), f.size, _p(c))
    return [int(x) for x in c]


# ---------------------------------------------------------------- batch runners
def sample_instances(g: Graph, workload: str, seeds, instance_base, rng_seed, fanout=(), depth=0,
                     pf=0.0, a_max=A_MAX_DEFAULT, instances=None):
    """Run the oracle for instances (local ids) -> list of (src, dst, depth) per instance."""
    seeds = np.asarray(seeds).astype(np.uint32)
    ids = range(len(seeds)) if instances is None else instances
    out = []
    for i in ids:
        gi = instance_base + int(i)
        if workload == "layer":
            out.append(layer_sample(g, fanout, depth, int(seeds[i]), gi, rng_seed, a_max))
        else:
            kind = {"uniform": KIND_UNIFORM, "degree": KIND_DEGREE, "forest_fire": KIND_FF,
                    "snowball": KIND_SNOWBALL}[workload]
            out.append(neighbor_sample(g, kind, fanout, depth, int(seeds[i]), gi, rng_seed, pf, a_max))
    return out


# process-pool helpers (fork inherits the graph arrays copy-on-write)
_G: Graph | None = None


def _init_pool(g):
    global _G
    _G = g


def _walk_job(args):
    kind, length, seeds, base, first, rng_seed = args
    return [walk(_G, kind, length, int(s), base + first + j, rng_seed) for j, s in enumerate(seeds)]


def parallel_walks(g: Graph, kind, length, seeds, instance_base, rng_seed, workers=None):
    """Oracle walks on all host cores over disjoint walker ranges (instances are
    independent).  Returns uint32 [n, length+1]."""
    seeds = np.asarray(seeds).astype(np.uint32)
    workers = workers or os.cpu_count() or 1
    n = seeds.size
    chunks = np.array_split(np.arange(n), min(n, workers * 4) or 1)
    jobs = [(kind, length, seeds[c], instance_base, int(c[0]) if c.size else 0, rng_seed) for c in chunks if c.size]
    import multiprocessing as mp
    with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("fork"),
                             initializer=_init_pool, initargs=(g,)) as ex:
        res = list(ex.map(_walk_job, jobs))
    return np.stack([p for r in res for p in r]) if n else np.zeros((0, length + 1), np.uint32)


def _run_job(args):
    """One chunk of independent instances (fork worker; the graph is inherited)."""
    workload, params, ids, seeds, instance_base, rng_seed = args
    out = []
    for i, s in zip(ids, seeds):
        gi = instance_base + int(i)
        if workload == "walk":
            out.append(walk(_G, params["kind"], params["length"], int(s), gi, rng_seed))
        elif workload == "node2vec":
            out.append(node2vec(_G, params["p"], params["q"], params["length"], int(s), gi, rng_seed))
        elif workload == "mdrw":
            out.append(mdrw(_G, s, params["length"], gi, rng_seed))
        elif workload == "layer":
            out.append(layer_sample(_G, params["fanout"], params["depth"], int(s), gi, rng_seed))
        elif workload == "weight_walk":
            out.append(weight_walk(_G, params["length"], int(s), gi, rng_seed, with_margins=True))
        elif workload == "weight":
            out.append(weight_sample(_G, params["fanout"], params["depth"], int(s), gi, rng_seed))
        elif workload == "node2vec_w":
            out.append(node2vec_w(_G, params["p"], params["q"], params["length"], int(s), gi, rng_seed,
                                  with_margins=True))
        else:
            kind = {"uniform": KIND_UNIFORM, "degree": KIND_DEGREE, "forest_fire": KIND_FF,
                    "snowball": KIND_SNOWBALL}[workload]
            out.append(neighbor_sample(_G, kind, params.get("fanout", ()), params["depth"], int(s), gi, rng_seed,
                                       params.get("pf", 0.0)))
    return out


def parallel_run(g: Graph, workload: str, seeds, instance_base, rng_seed, ids=None, workers=None, **params):
    """The oracle over instances `ids` (local ids into `seeds`; default all) on all host
    cores, fanned out over disjoint chunks (instances are independent).
    workload: walk (params kind, length) | node2vec (p, q, length) | mdrw (length;
    seeds[i] is the instance's pool) | layer (fanout, depth) | degree / uniform /
    forest_fire / snowball (fanout, depth, pf) | weight_walk (length; -> (path, margins)) |
    weight (fanout, depth; -> (src, dst, depth, margin)).  Returns the per-instance results in
    the order of ids (walks: path arrays; MDRW: edge arrays; sampling: (src, dst, depth))."""
    import multiprocessing as mp
    seeds = np.asarray(seeds)
    ids = np.arange(len(seeds)) if ids is None else np.asarray(ids, dtype=np.int64)
    if ids.size == 0:
        return []
    workers = workers or os.cpu_count() or 1
    chunks = np.array_split(ids, min(ids.size, workers * 8))
    jobs = [(workload, params, c, seeds[c], instance_base, rng_seed) for c in chunks if c.size]
    if workers == 1:
        global _G
        _G = g
        return [r for j in jobs for r in _run_job(j)]
    with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("fork"),
                             initializer=_init_pool, initargs=(g,)) as ex:
        res = list(ex.map(_run_job, jobs))
    return [r for chunk in res for r in chunk]
