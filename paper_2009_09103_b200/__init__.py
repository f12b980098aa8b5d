"""paper_2009_09103_b200 — B200-native C-SAW hot path (arXiv 2009.09103).

Thin Python binding over the C ABI in include/csaw.h (libcsaw.so, hand-written
sm_100a CUDA).  The functions keep the C names; they only marshal torch
tensors / numpy arrays into pointers.  PyTorch supplies device memory and
streams; every sampling step runs in the library's kernels.

    g = csaw_graph_create(row_ptr, col_idx, device=0)          # CSR -> device graph
    path = csaw_walk(g, "degree", seeds, length=2000, rng_seed=1)
    offs, src, dst, dep = csaw_sample(g, "degree", seeds, fanout=[2, 2], rng_seed=1)
"""
from __future__ import annotations

import ctypes as C

import torch

from ._lib import (BIAS, CSAW_ERR_CAPACITY, CSAW_OK, CsawError, build, check, csaw_bias, csaw_csr,
                   csaw_graph_info_t, csaw_graph_opts, csaw_run_stats, header_symbols, lib)

__all__ = ["csaw_graph_create", "csaw_graph_destroy", "csaw_graph_info", "csaw_sample", "csaw_sample_capacity",
           "csaw_walk", "csaw_stats", "csaw_philox", "csaw_selftest_curand", "csaw_version", "Graph",
           "make_bias", "CsawError", "build", "header_symbols", "NONE"]

NONE = 0xFFFFFFFF


def _ptr(t) -> int:
    if t is None:
        return 0
    if isinstance(t, torch.Tensor):
        if not t.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return t.data_ptr()
    import numpy as np
    if isinstance(t, np.ndarray):
        if not t.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return t.ctypes.data
    raise TypeError(f"unsupported buffer type {type(t)}")


def _stream_ptr(stream, device: int = 0) -> int:
    """None -> the current torch stream of the graph's device."""
    if stream is None:
        return torch.cuda.current_stream(device).cuda_stream if torch.cuda.is_available() else 0
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


MIGRATION = {"brs": 0, "repeated": 1, "updated": 2}


def make_bias(kind, p=1.0, q=1.0, pf=0.0, pool_size=0, a_max=0, migration="brs") -> csaw_bias:
    k = BIAS[kind] if isinstance(kind, str) else int(kind)
    mig = MIGRATION[migration] if isinstance(migration, str) else int(migration)
    return csaw_bias(k, float(p), float(q), float(pf), int(pool_size), int(a_max), mig)


class Graph:
    """Owning handle of a csaw_graph (destroyed on close / garbage collection)."""

    def __init__(self, handle: int, device: int):
        self.handle = C.c_void_p(handle)
        self.device = device

    def close(self):
        if self.handle:
            lib().csaw_graph_destroy(self.handle)
            self.handle = C.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        return csaw_graph_info(self)


CSAW_GRAPH_CTPS_CACHE = 0x1
CSAW_GRAPH_OOM_ZEROCOPY = 0x2
CSAW_GRAPH_SAMPLE_BATCHED = 0x4
CSAW_GRAPH_OOM_NO_WS = 0x8
CSAW_GRAPH_OOM_NO_BAL = 0x10
CSAW_GRAPH_NO_WALK_INDEX = 0x20
CSAW_GRAPH_N2V_TRI = 0x40
CSAW_GRAPH_NEXT_META = 0x80
CSAW_GRAPH_CHUNK_CACHE = 0x100
CSAW_GRAPH_N2V_INDEX = 0x200
CSAW_GRAPH_EDGE_BIAS = 0x400
# variant selectors (results identical; tests / A/B), csaw.h
CSAW_GRAPH_WALK_NO_HEADS = 0x800
CSAW_GRAPH_WALK_LEAF_64 = 0x1000
CSAW_GRAPH_WALK_LEAF_32 = 0x2000
CSAW_GRAPH_WALK_GROUP_16 = 0x4000
CSAW_GRAPH_WALK_GROUP_8 = 0x8000
CSAW_GRAPH_SAMPLE_NO_HEADS = 0x10000
CSAW_GRAPH_OOM_NO_CHUNK_CACHE = 0x20000
CSAW_GRAPH_OOM_ZC_NO_PREFIX = 0x40000
CSAW_GRAPH_MDRW_GENERIC = 0x80000
CSAW_GRAPH_MDRW_ALT_RECORDS = 0x100000
CSAW_GRAPH_NEXT_RECORD = 0x800000
CSAW_GRAPH_WALK_BUCKETS = 0x1000000
CSAW_GRAPH_OOM_PEER_STORE = 0x200000


def csaw_graph_create(row_ptr, col_idx, device: int = 0, budget_bytes: int = 0, num_partitions: int = 0,
                      max_resident: int = 0, num_streams: int = 0, ctps_cache: bool = False,
                      zerocopy: bool = False, batched_only: bool = False, oom_ws: bool = True,
                      oom_bal: bool = True, walk_index: bool = True, node2vec_tri: bool = False,
                      next_meta: bool = False, chunk_cache: bool = False, node2vec_index: bool = False,
                      weights=None, edge_bias: bool = False, flags: int = 0, store_device=None,
                      next_record: bool = False, walk_buckets: bool = False) -> Graph:
    """row_ptr int64[V+1], col_idx int32/uint32[E] (torch tensors, host or device).
    ctps_cache=True builds the static-bias CTPS cache (CSAW_GRAPH_CTPS_CACHE);
    zerocopy=True (with budget_bytes > 0) reads col_idx from pinned host memory;
    oom_ws / oom_bal=False switch off workload-aware scheduling / thread-block
    balancing (OOM ablation, Fig. 13-15); walk_index=False skips the narrow
    walk index built with the cache (degree walks then use the u64 index);
    node2vec_tri=True builds per-edge triangle counts (CSAW_GRAPH_N2V_TRI); next_meta=True
    the per-entry next-vertex metadata used by MDRW (CSAW_GRAPH_NEXT_META); chunk_cache=True
    the degree-bias chunk-total cache (CSAW_GRAPH_CHUNK_CACHE; automatic in OOM mode); node2vec_index=True
    the node2vec per-edge intersection index (CSAW_GRAPH_N2V_INDEX, best-effort); weights = float32[E]
    edge weights (csaw_csr.weights, EdgeBias of the "weight" selector); edge_bias=True the materialised
    degree bias deg(col[e]) (CSAW_GRAPH_EDGE_BIAS: degree walks without the cache stream it); flags = extra
    CSAW_GRAPH_* bits (the variant selectors); store_device = GPU whose HBM holds the OOM partition store
    (CSAW_GRAPH_OOM_PEER_STORE; == device: a same-device stand-in); next_record=True the 16 B per-entry
    next-vertex records MDRW reads instead of col + next_meta (CSAW_GRAPH_NEXT_RECORD); walk_buckets=True (with
    ctps_cache) the bucketed degree-walk index (CSAW_GRAPH_WALK_BUCKETS, one DRAM round trip per step)."""
    V = row_ptr.numel() - 1
    if weights is not None and weights.dtype != torch.float32:
        raise TypeError("weights must be float32")
    csr = csaw_csr(V, col_idx.numel(), _ptr(row_ptr), _ptr(col_idx), _ptr(weights) or None)
    opt = csaw_graph_opts(device, budget_bytes, num_partitions, max_resident, num_streams,
                          (CSAW_GRAPH_CTPS_CACHE if ctps_cache else 0) | (CSAW_GRAPH_OOM_ZEROCOPY if zerocopy else 0)
                          | (CSAW_GRAPH_SAMPLE_BATCHED if batched_only else 0)
                          | (0 if oom_ws else CSAW_GRAPH_OOM_NO_WS) | (0 if oom_bal else CSAW_GRAPH_OOM_NO_BAL)
                          | (0 if walk_index else CSAW_GRAPH_NO_WALK_INDEX)
                          | (CSAW_GRAPH_N2V_TRI if node2vec_tri else 0)
                          | (CSAW_GRAPH_NEXT_META if next_meta else 0)
                          | (CSAW_GRAPH_NEXT_RECORD if next_record else 0)
                          | (CSAW_GRAPH_WALK_BUCKETS if walk_buckets else 0)
                          | (CSAW_GRAPH_CHUNK_CACHE if chunk_cache else 0)
                          | (CSAW_GRAPH_N2V_INDEX if node2vec_index else 0)
                          | (CSAW_GRAPH_EDGE_BIAS if edge_bias else 0) | int(flags)
                          | (CSAW_GRAPH_OOM_PEER_STORE if store_device is not None else 0),
                          -1 if store_device is None else int(store_device))
    out = C.c_void_p()
    check(lib().csaw_graph_create(C.byref(csr), C.byref(opt), C.byref(out)))
    return Graph(out.value, device)


def csaw_graph_destroy(g: Graph):
    g.close()


def csaw_graph_info(g: Graph) -> dict:
    info = csaw_graph_info_t()
    check(lib().csaw_graph_info(g.handle, C.byref(info)))
    return {f: getattr(info, f) for f, _ in info._fields_}


def csaw_stats(g: Graph) -> dict:
    s = csaw_run_stats()
    check(lib().csaw_stats(g.handle, C.byref(s)))
    return {f: getattr(s, f) for f, _ in s._fields_}


def csaw_sample_capacity(bias, fanout, depth, n_instances) -> int:
    b = bias if isinstance(bias, csaw_bias) else make_bias(bias)
    fan = (C.c_int32 * max(1, depth))(*([int(x) for x in fanout] + [0] * (depth - len(fanout))))
    cap = C.c_int64()
    check(lib().csaw_sample_capacity(C.byref(b), fan, depth, n_instances, C.byref(cap)))
    return cap.value


def csaw_sample(g: Graph, bias, seeds, fanout=(), depth=None, instance_base=0, rng_seed=1, capacity=None,
                out=None, stream=None, **bias_kw):
    """Traversal sampling.  seeds: uint32/int32 tensor [n] (device or pinned/host).
    Returns (offsets uint64[n+1], src, dst, depth) -- on the seeds' device.
    `out` = (offsets, src, dst, edge_depth) preallocated buffers (host or device)."""
    b = bias if isinstance(bias, csaw_bias) else make_bias(bias, **bias_kw)
    depth = len(fanout) if depth is None else depth
    n = seeds.numel()
    fan = (C.c_int32 * max(1, depth))(*([int(x) for x in fanout] + [0] * (depth - len(fanout))))
    dev = seeds.device if isinstance(seeds, torch.Tensor) else torch.device("cpu")
    if out is None:
        if capacity is None:
            capacity = csaw_sample_capacity(b, fanout, depth, n)
        offs = torch.empty(n + 1, dtype=torch.int64, device=dev)
        src = torch.empty(max(capacity, 1), dtype=torch.int32, device=dev)
        dst = torch.empty(max(capacity, 1), dtype=torch.int32, device=dev)
        dep = torch.empty(max(capacity, 1), dtype=torch.uint8, device=dev)
    else:
        offs, src, dst, dep = out
        capacity = src.numel()
    ne = C.c_int64()
    st = check(lib().csaw_sample(g.handle, C.byref(b), fan, depth, _ptr(seeds), n, instance_base, rng_seed,
                                 _ptr(offs), _ptr(src), _ptr(dst), _ptr(dep), capacity, C.byref(ne),
                                 C.c_void_p(_stream_ptr(stream, g.device))), allow=(CSAW_OK, CSAW_ERR_CAPACITY))
    if st == CSAW_ERR_CAPACITY:
        if out is not None:
            raise CsawError(st, lib().csaw_last_error().decode())
        return csaw_sample(g, b, seeds, fanout, depth, instance_base, rng_seed, capacity=ne.value, stream=stream)
    m = ne.value
    return offs, src[:m], dst[:m], dep[:m]


def csaw_walk(g: Graph, bias, seeds, length: int, instance_base=0, rng_seed=1, out=None, stream=None, **bias_kw):
    """Random walks.  degree/uniform/node2vec: seeds [n] -> path [n, length+1];
    mdrw: seeds [n, pool_size] -> edges [n, length, 2]."""
    b = bias if isinstance(bias, csaw_bias) else make_bias(bias, **bias_kw)
    if b.kind == BIAS["mdrw"]:
        n = seeds.shape[0]
        b.pool_size = seeds.shape[1]
        shape = (n, length, 2)
    else:
        n = seeds.numel()
        shape = (n, length + 1)
    if out is None:
        dev = seeds.device if isinstance(seeds, torch.Tensor) else torch.device("cpu")
        out = torch.empty(shape, dtype=torch.int32, device=dev)
    check(lib().csaw_walk(g.handle, C.byref(b), length, _ptr(seeds), n, instance_base, rng_seed, _ptr(out),
                          C.c_void_p(_stream_ptr(stream, g.device))))
    return out


def csaw_philox(ctr, key, out=None):
    n = ctr.shape[0]
    if out is None:
        out = torch.empty((n, 4), dtype=torch.int32, device=ctr.device)
    check(lib().csaw_philox(_ptr(ctr), _ptr(key), _ptr(out), n))
    return out


def csaw_selftest_curand(n: int) -> int:
    m = C.c_int64()
    check(lib().csaw_selftest_curand(n, C.byref(m)))
    return m.value


def csaw_version() -> str:
    return lib().csaw_version().decode()
