"""ctypes loader for libcsaw.so (the C ABI declared in include/csaw.h).

Marshalling only: every step of the sampling path runs in the CUDA library.
There is deliberately no fallback -- if the shared library is missing, or no
CUDA device is present, calls raise CsawError.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG_DIR)
CSRC = os.path.join(PKG_DIR, "csrc")
LIB_PATH = os.environ.get("CSAW_LIB") or os.path.join(PKG_DIR, "libcsaw.so")   # override: A/B experiments
HEADER = os.path.join(ROOT, "include", "csaw.h")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC,-fvisibility=hidden", "-shared"]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def build(force: bool = False, verbose: bool = False) -> str:
    """nvcc-compile every .cu under csrc/ into libcsaw.so for sm_100a (in-tree)."""
    deps = sources() + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))] + [HEADER]
    if (not force and os.path.exists(LIB_PATH)
            and os.path.getmtime(LIB_PATH) >= max(os.path.getmtime(d) for d in deps)):
        return LIB_PATH
    cmd = ["nvcc", *NVCC_FLAGS, "-o", LIB_PATH + ".tmp", *sources()]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    os.replace(LIB_PATH + ".tmp", LIB_PATH)
    return LIB_PATH


class CsawError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"csaw status {status} ({STATUS_NAMES.get(status, '?')}): {msg}")
        self.status = status


STATUS_NAMES = {0: "OK", 1: "INVALID_ARG", 2: "OUT_OF_RANGE", 3: "BAD_GRAPH", 4: "DEGENERATE_POOL",
                5: "CAPACITY", 6: "NO_MEMORY", 7: "CUDA", 8: "UNSUPPORTED"}
CSAW_OK, CSAW_ERR_CAPACITY = 0, 5

# csaw_bias_kind
BIAS = {"uniform": 0, "degree": 1, "node2vec": 2, "forest_fire": 3, "layer": 4, "mdrw": 5, "mh": 6, "restart": 7,
        "jump": 8, "snowball": 9, "weight": 10}


class csaw_bias(C.Structure):
    _fields_ = [("kind", C.c_int32), ("p", C.c_double), ("q", C.c_double), ("pf", C.c_double),
                ("pool_size", C.c_int32), ("a_max", C.c_int32), ("migration", C.c_int32)]


class csaw_csr(C.Structure):
    _fields_ = [("num_vertices", C.c_int64), ("num_edges", C.c_int64), ("row_ptr", C.c_void_p),
                ("col_idx", C.c_void_p), ("weights", C.c_void_p)]


class csaw_graph_opts(C.Structure):
    _fields_ = [("device", C.c_int32), ("device_budget_bytes", C.c_int64), ("num_partitions", C.c_int32),
                ("max_resident", C.c_int32), ("num_streams", C.c_int32), ("flags", C.c_uint32),
                ("store_device", C.c_int32)]


class csaw_graph_info_t(C.Structure):
    _fields_ = [("num_vertices", C.c_int64), ("num_edges", C.c_int64), ("max_degree", C.c_int64),
                ("nonisolated", C.c_int64), ("rows_sorted", C.c_int32), ("oom_mode", C.c_int32),
                ("device_bytes", C.c_int64), ("ctps_cache", C.c_int32), ("walk_index_leaf", C.c_int32),
                ("cache_build_ms", C.c_double), ("walk_index_group", C.c_int32), ("node2vec_tri", C.c_int32), ("walk_index_heads", C.c_int32), ("node2vec_index", C.c_int32),
                ("has_weights", C.c_int32), ("edge_bias", C.c_int32), ("walk_buckets", C.c_int32),
                ("reserved0", C.c_int32)]


class csaw_run_stats(C.Structure):
    _fields_ = [("sampled_edges", C.c_uint64), ("pools", C.c_uint64), ("neighbours_scanned", C.c_uint64),
                ("partition_loads", C.c_uint64), ("h2d_bytes", C.c_uint64), ("cache_probes", C.c_uint64), ("draws", C.c_uint64),
                ("kernel_launches", C.c_uint64),
                ("hot_launches", C.c_uint64), ("kernel_ms", C.c_double), ("hot_kernel_ms", C.c_double),
                ("transfer_ms", C.c_double), ("index_bytes", C.c_uint64)]


_lib = None


def lib():
    """Load libcsaw.so (raises if it is missing: no CPU fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CsawError(7, f"{LIB_PATH} not built (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        P, i32, i64, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
        sig = {
            "csaw_graph_create": [P, P, P],
            "csaw_graph_destroy": [P],
            "csaw_graph_info": [P, P],
            "csaw_sample_capacity": [P, P, i32, i64, P],
            "csaw_sample": [P, P, P, i32, P, i64, u64, u64, P, P, P, P, i64, P, P],
            "csaw_walk": [P, P, i32, P, i64, u64, u64, P, P],
            "csaw_stats": [P, P],
            "csaw_philox": [P, P, P, i64],
            "csaw_selftest_curand": [i64, P],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.csaw_last_error.restype = C.c_char_p
        L.csaw_last_error.argtypes = []
        L.csaw_version.restype = C.c_char_p
        L.csaw_version.argtypes = []
        _lib = L
    return _lib


def check(status: int, allow=(CSAW_OK,)):
    if status not in allow:
        raise CsawError(status, lib().csaw_last_error().decode())
    return status


def header_symbols():
    """Every CSAW_API function declared in include/csaw.h."""
    import re
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"CSAW_API\s+[\w\s\*]+?\b(csaw_\w+)\s*\(", txt)))
