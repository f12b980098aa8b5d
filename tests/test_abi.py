"""CPU-side checks of the C ABI boundary (no compute calls without a GPU)."""
import ctypes as C
import os
import re
import subprocess

import pytest
import torch

import paper_2009_09103_b200 as cs
from paper_2009_09103_b200 import _lib


def test_library_builds_and_loads():
    _lib.build()
    assert os.path.exists(_lib.LIB_PATH)
    assert cs.csaw_version().startswith("csaw-b200")


def test_every_header_symbol_is_exported():
    syms = _lib.header_symbols()
    assert {"csaw_graph_create", "csaw_sample", "csaw_walk", "csaw_last_error"} <= set(syms)
    out = subprocess.check_output(["nm", "-D", "--defined-only", _lib.LIB_PATH]).decode()
    exported = set(re.findall(r"\bT (csaw_\w+)", out))
    assert set(syms) <= exported, set(syms) - exported
    # nothing exported beyond the header (C++ internals are hidden)
    assert exported <= set(syms), exported - set(syms)


def test_header_is_plain_c():
    src = open(_lib.HEADER).read()
    assert 'extern "C"' in src
    for bad in ("torch", "at::", "std::", "#include <cuda"):
        assert bad not in src
    # compiles as C99 without CUDA headers
    subprocess.check_call(["gcc", "-std=c99", "-fsyntax-only", "-x", "c", _lib.HEADER])


def test_struct_layouts_match_header():
    # offsets of the ctypes mirrors equal the C layout (compiled probe)
    probe = r'''
#include <stdio.h>
#include <stddef.h>
#include "csaw.h"
int main(void){
 printf("%zu %zu %zu %zu %zu\n", sizeof(csaw_bias), offsetof(csaw_bias,pf), offsetof(csaw_bias,a_max),
        sizeof(csaw_csr), sizeof(csaw_graph_opts));
 printf("%zu %zu\n", sizeof(csaw_graph_info_t), sizeof(csaw_run_stats));
 return 0; }'''
    import tempfile
    d = tempfile.mkdtemp()
    with open(os.path.join(d, "p.c"), "w") as f:
        f.write(probe)
    exe = os.path.join(d, "p")
    subprocess.check_call(["gcc", "-I", os.path.dirname(_lib.HEADER), "-o", exe, os.path.join(d, "p.c")])
    a = subprocess.check_output([exe]).decode().split()
    assert int(a[0]) == C.sizeof(_lib.csaw_bias)
    assert int(a[1]) == _lib.csaw_bias.pf.offset and int(a[2]) == _lib.csaw_bias.a_max.offset
    assert int(a[3]) == C.sizeof(_lib.csaw_csr) and int(a[4]) == C.sizeof(_lib.csaw_graph_opts)
    assert int(a[5]) == C.sizeof(_lib.csaw_graph_info_t) and int(a[6]) == C.sizeof(_lib.csaw_run_stats)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    rp = torch.tensor([0, 1, 2], dtype=torch.int64)
    col = torch.tensor([1, 0], dtype=torch.int32)
    with pytest.raises(cs.CsawError) as ei:
        cs.csaw_graph_create(rp, col)
    assert ei.value.status == 7 and "no CPU fallback" in str(ei.value)


def test_host_capacity_bounds():
    # neighbor sampling: n * (k1 + k1 k2); layer: n * (k1 + k2)
    assert cs.csaw_sample_capacity("degree", [2, 2], 2, 64) == 64 * (2 + 4)
    assert cs.csaw_sample_capacity("uniform", [3, 1, 2], 3, 10) == 10 * (3 + 3 + 6)
    assert cs.csaw_sample_capacity("layer", [2, 2], 2, 8192) == 8192 * 4
    assert cs.csaw_sample_capacity(cs.make_bias("forest_fire", pf=0.7), [], 2, 100) > 0


def test_graph_flags_match_header():
    """Every CSAW_GRAPH_* macro of csaw.h equals the binding's constant of the same name, and the
    flags are distinct single bits (graph-creation options OR together)."""
    src = open(_lib.HEADER).read()
    macros = {m.group(1): int(m.group(2), 16) for m in re.finditer(r"#define (CSAW_GRAPH_\w+) (0x[0-9a-fA-F]+)u", src)}
    assert len(macros) >= 24 and "CSAW_GRAPH_WALK_BUCKETS" in macros and "CSAW_GRAPH_NEXT_RECORD" in macros
    for name, val in macros.items():
        assert getattr(cs, name) == val, name
        assert val & (val - 1) == 0, name
    assert len(set(macros.values())) == len(macros)
    # the info struct mirror carries the fields the binding reports
    fields = [f for f, _ in _lib.csaw_graph_info_t._fields_]
    assert "walk_buckets" in fields and fields.index("walk_buckets") == len(fields) - 2
