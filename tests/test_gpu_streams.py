"""ABI conventions under concurrent use: calls on one graph issued on
different streams without host synchronisation must not share scratch while an
earlier call still runs, and buffers of mixed location classes are rejected."""
import numpy as np
import pytest
import torch

import paper_2009_09103_b200 as cs
from synth import instance_seeds, mdrw_seeds, rmat_csr
from tests._parity import DEV

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def graph():
    g = rmat_csr(1 << 15, 1 << 19, 7, device=DEV)
    G = cs.csaw_graph_create(g.row_ptr, g.col_idx, device=0)
    return g, G


def test_mdrw_calls_on_two_streams_equal_sequential(graph):
    g, G = graph
    sa = mdrw_seeds(g, 64, 500, set_id=1).to(DEV)
    sb = mdrw_seeds(g, 64, 500, set_id=2).to(DEV)
    ref_a = cs.csaw_walk(G, "mdrw", sa, 400, rng_seed=3)
    ref_b = cs.csaw_walk(G, "mdrw", sb, 400, rng_seed=4)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for _ in range(3):
        a = torch.empty_like(ref_a)
        b = torch.empty_like(ref_b)
        cs.csaw_walk(G, "mdrw", sa, 400, rng_seed=3, out=a, stream=s1)    # MDRW pool state in scratch
        cs.csaw_walk(G, "mdrw", sb, 400, rng_seed=4, out=b, stream=s2)    # same scratch, other stream
        outs.append((a, b))
    torch.cuda.synchronize()
    for a, b in outs:
        assert torch.equal(a, ref_a) and torch.equal(b, ref_b)


def test_sampling_calls_on_two_streams_equal_sequential(graph):
    g, G = graph
    seeds = instance_seeds(g, 2000).to(DEV)
    ref = cs.csaw_sample(G, "degree", seeds, fanout=[8, 4], rng_seed=2)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(s1):
        r1 = cs.csaw_sample(G, "degree", seeds, fanout=[8, 4], rng_seed=2, stream=s1)
    with torch.cuda.stream(s2):
        r2 = cs.csaw_sample(G, "degree", seeds, fanout=[8, 4], rng_seed=2, stream=s2)
    torch.cuda.synchronize()
    for x, y, z in zip(ref, r1, r2):
        assert torch.equal(x, y) and torch.equal(x, z)


def test_mixed_output_locations_rejected(graph):
    g, G = graph
    seeds = instance_seeds(g, 16).to(DEV)
    cap = cs.csaw_sample_capacity(cs.make_bias("degree"), [2, 2], 2, 16)
    offs = torch.empty(17, dtype=torch.int64, device=DEV)
    src = torch.empty(cap, dtype=torch.int32, device=DEV)
    dst = torch.empty(cap, dtype=torch.int32).pin_memory()
    dep = torch.empty(cap, dtype=torch.uint8, device=DEV)
    with pytest.raises(cs.CsawError) as e:
        cs.csaw_sample(G, "degree", seeds, fanout=[2, 2], out=(offs, src, dst, dep))
    assert e.value.status == 1
