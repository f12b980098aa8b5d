"""Chunk-total cache of the degree bias (CSAW_GRAPH_CHUNK_CACHE; automatic in OOM mode):
pools of more than 256 candidates read their chunk prefix sums instead of scanning, and
rescan one chunk per draw.  Degree-biased sampling (fused and batched drivers) and walks
must stay bit-identical to the oracle, including 300,000-candidate hub pools, collision
fallbacks and the OOM drivers."""
import numpy as np
import pytest
import torch

import paper_2009_09103_b200 as cs
from synth import instance_seeds, rmat_csr
from tests._parity import DEV, check_sample, check_walk
from tests.test_gpu_parity import hub_csr

import oracle as O

pytestmark = pytest.mark.gpu


def pair(rp, col, **kw):
    rpt = torch.as_tensor(np.asarray(rp, dtype=np.int64))
    ct = torch.as_tensor(np.asarray(col).astype(np.uint32).view(np.int32))
    G = cs.csaw_graph_create(rpt.to(DEV), ct.to(DEV), chunk_cache=True, **kw)
    assert G.info()["device_bytes"] >= 8 * (ct.numel() // 64)
    return G, O.Graph(rpt.numpy(), ct.numpy().view(np.uint32))


@pytest.fixture(scope="module")
def hubcc():
    return pair(*hub_csr())


@pytest.fixture(scope="module")
def densecc():
    g = rmat_csr(1 << 13, 1 << 20, 17)
    return pair(g.row_ptr, g.col_idx) + (g,)


@pytest.mark.parametrize("batched", [False, True])
def test_ccache_hub_sampling(hubcc, batched):
    G, og = hubcc
    if batched:
        G = cs.csaw_graph_create(torch.as_tensor(og.row_ptr).to(DEV),
                                 torch.as_tensor(og.col.view(np.int32)).to(DEV), chunk_cache=True, batched_only=True)
    seeds = np.array([0, 1, 0, 1, 5, 0, 1, 17, 299_999], dtype=np.uint32)
    check_sample(G, og, "degree", seeds, fanout=[3, 2], rng_seed=3)
    check_sample(G, og, "degree", seeds, fanout=[20, 2], rng_seed=4, a_max=2)   # collisions, fallback
    check_walk(G, og, "degree", seeds, 25, rng_seed=8)


def test_ccache_dense(densecc):
    G, og, g = densecc
    seeds = instance_seeds(g, 400, set_id=6).numpy()
    check_sample(G, og, "degree", seeds, fanout=[4, 3], rng_seed=12)
    check_walk(G, og, "degree", seeds[:128], 80, rng_seed=13)
