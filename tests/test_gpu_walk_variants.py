"""NEXT-3 Table-1 variants on the GPU (MH, restart, jump walks; snowball sampling) vs the oracle, bit-exact."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2009_09103_b200 as cs
from synth import instance_seeds, rmat_csr
from tests._parity import DEV, check_sample, graph_pair, u32

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def medium():
    g = rmat_csr(1 << 15, 1 << 19, 7, device=DEV).to("cpu")
    G, og = graph_pair(g.row_ptr, g.col_idx)
    return G, og, g


@pytest.mark.parametrize("kind,pr", [("mh", 0.0), ("restart", 0.15), ("jump", 0.2), ("restart", 0.0)])
def test_walk_variants_parity(medium, kind, pr):
    G, og, g = medium
    seeds = instance_seeds(g, 200, set_id=3).numpy()
    st = torch.as_tensor(seeds.astype(np.uint32).view(np.int32)).to(DEV)
    path = u32(cs.csaw_walk(G, cs.make_bias(kind, pf=pr), st, 150, rng_seed=8, instance_base=11))
    k = {"mh": O.KIND_MH, "restart": O.KIND_RESTART, "jump": O.KIND_JUMP}[kind]
    for w in range(len(seeds)):
        ref = O.walk_variant(og, k, 150, int(seeds[w]), 11 + w, 8, pr)
        assert np.array_equal(path[w], ref), w


def test_walk_variant_errors(medium):
    G, og, g = medium
    s = instance_seeds(g, 4).to(DEV)
    with pytest.raises(cs.CsawError):
        cs.csaw_walk(G, cs.make_bias("restart", pf=1.5), s, 10)
    with pytest.raises(cs.CsawError):
        cs.csaw_sample(G, cs.make_bias("mh"), s, fanout=[2])


@pytest.mark.parametrize("depth", [1, 2, 3])
def test_snowball_parity_small(depth):
    """NEXT-3 snowball (select-all to depth) on the config-1 graph, every instance vs the oracle."""
    g = rmat_csr(1024, 16384, 1)
    G, og = graph_pair(g.row_ptr, g.col_idx)
    seeds = instance_seeds(g, 64).numpy()
    _, total = check_sample(G, og, "snowball", seeds, depth=depth, rng_seed=2)
    assert total > 0


def test_snowball_parity_medium(medium):
    G, og, g = medium
    seeds = instance_seeds(g, 24, set_id=5).numpy()
    _, total = check_sample(G, og, "snowball", seeds, depth=2, rng_seed=1, instance_base=3)
    assert total > 24
    with pytest.raises(cs.CsawError):
        cs.csaw_walk(G, cs.make_bias("snowball"), torch.as_tensor(seeds[:2].view(np.int32)).to(DEV), 5)
