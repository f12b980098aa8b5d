"""NEXT-3 Table-1 walk variants on the GPU (MH, restart, jump) vs the oracle, bit-exact."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2009_09103_b200 as cs
from synth import instance_seeds, rmat_csr
from tests._parity import DEV, graph_pair, u32

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
