"""NEXT-4(i): the out-of-memory partition store in a peer GPU's HBM (CSAW_GRAPH_OOM_PEER_STORE).

Partition loads are then device-to-device copies (NVLink between GPUs) and zero-copy kernels
read the store in place; the §5 planner and every output are unchanged (R7, R22).  On one GPU
the store sits on the same device (store_device == device), which exercises the same code
path; with two or more GPUs the store is placed on the next GPU as well.
"""
import numpy as np
import pytest
import torch

import paper_2009_09103_b200 as cs
from synth import instance_seeds, mdrw_seeds, rmat_csr
from tests._parity import DEV
from tests.test_gpu_oom import budget_for

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def medium():
    return rmat_csr(1 << 15, 1 << 19, 7, device=DEV).to("cpu")


def store_devices():
    n = torch.cuda.device_count()
    return [0] + ([1] if n > 1 else [])


@pytest.mark.parametrize("store", store_devices())
@pytest.mark.parametrize("zerocopy", [False, True])
def test_peer_store_mdrw_and_walks_equal_in_memory(medium, store, zerocopy):
    g = medium
    n, m, L = 64, 200, 300
    seeds = mdrw_seeds(g, n, m).to(DEV)
    Gm = cs.csaw_graph_create(g.row_ptr.to(DEV), g.col_idx.to(DEV))
    P, R = 4, 2
    kw = dict(budget_bytes=budget_for(g, P, R, n, m) + (64 << 20 if zerocopy else 0), num_partitions=P,
              max_resident=1 if zerocopy else R, num_streams=2, zerocopy=zerocopy, store_device=store)
    Gp = cs.csaw_graph_create(g.row_ptr, g.col_idx, **kw)
    Gh = cs.csaw_graph_create(g.row_ptr, g.col_idx, **{**kw, "store_device": None})   # the paper's host store
    assert Gp.info()["oom_mode"] == 1
    for G in (Gp, Gh):
        got = cs.csaw_walk(G, cs.make_bias("mdrw"), seeds, L, rng_seed=5)
        assert torch.equal(cs.csaw_walk(Gm, cs.make_bias("mdrw"), seeds, L, rng_seed=5), got)
    st = cs.csaw_stats(Gp)
    if not zerocopy:
        assert st["partition_loads"] > R and st["h2d_bytes"] > 0   # partitions were copied from the store
    s1 = instance_seeds(g, 200).to(DEV)
    for kind in ("degree", "uniform"):
        a = cs.csaw_walk(Gm, kind, s1, 50, rng_seed=3)
        b = cs.csaw_walk(Gp, kind, s1, 50, rng_seed=3)
        assert torch.equal(a, b), kind
    offs_m, src_m, dst_m, dep_m = cs.csaw_sample(Gm, "degree", s1, fanout=[3, 2], rng_seed=4)
    offs_p, src_p, dst_p, dep_p = cs.csaw_sample(Gp, "degree", s1, fanout=[3, 2], rng_seed=4)
    assert torch.equal(offs_m, offs_p) and torch.equal(src_m, src_p) and torch.equal(dst_m, dst_p)
    for G in (Gm, Gp, Gh):
        G.close()


def test_peer_store_bad_device(medium):
    g = medium
    with pytest.raises(cs.CsawError) as e:
        cs.csaw_graph_create(g.row_ptr, g.col_idx, budget_bytes=1 << 30, store_device=64)
    assert e.value.status == 1
