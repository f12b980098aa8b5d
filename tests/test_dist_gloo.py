"""Multi-process host logic of the sharded path (§5.4), world_size 2 on
gloo (CPU): instance sharding by contiguous ranges with instance_base, and the
end-of-run gather of walks / sampled subgraphs.  The per-rank "sampler" here is
the oracle (CPU), so the test checks the plumbing + the determinism contract:
the gathered sharded result equals the single-process result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2009_09103_b200.dist import gather_samples, gather_walks, shard_range
from synth import instance_seeds, rmat_csr


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_partitions_exactly():
    for n in (0, 1, 7, 64, 4000, 8192):
        for w in (1, 2, 3, 4, 8):
            rs = [shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = rmat_csr(1024, 16384, 1)
    og = O.Graph.from_torch(g)
    n = 37                                       # ragged split
    seeds = instance_seeds(g, n).numpy().astype(np.uint32)
    lo, hi = shard_range(n, rank, world)
    # walks: this rank's instances, global ids via instance_base
    paths = np.stack([O.walk(og, O.KIND_DEGREE, 20, int(seeds[i]), i, 5) for i in range(lo, hi)]) \
        if hi > lo else np.zeros((0, 21), np.uint32)
    allp = gather_walks(torch.from_numpy(paths.view(np.int32)))
    # sampling: per-instance variable-size outputs -> offsets + edge arrays
    outs = O.sample_instances(og, "degree", seeds[lo:hi], lo, 5, fanout=[2, 2], depth=2)
    offs = [0]
    for s, d, e in outs:
        offs.append(offs[-1] + s.size)
    cat = (lambda k, dt: np.concatenate([o[k] for o in outs]).astype(dt) if outs else np.zeros(0, dt))
    res = gather_samples(torch.tensor(offs, dtype=torch.int64), torch.from_numpy(cat(0, np.uint32).view(np.int32)),
                         torch.from_numpy(cat(1, np.uint32).view(np.int32)), torch.from_numpy(cat(2, np.uint8)))
    if rank == 0:
        q.put((allp.numpy(), [t.numpy() for t in res]))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_gather_equals_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    allp, (offs, src, dst, dep) = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = rmat_csr(1024, 16384, 1)
    og = O.Graph.from_torch(g)
    n = 37
    seeds = instance_seeds(g, n).numpy().astype(np.uint32)
    ref_p = np.stack([O.walk(og, O.KIND_DEGREE, 20, int(seeds[i]), i, 5) for i in range(n)])
    assert np.array_equal(allp.view(np.uint32), ref_p)
    ref = O.sample_instances(og, "degree", seeds, 0, 5, fanout=[2, 2], depth=2)
    assert offs.size == n + 1
    for i, (s, d, e) in enumerate(ref):
        a, b = int(offs[i]), int(offs[i + 1])
        assert np.array_equal(src[a:b].view(np.uint32), s)
        assert np.array_equal(dst[a:b].view(np.uint32), d)
        assert np.array_equal(dep[a:b], e)
