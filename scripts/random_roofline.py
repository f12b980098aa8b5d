"""Random-access DRAM roofline on this GPU: gathers of independent G-byte records at random
offsets from an array far larger than L2 (the access pattern of the node2vec index and MDRW
kernels), timed with CUDA events.  torch.index_select does the gathering (a measurement, not
the product path).  Prints GB/s of requested bytes for G = 32, 64, 128, 512 B."""
import json
import sys

import torch

dev = torch.device("cuda:0")
nbytes = int(float(sys.argv[1]) * 2**30) if len(sys.argv) > 1 else 32 << 30
res = {}
for G in (32, 64, 128, 512):
    cols = G // 4
    rows = nbytes // G
    a = torch.empty((rows, cols), dtype=torch.int32, device=dev)
    n = 1 << 25
    idx = torch.randint(0, rows, (n,), device=dev)
    out = torch.empty((n, cols), dtype=torch.int32, device=dev)
    torch.index_select(a, 0, idx, out=out)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.index_select(a, 0, idx, out=out)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, n * G / (e0.elapsed_time(e1) / 1e3) / 1e9)
    res[f"{G}B"] = best
    del a, out, idx
    torch.cuda.empty_cache()
print(json.dumps({"random_gather_gbs": res, "array_bytes": nbytes,
                  "what": "index_select of G-byte rows at uniform random row indices, best of 5 (requested bytes / time; "
                          "the writes of the gathered rows are not counted)"}))
