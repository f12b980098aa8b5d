"""Loaders for tests/golden fixtures (each file carries its citation)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def philox_kats():
    out = []
    for line in open(os.path.join(GOLDEN, "philox_kat.txt")):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        lhs, rhs = line.split("->")
        w = [int(x, 16) for x in lhs.split()]
        o = [int(x, 16) for x in rhs.split()]
        out.append((w[:4], w[4:6], o))
    return out


def paper_examples():
    with open(os.path.join(GOLDEN, "paper_examples.json")) as f:
        return json.load(f)


def gtoy():
    rows = {}
    for line in open(os.path.join(GOLDEN, "gtoy.txt")):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        name, *vals = line.split()
        rows[name] = [int(v) for v in vals]
    return np.array(rows["row_ptr"], np.int64), np.array(rows["col_idx"], np.uint32)
