#!/bin/bash
mkdir -p gpurun_out/r3v
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python scripts/prof_n2x_build.py; python scripts/prof_n2x_build.py
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r3v/build_launches.csv python scripts/prof_n2x_build.py > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/r3v/build_launches.csv")))
h = None; agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID": h = r; continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            k = d["Kernel Name"][:60]; agg.setdefault(k, [0, 0.0]); agg[k][0] += 1; agg[k][1] += float(d["Metric Value"].replace(",", "")) / 1e6
for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:15]:
    print(f"{ms:9.2f} ms  x{n:4d}  {k}")
PY
