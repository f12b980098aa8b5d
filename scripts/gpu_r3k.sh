#!/bin/bash
# DRAM bytes per random 64 B record fetched by cp.async.bulk (TMA) vs vector loads
mkdir -p gpurun_out/r3k
O=gpurun_out/r3k
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rrt scripts/random_roofline_tma.cu && /tmp/rrt 16 > $O/tma.txt
timeout 900 ncu --clock-control none --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read.sum --csv --log-file $O/tma_ncu.csv /tmp/rrt 16 > /dev/null 2>&1
cat $O/tma.txt
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/r3k/tma_ncu.csv")))
hdr = None
by = {}
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r)); by.setdefault((d["ID"], d["Kernel Name"][:60]), {})[d["Metric Name"]] = d["Metric Value"]
for (i, k), m in by.items():
    t = float(m["gpu__time_duration.sum"].replace(",", "")); b = float(m["dram__bytes_read.sum"].replace(",", ""))
    print(i, k, "dram GB/s %.0f" % (b / t), "sectors", m.get("lts__t_sectors_srcunit_tex_op_read.sum"), "req", m.get("lts__t_requests_srcunit_tex_op_read.sum"))
PY
