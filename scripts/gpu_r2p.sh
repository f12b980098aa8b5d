#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r2p_build_ll.csv python scripts/build_n2x.py > gpurun_out/r2p.log 2>&1; echo "rc=$?"
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/r2p_build_ll.csv')) if r]
hi=[i for i,r in enumerate(rows) if r[0]=='ID'][0]
h=rows[hi]
agg={}
for r in rows[hi+1:]:
    d=dict(zip(h,r))
    if d.get('Metric Name')=='gpu__time_duration.sum':
        k=d['Kernel Name'].split('(')[0]; agg[k]=agg.get(k,0)+float(d['Metric Value'].replace(',',''))
for k,v in sorted(agg.items(), key=lambda x:-x[1])[:12]: print(f"{v/1e6:10.2f} ms  {k}")
PY
