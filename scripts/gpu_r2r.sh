#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in default hub256 hub4k; do
  if [ $v = default ]; then unset CSAW_LIB; else export CSAW_LIB=$PWD/exp/libcsaw_$v.so; fi
  timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r2r_$v.csv python scripts/build_n2x.py > /dev/null 2>&1
  python - $v <<'PY'
import csv, sys
v = sys.argv[1]
rows=[r for r in csv.reader(open(f'gpurun_out/r2r_{v}.csv')) if r]
hi=[i for i,r in enumerate(rows) if r[0]=='ID'][0]
h=rows[hi]; agg={}
for r in rows[hi+1:]:
    d=dict(zip(h,r))
    if d.get('Metric Name')=='gpu__time_duration.sum':
        k=d['Kernel Name'].split('(')[0]
        if 'csaw' in k: agg[k]=agg.get(k,0)+float(d['Metric Value'].replace(',',''))
print(v, {k: round(x/1e6,1) for k,x in sorted(agg.items(), key=lambda x:-x[1])[:6]})
PY
done
