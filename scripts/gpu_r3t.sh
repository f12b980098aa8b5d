#!/bin/bash
# A/B: MDRW 16 B slot records (alt) vs packed; cfg2 bench without the walk index / heads (buckets only)
mkdir -p gpurun_out/r3t
O=gpurun_out/r3t
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
for rep in 1 2; do
for v in packed alt; do
  f=""; [ $v = alt ] && f="--mdrw-alt-records"
  timeout 900 python bench.py --config cfg5 --in-memory --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --scan-path-steps 0 $f > $O/b5_$v.json 2> $O/b5_$v.err
  python -c "import json; d=json.loads(open('$O/b5_$v.json').read().strip().splitlines()[-1]); print('cfg5 $v', d['value'], d['ms_per_step'])"
done
done
timeout 900 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --scan-path-steps 0 > $O/b2.json 2> $O/b2.err
python -c "import json; d=json.loads(open('$O/b2.json').read().strip().splitlines()[-1]); c=d['detail']['cache']; print('cfg2', d['value'], d['ms_per_step'], c['build_ms'], c['graph_device_bytes'], c['one_call_seps'], d['e2e']['value'])"
