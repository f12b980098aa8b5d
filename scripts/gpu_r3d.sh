#!/bin/bash
# Re-entry check of HEAD: build, smoke, the GPU suite, default bench + cfg2 / cfg5 lines
mkdir -p gpurun_out/r3d
O=gpurun_out/r3d
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 900 python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo "cfg3 rc=$?"
timeout 600 python bench.py --config cfg2 --scan-path-steps 3 > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "cfg2 rc=$?"
timeout 900 python bench.py --config cfg5 --in-memory > $O/bench_cfg5_inmem.json 2> $O/bench_cfg5_inmem.err; echo "cfg5 rc=$?"
for f in $O/bench_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline') or {}
print('$f', d.get('value'), d.get('ms_per_step'), r.get('kernel'), r.get('frac'), d.get('e2e',{}).get('value'))"; done
