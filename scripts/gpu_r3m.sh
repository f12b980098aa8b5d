#!/bin/bash
# node2vec index: division-free region arithmetic (shift / fp64 estimate) + 32x32 products; parity + bench
mkdir -p gpurun_out/r3m
O=gpurun_out/r3m
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_n2v_index.py tests/test_gpu_parity.py -x -q -k "node2vec or n2x or index" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
for rep in 1 2 3; do
  timeout 900 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --scan-path-steps 0 > $O/b.json 2> $O/b.err
  python -c "import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); print('cfg3', d['value'], d['ms_per_step'])"
done
