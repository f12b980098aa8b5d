#!/bin/bash
# node2vec index build: inline members written by the count pass, list pass only for C > 24
mkdir -p gpurun_out/r3w
O=gpurun_out/r3w
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_n2v_index.py tests/test_gpu_parity.py -x -q -k "node2vec or n2x or index" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
python scripts/prof_n2x_build.py
timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q -k "cfg3" > $O/pytest_cfg3.log 2>&1; echo "cfg3 full rc=$?"; tail -1 $O/pytest_cfg3.log
timeout 900 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline --scan-path-steps 0 > $O/b3.json 2> $O/b3.err
python -c "import json; d=json.loads(open('$O/b3.json').read().strip().splitlines()[-1]); c=d['detail']['cache']; print('cfg3', d['value'], d['ms_per_step'], c['build_ms'], c['one_call_seps'], d['e2e']['value'])"
