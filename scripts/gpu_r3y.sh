#!/bin/bash
# layer sampler at 8 blocks / SM (64-entry frontier, 256-entry visited): parity + cfg4 bench
mkdir -p gpurun_out/r3y
O=gpurun_out/r3y
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batched.py tests/test_gpu_cache.py tests/test_gpu_wix.py tests/test_gpu_ccache.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q -k "cfg4" > $O/pytest_cfg4.log 2>&1; echo "cfg4 full rc=$?"; tail -1 $O/pytest_cfg4.log
for c in cfg4_layer cfg4_ff; do
  timeout 900 python bench.py --config $c > $O/b_$c.json 2> $O/b_$c.err
  python -c "import json; d=json.loads(open('$O/b_$c.json').read().strip().splitlines()[-1]); print('$c', d['value'], d['ms_per_step'], d['roofline']['hot_ms_per_launch'], d['e2e']['value'])"
done
