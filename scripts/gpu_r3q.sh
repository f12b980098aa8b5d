#!/bin/bash
# weighted bucketed index (k_walk_gbw) + pipelined node2vec host copies: parity + bench lines
mkdir -p gpurun_out/r3q
O=gpurun_out/r3q
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_buckets.py tests/test_gpu_n2v_index.py tests/test_abi.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for v in buckets scan; do
  f=""; [ $v = scan ] && f="--no-walk-buckets"
  timeout 900 python bench.py --config cfg2_weight --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --scan-path-steps 0 $f > $O/bw_$v.json 2> $O/bw_$v.err
  python -c "import json; d=json.loads(open('$O/bw_$v.json').read().strip().splitlines()[-1]); c=d['detail']['cache']; print('cfg2_weight $v', d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], c['build_ms'])"
done
timeout 900 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline --scan-path-steps 0 > $O/b3.json 2> $O/b3.err
python -c "import json; d=json.loads(open('$O/b3.json').read().strip().splitlines()[-1]); print('cfg3', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'])"
timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q -k "cfg2_weight" > $O/pytest_cfg2w.log 2>&1; echo "cfg2w full rc=$?"; tail -2 $O/pytest_cfg2w.log
