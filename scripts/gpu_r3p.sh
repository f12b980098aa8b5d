#!/bin/bash
# bucketed degree-walk index (k_walk_gb): parity (small + full cfg2) + bench vs vertex heads + ncu metrics
mkdir -p gpurun_out/r3p
O=gpurun_out/r3p
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_buckets.py tests/test_abi.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for rep in 1 2; do
for v in buckets heads; do
  f=""; [ $v = buckets ] && f="--walk-buckets"
  timeout 900 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --scan-path-steps 0 $f > $O/b_$v.json 2> $O/b_$v.err
  python -c "import json; d=json.loads(open('$O/b_$v.json').read().strip().splitlines()[-1]); c=d['detail']['cache']; print('$v', d['value'], d['ms_per_step'], d['roofline']['kernel'], c['build_ms'], c['graph_device_bytes'])"
done
done
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct -k regex:k_walk_gb --csv --log-file $O/ncu.csv python bench.py --config cfg2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --scan-path-steps 0 --walk-buckets > /dev/null 2>&1
grep -E "dram__bytes|time_dur|hit_rate" $O/ncu.csv | tail -4 | awk -F'","' '{print $(NF-2), $NF}'
timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q -k "cfg2_degree" > $O/pytest_cfg2.log 2>&1; echo "cfg2 full rc=$?"; tail -2 $O/pytest_cfg2.log
