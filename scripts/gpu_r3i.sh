#!/bin/bash
# MDRW next-vertex records (16 B, CSAW_GRAPH_NEXT_RECORD) vs 8 B metadata + col: parity (incl. full cfg5) + time + DRAM
mkdir -p gpurun_out/r3i
O=gpurun_out/r3i
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "mdrw" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
timeout 1200 python -m pytest tests/test_gpu_configs.py -x -q -k "cfg5_mdrw" > $O/pytest_cfg5.log 2>&1; echo "pytest cfg5 rc=$?"; tail -1 $O/pytest_cfg5.log
for rep in 1 2; do
for v in record meta; do
  f=""; [ $v = meta ] && f="--next-meta"
  timeout 900 python bench.py --config cfg5 --in-memory --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --scan-path-steps 0 $f > $O/b_$v.json 2> $O/b_$v.err
  python -c "import json; d=json.loads(open('$O/b_$v.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], d['detail']['cache'].get('build_ms'))"
done
done
for v in record meta; do
  f=""; [ $v = meta ] && f="--next-meta"
  timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct -k regex:k_mdrw --csv --log-file $O/ncu_$v.csv python bench.py --config cfg5 --in-memory --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --scan-path-steps 0 $f > /dev/null 2>&1
  echo "$v"; grep -E "dram__bytes|time_dur|hit_rate" $O/ncu_$v.csv | tail -4 | awk -F'","' '{print $(NF-2), $NF}'
done
