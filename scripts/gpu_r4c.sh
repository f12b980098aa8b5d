#!/bin/bash
# MDRW 16-slot blocks (k_mdrw_b16) vs 32-slot blocks: parity (incl. full cfg5) + time + DRAM
mkdir -p gpurun_out/r4c
O=gpurun_out/r4c
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_oom.py tests/test_gpu_streams.py -x -q -k "mdrw or oom or stream" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
for rep in 1 2; do
for v in default b32; do
  if [ $v = default ]; then unset CSAW_LIB; else export CSAW_LIB=$PWD/exp/libcsaw_$v.so; fi
  timeout 900 python bench.py --config cfg5 --in-memory --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --scan-path-steps 0 > $O/b_$v.json 2> $O/b_$v.err
  python -c "import json; d=json.loads(open('$O/b_$v.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'])"
done
done
unset CSAW_LIB
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct -k regex:k_mdrw --csv --log-file $O/ncu.csv python bench.py --config cfg5 --in-memory --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --scan-path-steps 0 > /dev/null 2>&1
grep -E "dram__bytes|time_dur|hit_rate" $O/ncu.csv | tail -4 | awk -F'","' '{print $(NF-2), $NF}'
timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q -k "cfg5_mdrw" > $O/pytest_cfg5.log 2>&1; echo "cfg5 full rc=$?"; tail -1 $O/pytest_cfg5.log
