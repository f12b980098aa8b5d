#!/bin/bash
# MDRW 16 B slot records by default: parity (incl. OOM zero-copy + full cfg5) + bench lines
mkdir -p gpurun_out/r3u
O=gpurun_out/r3u
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_oom.py tests/test_gpu_streams.py -x -q -k "mdrw or oom or stream" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q -k "cfg5_mdrw" > $O/pytest_cfg5.log 2>&1; echo "cfg5 full rc=$?"; tail -1 $O/pytest_cfg5.log
timeout 900 python bench.py --config cfg5 --in-memory > $O/b5.json 2> $O/b5.err
python -c "import json; d=json.loads(open('$O/b5.json').read().strip().splitlines()[-1]); print('cfg5', d['value'], d['ms_per_step'], d['e2e']['value'])"
timeout 900 python bench.py --config cfg5 --oom-variant zerocopy --steps 3 --warmup 2 --no-cpu-baseline > $O/b5zc.json 2> $O/b5zc.err
python -c "import json; d=json.loads(open('$O/b5zc.json').read().strip().splitlines()[-1]); print('cfg5 zc', d['value'], d['ms_per_step'])"
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct -k regex:k_mdrw --csv --log-file $O/ncu.csv python bench.py --config cfg5 --in-memory --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --scan-path-steps 0 > /dev/null 2>&1
grep -E "dram__bytes|time_dur|hit_rate" $O/ncu.csv | tail -4 | awk -F'","' '{print $(NF-2), $NF}'
