#!/bin/bash
# MDRW slot degrees in shared memory (k_mdrw_sdeg) vs slot records in memory (k_mdrw_fast): parity, time, DRAM
mkdir -p gpurun_out/r3e
O=gpurun_out/r3e
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_oom.py tests/test_gpu_streams.py -x -q -k "mdrw or oom or stream" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
for v in sdeg global; do
  f=""; [ $v = global ] && f="--mdrw-global-pool"
  timeout 600 python bench.py --config cfg5 --in-memory --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --scan-path-steps 0 $f > $O/bench_$v.json 2> $O/bench_$v.err
  python -c "import json; d=json.loads(open('$O/bench_$v.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], d['roofline'].get('kernel'))"
  timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct -k regex:k_mdrw --csv --log-file $O/ncu_$v.csv python bench.py --config cfg5 --in-memory --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --scan-path-steps 0 $f > /dev/null 2>&1
  grep -E "dram__bytes|time_dur|hit_rate" $O/ncu_$v.csv | tail -4
done
timeout 900 python bench.py --config cfg5 --oom-variant zerocopy --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --scan-path-steps 0 > $O/bench_zc.json 2> $O/bench_zc.err
python -c "import json; d=json.loads(open('$O/bench_zc.json').read().strip().splitlines()[-1]); print('zc', d['value'], d['ms_per_step'])"
