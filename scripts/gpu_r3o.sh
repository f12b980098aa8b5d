#!/bin/bash
# node2vec index: 128 B records with 24 inline values (default) vs 64 B / 8 (N2X_P=8): parity + bench + build time
mkdir -p gpurun_out/r3o
O=gpurun_out/r3o
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_n2v_index.py tests/test_gpu_parity.py tests/test_gpu_n2v_tri.py -x -q -k "node2vec or n2x or index" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
for rep in 1 2; do
for v in default p8; do
  if [ $v = default ]; then unset CSAW_LIB; else export CSAW_LIB=$PWD/exp/libcsaw_$v.so; fi
  timeout 900 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --scan-path-steps 0 > $O/b_$v.json 2> $O/b_$v.err
  python -c "import json; d=json.loads(open('$O/b_$v.json').read().strip().splitlines()[-1]); c=d['detail']['cache']; print('$v', d['value'], d['ms_per_step'], c['build_ms'], c['graph_device_bytes'], d['roofline']['alg_bytes_per_launch'])"
done
done
unset CSAW_LIB
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct -k regex:k_node2vec_tma --csv --log-file $O/ncu.csv python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --scan-path-steps 0 > /dev/null 2>&1
grep -E "dram__bytes|time_dur|hit_rate" $O/ncu.csv | tail -4 | awk -F'","' '{print $(NF-2), $NF}'
