#!/bin/bash
# .L2::64B prefetch size on the random single-word loads (node2vec probes, MDRW entry + metadata): A/B + parity
mkdir -p gpurun_out/r3h
O=gpurun_out/r3h
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_n2v_tri.py -x -q -k "mdrw or node2vec" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
for rep in 1 2; do
for v in default ld128; do
  if [ $v = default ]; then unset CSAW_LIB; else export CSAW_LIB=$PWD/exp/libcsaw_$v.so; fi
  for c in cfg3 cfg5; do
    timeout 900 python bench.py --config $c --in-memory --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --scan-path-steps 0 > $O/b_${c}_$v.json 2> $O/b_${c}_$v.err
    python -c "import json; d=json.loads(open('$O/b_${c}_$v.json').read().strip().splitlines()[-1]); print('$c $v', d['value'], d['ms_per_step'])"
  done
done
done
unset CSAW_LIB
for c in cfg3 cfg5; do
  k=k_node2vec_tma; [ $c = cfg5 ] && k=k_mdrw_fast
  for v in default ld128; do
    if [ $v = default ]; then unset CSAW_LIB; else export CSAW_LIB=$PWD/exp/libcsaw_$v.so; fi
    timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct -k regex:$k --csv --log-file $O/ncu_${c}_$v.csv python bench.py --config $c --in-memory --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --scan-path-steps 0 > /dev/null 2>&1
    echo "$c $v"; grep -E "dram__bytes|time_dur|hit_rate" $O/ncu_${c}_$v.csv | tail -4 | awk -F'","' '{print $(NF-2), $NF}'
  done
done
