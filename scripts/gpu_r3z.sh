#!/bin/bash
# node2vec index: u16 inline positions for rows of degree <= 65,536 (48 inline) vs u32 only (24)
mkdir -p gpurun_out/r3z2
O=gpurun_out/r3z2
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_n2v_index.py tests/test_gpu_parity.py -x -q -k "node2vec or n2x or index" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
for rep in 1 2; do
for v in default; do
  if [ $v = default ]; then unset CSAW_LIB; else export CSAW_LIB=$PWD/exp/libcsaw_$v.so; fi
  timeout 900 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --scan-path-steps 0 > $O/b_$v.json 2> $O/b_$v.err
  python -c "import json; d=json.loads(open('$O/b_$v.json').read().strip().splitlines()[-1]); c=d['detail']['cache']; print('$v', d['value'], d['ms_per_step'], d['roofline']['alg_bytes_per_launch'], c['build_ms'], c['graph_device_bytes'])"
done
done
unset CSAW_LIB
timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q -k "cfg3" > $O/pytest_cfg3.log 2>&1; echo "cfg3 full rc=$?"; tail -1 $O/pytest_cfg3.log
