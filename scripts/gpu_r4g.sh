#!/bin/bash
# fused sampler: 2-warp blocks vs 4-warp blocks (same warps per SM)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do
for v in default f2; do
  if [ $v = default ]; then unset CSAW_LIB; else export CSAW_LIB=$PWD/exp/libcsaw_$v.so; fi
  for c in cfg4_layer cfg4_ff cfg1; do
    timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --scan-path-steps 0 > /tmp/b_${c}_$v.json 2>/dev/null
    python -c "import json; d=json.loads(open('/tmp/b_${c}_$v.json').read().strip().splitlines()[-1]); print('$c $v', d['value'], d['ms_per_step'], d['roofline']['hot_ms_per_launch'])"
  done
done
done
