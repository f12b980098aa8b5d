#!/bin/bash
# node2vec TMA kernel: staged records at an 80 B smem stride (conflict-free) vs 64 B (A/B) + parity
mkdir -p gpurun_out/r3l
O=gpurun_out/r3l
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_n2v_index.py tests/test_gpu_parity.py -x -q -k "node2vec or n2x or index" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
for rep in 1 2; do
for v in default s4; do
  if [ $v = default ]; then unset CSAW_LIB; else export CSAW_LIB=$PWD/exp/libcsaw_$v.so; fi
  timeout 900 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --scan-path-steps 0 > $O/b_$v.json 2> $O/b_$v.err
  python -c "import json; d=json.loads(open('$O/b_$v.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'])"
done
done
unset CSAW_LIB
timeout 900 ncu --clock-control none --set full --import-source on -k regex:k_node2vec_tma -c 1 -o $O/cfg3_tma python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --scan-path-steps 0 > /dev/null 2>&1
ncu -i $O/cfg3_tma.ncu-rep --page details --csv > $O/cfg3_tma_details.csv 2>/dev/null
ncu -i $O/cfg3_tma.ncu-rep --page raw --csv > $O/cfg3_tma_raw.csv 2>/dev/null
grep -i "bank conflict\|excessive wavefronts" $O/cfg3_tma_details.csv | cut -c1-400
find $O -name '*.ncu-rep' -size +30M -delete
