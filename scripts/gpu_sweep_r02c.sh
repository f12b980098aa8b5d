#!/bin/bash
# r02c: ncu + bench lines for the kernels changed after the r02b sweep (k_walk_gbw, k_mdrw_fast 16 B records)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
P=gpurun_out/prof3; B=gpurun_out/final3
mkdir -p $P $B
cp profiles/ncu_traffic.json $P/ncu_traffic_before.json
NCU="ncu --clock-control none --nvtx --nvtx-include csaw_step/"
Q="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-zerocopy --scan-path-steps 0"
run() {
  n=$1; kre=$2; shift 2
  timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file $P/${n}_launches.csv $Q "$@" > /dev/null 2>&1
  timeout 1200 $NCU --set full --import-source on -k regex:$kre -c 1 -o $P/${n} $Q "$@" > /dev/null 2>&1
  ncu -i $P/${n}.ncu-rep --page raw --csv > $P/${n}_raw.csv 2>/dev/null
  ncu -i $P/${n}.ncu-rep --page details --csv > $P/${n}_details.csv 2>/dev/null
  echo "ncu $n done"
}
run cfg2_weight k_walk_gbw --config cfg2_weight
run cfg5_inmem k_mdrw_fast --config cfg5 --in-memory
find $P -name "*.ncu-rep" -delete
python scripts/ncu_summary.py $P r02c > $P/ncu_summary.md 2> $P/ncu_summary.err; echo "summary rc=$?"
cp profiles/ncu_traffic.json $P/ncu_traffic.json
timeout 900 python bench.py --config cfg2_weight --scan-path-steps 2 > $B/bench_cfg2_weight.json 2> $B/bench_cfg2_weight.err; echo "cfg2w rc=$?"
timeout 900 python bench.py --config cfg5 --in-memory > $B/bench_cfg5_inmem.json 2> $B/bench_cfg5_inmem.err; echo "cfg5 rc=$?"
for f in $B/bench_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline') or {}
print('$f', d.get('value'), d.get('ms_per_step'), r.get('kernel'), r.get('frac'), r.get('f_dram'), (d.get('e2e') or {}).get('value'))"; done
