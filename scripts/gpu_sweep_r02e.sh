#!/bin/bash
# Round-2 final sweep (all configs, final code): ncu first (launch lists + one --set full capture per hot kernel ->
# profiles/ncu_traffic.json, which bench.py reports), then the bench line of every config.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
P=gpurun_out/prof5; B=gpurun_out/final5
mkdir -p $P $B
NCU="ncu --clock-control none --nvtx --nvtx-include csaw_step/"
Q="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-zerocopy --scan-path-steps 0"
run() {  # name kernel-regex args
  n=$1; kre=$2; shift 2
  timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file $P/${n}_launches.csv $Q "$@" > /dev/null 2>&1
  timeout 1200 $NCU --set full --import-source on -k regex:$kre -c 1 -o $P/${n} $Q "$@" > /dev/null 2>&1
  ncu -i $P/${n}.ncu-rep --page raw --csv > $P/${n}_raw.csv 2>/dev/null
  ncu -i $P/${n}.ncu-rep --page details --csv > $P/${n}_details.csv 2>/dev/null
  echo "ncu $n done"
}
run cfg3 k_node2vec_tma --config cfg3
run cfg2 k_walk_gb --config cfg2
run cfg2_stream k_walk_vscan --config cfg2 --no-cache
run cfg2_weight k_walk_gbw --config cfg2_weight
run cfg1 k_sample_fused --config cfg1
run cfg4_layer k_sample_fused --config cfg4_layer
run cfg4_ff k_sample_fused --config cfg4_ff
run cfg5_inmem k_mdrw_fast --config cfg5 --in-memory
find $P -name "*.ncu-rep" -delete
python scripts/ncu_summary.py $P r02e > $P/ncu_summary.md 2> $P/ncu_summary.err; echo "summary rc=$?"
cp profiles/ncu_traffic.json $P/ncu_traffic.json
timeout 900 python bench.py > $B/bench_cfg3.json 2> $B/bench_cfg3.err; echo "cfg3 rc=$?"
timeout 600 python bench.py --config cfg2 --scan-path-steps 3 > $B/bench_cfg2.json 2> $B/bench_cfg2.err; echo "cfg2 rc=$?"
timeout 600 python bench.py --config cfg2_weight > $B/bench_cfg2_weight.json 2> $B/bench_cfg2_weight.err; echo "cfg2w rc=$?"
for c in cfg1 cfg4_layer cfg4_ff; do
  timeout 900 python bench.py --config $c > $B/bench_$c.json 2> $B/bench_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --config cfg5 --in-memory > $B/bench_cfg5_inmem.json 2> $B/bench_cfg5_inmem.err; echo "cfg5 inmem rc=$?"
timeout 900 python bench.py --config cfg5 --oom-variant zerocopy > $B/bench_cfg5_zerocopy.json 2> $B/bench_cfg5_zerocopy.err; echo "cfg5 zc rc=$?"
timeout 900 python bench.py --config cfg5 --oom-store peer --steps 3 --warmup 1 --no-zerocopy > $B/bench_cfg5_oom_peer.json 2> $B/bench_cfg5_oom_peer.err; echo "cfg5 peer rc=$?"
timeout 900 python bench.py --config cfg5_ns --steps 3 --warmup 2 > $B/bench_cfg5_ns.json 2> $B/bench_cfg5_ns.err; echo "cfg5_ns rc=$?"
timeout 900 python bench.py --impl reference > $B/bench_reference_cfg3.json 2> $B/bench_reference_cfg3.err; echo "ref rc=$?"
for f in $B/bench_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline') or {}
print('$f', d.get('value'), d.get('ms_per_step'), r.get('kernel'), r.get('frac'), r.get('f_dram'), (d.get('e2e') or {}).get('value'))"; done
