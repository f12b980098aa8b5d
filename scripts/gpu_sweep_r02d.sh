#!/bin/bash
# r02d: the default line (cfg3) after the last node2vec-index change: ncu (launch list + --set full) then the bench line
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
P=gpurun_out/prof4; B=gpurun_out/final4
mkdir -p $P $B
NCU="ncu --clock-control none --nvtx --nvtx-include csaw_step/"
Q="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-zerocopy --scan-path-steps 0"
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file $P/cfg3_launches.csv $Q --config cfg3 > /dev/null 2>&1
timeout 1200 $NCU --set full --import-source on -k regex:k_node2vec_tma -c 1 -o $P/cfg3 $Q --config cfg3 > /dev/null 2>&1
ncu -i $P/cfg3.ncu-rep --page raw --csv > $P/cfg3_raw.csv 2>/dev/null
ncu -i $P/cfg3.ncu-rep --page details --csv > $P/cfg3_details.csv 2>/dev/null
ncu -i $P/cfg3.ncu-rep --page source --csv > $P/cfg3_source.csv 2>/dev/null
find $P -name "*.ncu-rep" -delete
python scripts/ncu_summary.py $P r02d > $P/ncu_summary.md 2> $P/ncu_summary.err; echo "summary rc=$?"
cp profiles/ncu_traffic.json $P/ncu_traffic.json
timeout 900 python bench.py > $B/bench_cfg3.json 2> $B/bench_cfg3.err; echo "cfg3 rc=$?"
timeout 900 python bench.py --impl reference > $B/bench_reference_cfg3.json 2> $B/bench_reference_cfg3.err; echo "ref rc=$?"
python -c "
import json; d=json.loads(open('$B/bench_cfg3.json').read().strip().splitlines()[-1]); r=d['roofline']
print(d['value'], d['ms_per_step'], r['frac'], r['f_dram'], r.get('dram_frac_of_random_line_ceiling'), d['e2e']['value'], d['detail']['cache']['one_call_seps'])"
du -sh $P
