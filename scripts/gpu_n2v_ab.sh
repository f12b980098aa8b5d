set -x
mkdir -p gpurun_out/n2v
timeout 900 python bench.py --config cfg3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-cache > gpurun_out/n2v/bench_old.json 2> gpurun_out/n2v/bench_old.err
python -c "
import json; d=json.loads(open('gpurun_out/n2v/bench_old.json').read().strip().splitlines()[-1]); r=d['roofline']
print('old', d['value'], d['ms_per_step'], r['kernel'], r['achieved'], r['frac'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_node2vec_tri -c 1 -o gpurun_out/n2v/cfg3_tri python scripts/prof_n2v.py 40 cache > gpurun_out/n2v/ncu.log 2>&1
ncu -i gpurun_out/n2v/cfg3_tri.ncu-rep --page raw --csv > gpurun_out/n2v/cfg3_tri_raw.csv 2>/dev/null
ncu -i gpurun_out/n2v/cfg3_tri.ncu-rep --page details --csv > gpurun_out/n2v/cfg3_tri_details.csv 2>/dev/null
ncu -i gpurun_out/n2v/cfg3_tri.ncu-rep --page source --csv > gpurun_out/n2v/cfg3_tri_source.csv 2>/dev/null
tail -3 gpurun_out/n2v/ncu.log
