# node2vec triangle-count kernel: parity (small + full cfg3) and cfg3 bench (+ optional ncu of a 1/40 subset).
set -x
mkdir -p gpurun_out/n2v
timeout 900 python -m pytest tests/test_gpu_n2v_tri.py -x -q --timeout 600 > gpurun_out/n2v/tests.log 2>&1; tail -15 gpurun_out/n2v/tests.log
timeout 1200 python -m pytest tests/test_gpu_configs.py -k "cfg3" -x -q --timeout 1100 > gpurun_out/n2v/tests_full.log 2>&1; tail -5 gpurun_out/n2v/tests_full.log
timeout 900 python bench.py --config cfg3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/n2v/bench_tri.json 2> gpurun_out/n2v/bench_tri.err
python -c "
import json; d=json.loads(open('gpurun_out/n2v/bench_tri.json').read().strip().splitlines()[-1]); r=d['roofline']
print('tri', d['value'], d['ms_per_step'], r['kernel'], r['achieved'], r['frac'], d['detail']['cache_build_ms'], d['detail'].get('neighbours_scanned_per_step'))"
if [ -n "$NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_node2vec_tri -c 1 -o gpurun_out/n2v/cfg3_tri python scripts/prof_n2v.py 40 cache > gpurun_out/n2v/ncu.log 2>&1
ncu -i gpurun_out/n2v/cfg3_tri.ncu-rep --page raw --csv > gpurun_out/n2v/cfg3_tri_raw.csv 2>/dev/null
ncu -i gpurun_out/n2v/cfg3_tri.ncu-rep --page details --csv > gpurun_out/n2v/cfg3_tri_details.csv 2>/dev/null
fi
