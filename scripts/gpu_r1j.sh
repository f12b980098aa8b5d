set -x
timeout 300 python scripts/prof_n2v.py 40 > gpurun_out/n2v_rev.log 2>&1; tail -n 2 gpurun_out/n2v_rev.log
for i in 1 2; do
timeout 600 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2_meta$i.json 2>&1; tail -c 200 gpurun_out/bench_cfg2_meta$i.json | head -c 120; echo
CSAW_NO_WALK_META=1 timeout 600 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2_nometa$i.json 2>&1; tail -c 200 gpurun_out/bench_cfg2_nometa$i.json | head -c 120; echo
done
for f in gpurun_out/bench_cfg2_meta1.json gpurun_out/bench_cfg2_nometa1.json gpurun_out/bench_cfg2_meta2.json gpurun_out/bench_cfg2_nometa2.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'])"; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q --timeout 600 -k "node2vec or cfg3 or hub" > gpurun_out/gpu_j.log 2>&1; tail -3 gpurun_out/gpu_j.log
