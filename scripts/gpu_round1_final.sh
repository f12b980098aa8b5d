# Full GPU test suite, bench lines for every config, then the ncu evidence.
set -x
mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 --durations=10 > gpurun_out/final/gpu_tests.log 2>&1; tail -20 gpurun_out/final/gpu_tests.log
timeout 600 python bench.py > gpurun_out/final/bench_cfg2.json 2> gpurun_out/final/bench_cfg2.err
for c in cfg1 cfg3 cfg4_layer cfg4_ff; do
  timeout 900 python bench.py --config $c > gpurun_out/final/bench_$c.json 2> gpurun_out/final/bench_$c.err
done
timeout 900 python bench.py --config cfg5 --in-memory > gpurun_out/final/bench_cfg5_inmem.json 2> gpurun_out/final/bench_cfg5_inmem.err
timeout 600 python bench.py --impl reference > gpurun_out/final/bench_reference_cfg2.json 2> gpurun_out/final/bench_reference_cfg2.err
for f in gpurun_out/final/bench_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline') or {}
print('$f', d.get('value'), d.get('ms_per_step'), r.get('kernel'), r.get('frac'))"; done
bash scripts/gpu_prof_all.sh > gpurun_out/final/prof.log 2>&1
