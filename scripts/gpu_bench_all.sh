# Bench lines for every config (default flags: cpu_baseline + e2e), into gpurun_out/final/.
set -x
mkdir -p gpurun_out/final
timeout 600 python bench.py > gpurun_out/final/bench_cfg2.json 2> gpurun_out/final/bench_cfg2.err
for c in cfg1 cfg3 cfg4_layer cfg4_ff; do
  timeout 900 python bench.py --config $c > gpurun_out/final/bench_$c.json 2> gpurun_out/final/bench_$c.err
done
timeout 900 python bench.py --config cfg5 --in-memory > gpurun_out/final/bench_cfg5_inmem.json 2> gpurun_out/final/bench_cfg5_inmem.err
timeout 900 python bench.py --config cfg5 --oom-variant zerocopy > gpurun_out/final/bench_cfg5_zerocopy.json 2> gpurun_out/final/bench_cfg5_zerocopy.err
timeout 600 python bench.py --impl reference > gpurun_out/final/bench_reference_cfg2.json 2> gpurun_out/final/bench_reference_cfg2.err
for f in gpurun_out/final/bench_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline') or {}
print('$f', d.get('value'), d.get('ms_per_step'), r.get('kernel'), r.get('frac'), (d.get('detail') or {}).get('step_ms'))"; done
