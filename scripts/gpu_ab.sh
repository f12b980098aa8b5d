# Generic A/B: CONFIG=<cfg> VARIANTS="name:ENV=1,ENV2=0 ..." bash scripts/gpu_ab.sh
set -x
mkdir -p gpurun_out/ab
[ -n "$TESTS" ] && { timeout 900 python -m pytest $TESTS -x -q --timeout 600 > gpurun_out/ab/tests.log 2>&1; tail -5 gpurun_out/ab/tests.log; }
for v in $VARIANTS; do
  name=${v%%:*}; envs=${v#*:}
  ( [ "$envs" != "-" ] && export $(echo $envs | tr ',' ' '); timeout 900 python bench.py --config ${CONFIG:-cfg2} ${BENCH_ARGS:---no-cpu-baseline --no-e2e} > gpurun_out/ab/$name.json 2> gpurun_out/ab/$name.err )
  python -c "
import json; d=json.loads(open('gpurun_out/ab/$name.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$name', d['value'], d['ms_per_step'], r['kernel'], r['frac'], d['detail'].get('cache_build_ms'))" 2>&1 | grep -v "^+"
done
