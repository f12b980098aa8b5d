# MDRW fast kernel: parity + cfg5 in-memory / zero-copy bench, fast vs slow.
set -x
mkdir -p gpurun_out/mdrw
timeout 900 python -m pytest tests/test_gpu_parity.py -k "mdrw" tests/test_gpu_oom.py -x -q --timeout 600 > gpurun_out/mdrw/tests.log 2>&1; tail -15 gpurun_out/mdrw/tests.log
for mode in fast slow; do
  if [ $mode = slow ]; then export CSAW_MDRW_SLOW=1; fi
  timeout 600 python bench.py --config cfg5 --in-memory --no-cpu-baseline --no-e2e > gpurun_out/mdrw/bench_inmem_$mode.json 2> gpurun_out/mdrw/bench_inmem_$mode.err
  timeout 600 python bench.py --config cfg5 --no-cpu-baseline --no-e2e > gpurun_out/mdrw/bench_oom_$mode.json 2> gpurun_out/mdrw/bench_oom_$mode.err
  for f in inmem oom; do python -c "
import json; d=json.loads(open('gpurun_out/mdrw/bench_${f}_$mode.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$f $mode', d['value'], d['ms_per_step'], r['kernel'], r['achieved'], r['frac'])" 2>&1 | grep -v "^+"; done
done
