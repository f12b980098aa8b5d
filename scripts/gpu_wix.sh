# Narrow walk index: parity + cfg2 A/B over leaf fanouts, next-vertex metadata, and the u64 index (leaf 0).
set -x
mkdir -p gpurun_out/wix
timeout 900 python -m pytest tests/test_gpu_wix.py tests/test_gpu_cache.py -x -q --timeout 600 > gpurun_out/wix/tests.log 2>&1; tail -15 gpurun_out/wix/tests.log
for v in ${VARIANTS:-0:8 64:32 64:8 32:8 128:8 64:16}; do
  leaf=${v%%:*}; meta=${v##*:}
  CSAW_WIX_LEAF=$leaf CSAW_WIX_GROUP=$meta timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/wix/bench_${leaf}_$meta.json 2> gpurun_out/wix/bench_${leaf}_$meta.err
  python -c "
import json; d=json.loads(open('gpurun_out/wix/bench_${leaf}_$meta.json').read().strip().splitlines()[-1]); r=d['roofline']
print('leaf $leaf group $meta', d['value'], d['ms_per_step'], r['kernel'], r['achieved'], r['frac'], d['detail']['cache_build_ms'])" 2>&1 | grep -v "^+"
done
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_walk_wix -c 1 -o gpurun_out/wix/cfg2_wix python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/wix/ncu.log 2>&1
  ncu -i gpurun_out/wix/cfg2_wix.ncu-rep --page raw --csv > gpurun_out/wix/cfg2_wix_raw.csv 2>/dev/null
  ncu -i gpurun_out/wix/cfg2_wix.ncu-rep --page details --csv > gpurun_out/wix/cfg2_wix_details.csv 2>/dev/null
  ncu -i gpurun_out/wix/cfg2_wix.ncu-rep --page source --csv > gpurun_out/wix/cfg2_wix_source.csv 2>/dev/null
  ls -la gpurun_out/wix
fi
