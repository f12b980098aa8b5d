#!/bin/bash
# weights parity (fused mode fix) + cfg2 scan-path A/B (VU, bulk L2 prefetch)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2g_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_weight.py tests/test_gpu_wix.py tests/test_gpu_cache.py -x -q > gpurun_out/r2g_pytest.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/r2g_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for v in default vu8 vmin8 nopf; do
  if [ $v = default ]; then unset CSAW_LIB; else export CSAW_LIB=$PWD/exp/libcsaw_$v.so; fi
  timeout 600 python bench.py --config cfg2 --no-cache --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --scan-path-steps 0 > gpurun_out/r2g_stream_$v.json 2>&1
  python - $v <<'PY'
import json, sys
v = sys.argv[1]
for l in open(f"gpurun_out/r2g_stream_{v}.json"):
    if l.startswith("{"):
        d = json.loads(l); r = d["roofline"]
        print(v, "ms", d["ms_per_step"], "SEPS", d["value"], "frac", r["frac"], r["kernel"], r["hot_ms_per_launch"])
        break
else:
    print(v, "FAILED", open(f"gpurun_out/r2g_stream_{v}.json").read()[-1500:])
PY
done
