#!/bin/bash
# weights (float path) + materialised degree-bias stream: parity, then cfg2 scan-path timings (A/B VU)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2f_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_weight.py -x -q > gpurun_out/r2f_pytest.log 2>&1; echo "weight tests rc=$?"; tail -15 gpurun_out/r2f_pytest.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2f_parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/r2f_parity.log
for v in default vu4; do
  if [ $v = default ]; then unset CSAW_LIB; else export CSAW_LIB=$PWD/exp/libcsaw_$v.so; fi
  timeout 600 python bench.py --config cfg2 --no-cache --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --scan-path-steps 0 > gpurun_out/r2f_stream_$v.json 2>&1
  python - $v <<'PY'
import json, sys
v = sys.argv[1]
for l in open(f"gpurun_out/r2f_stream_{v}.json"):
    if l.startswith("{"):
        d = json.loads(l); r = d["roofline"]
        print(v, "ms", d["ms_per_step"], "SEPS", d["value"], "frac", r["frac"], r["kernel"], r["hot_ms_per_launch"])
        break
else:
    print(v, "FAILED", open(f"gpurun_out/r2f_stream_{v}.json").read()[-1500:])
PY
done
unset CSAW_LIB
timeout 900 python bench.py --config cfg2 --no-cache --gather-bias --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --scan-path-steps 0 > gpurun_out/r2f_gather.json 2>&1
python -c "
import json
for l in open('gpurun_out/r2f_gather.json'):
    if l.startswith('{'): d=json.loads(l); print('gather ms', d['ms_per_step'], d['roofline']['kernel'])
"
