#!/bin/bash
# A/B: bench.py with each exp/libcsaw_<name>.so (CSAW_LIB), args after "--"
names=(); while [ "$1" != "--" ] && [ -n "$1" ]; do names+=("$1"); shift; done; shift
python -c "import __graft_entry__ as g; g.build()"
for rep in 1 2; do
for v in "${names[@]}"; do
  if [ $v = default ]; then unset CSAW_LIB; else export CSAW_LIB=$PWD/exp/libcsaw_$v.so; fi
  timeout 900 python bench.py "$@" > gpurun_out/ab_$v.json 2>&1
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
for l in open(f"gpurun_out/ab_{v}.json"):
    if l.startswith("{"):
        d = json.loads(l); r = d["roofline"]
        print(f"{v:12s} ms {d['ms_per_step']:.3f} SEPS {d['value']:.4g} frac {r.get('frac')} hot {r.get('hot_ms_per_launch')}")
        break
else:
    print(v, "FAILED", open(f"gpurun_out/ab_{v}.json").read()[-500:])
PY
done
done
