#!/bin/bash
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_n2v_index.py -x -q 2>&1 | tail -3
for v in default m5 m6; do
  if [ $v = default ]; then unset CSAW_LIB; else export CSAW_LIB=$PWD/exp/libcsaw_$v.so; fi
  timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r2d_$v.json 2>&1
  python - <<PY
import json
for l in open("gpurun_out/r2d_$v.json"):
    if l.startswith("{"):
        d=json.loads(l); r=d["roofline"]; print("$v", d["ms_per_step"], d["value"], r["frac"], r["alg_bytes_per_launch"], d["detail"]["cache"]["build_ms"], d["detail"]["cache"]["graph_device_bytes"])
PY
done
unset CSAW_LIB
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2d_e2e.json 2>&1
python -c "
import json
for l in open('gpurun_out/r2d_e2e.json'):
    if l.startswith('{'): d=json.loads(l); print('e2e', d['e2e'])
"
# ncu: launch list + one full capture of the index kernel
ncu --clock-control none --set full --import-source on -k regex:k_node2vec_idx -c 1 -o gpurun_out/r2d_n2x python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2d_ncu.log 2>&1
ncu -i gpurun_out/r2d_n2x.ncu-rep --page raw --csv > gpurun_out/r2d_n2x_raw.csv 2>/dev/null
ncu -i gpurun_out/r2d_n2x.ncu-rep --page details --csv > gpurun_out/r2d_n2x_details.csv 2>/dev/null
ncu -i gpurun_out/r2d_n2x.ncu-rep --page source --csv > gpurun_out/r2d_n2x_source.csv 2>/dev/null
ls -la gpurun_out/ | grep r2d
