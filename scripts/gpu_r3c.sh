#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_weight.py tests/test_gpu_oom.py -x -q -k "mdrw or weight or oom or walk" 2>&1 | tail -1
timeout 600 python bench.py --config cfg5 --in-memory --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --scan-path-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg5', d['ms_per_step'])"
timeout 600 python bench.py --config cfg2 --no-cache --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --scan-path-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg2 stream', d['ms_per_step'])"
timeout 600 python bench.py --config cfg2_weight --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg2_weight', d['ms_per_step'])"
