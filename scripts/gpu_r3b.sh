#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wix.py tests/test_gpu_cache.py tests/test_gpu_walk_variants.py tests/test_gpu_n2v_tri.py tests/test_gpu_streams.py -x -q 2>&1 | tail -1
timeout 600 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --scan-path-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg2', d['ms_per_step'])"
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --scan-path-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg3', d['ms_per_step'], 'scan', d['detail']['scan_path']['ms_per_step'])"
