#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_n2v_index.py tests/test_gpu_parity.py -x -q -k "node2vec or n2x or index" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q -k "cfg3" 2>&1 | tail -1
timeout 900 python scripts/strong_shares.py cfg3 2>/dev/null | grep "^| cfg3"
